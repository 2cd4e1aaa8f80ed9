// Persistent batched CTC beam-search kernel for sm_100a (the FlexCTC hot path).
//
// PAPER.md §III-C Algorithm 1 with Eq. (1), 1-best output:
//   per frame t < L_b:  candidates k·V'+w from every live hypothesis k and token w,
//   flat TopK, θ-prune, LM/BT state advance,
//   beams.update + RecombineHypotheses; then LM.Final, final merge and
//   backtrace of the token/pointer tensors.
//
// B200 design:
//  * one persistent CTA per in-flight utterance, utterances taken longest-first from a device
//    work queue (LPT); the whole frame loop runs in-kernel: zero host syncs, one launch;
//  * frame rows D[b,t,:] stream HBM -> shared memory with cp.async (16 B when aligned) in a ring
//    R frames ahead of the recurrence, so the only O(B·T·V') HBM stream overlaps it;
//  * exact pre-prune. Lower bound of the frame max mx: the blank and repeat candidates (no fusion
//    terms) and the exact candidates of the frame's best non-blank token from every live slot.
//    τ0 = fl(mx0 - θ) <= τ. A non-blank candidate is scored exactly (LM + boost lookups) only if
//    acc + D + ub(slot) can reach the running threshold (ub = β + α_LM·max_w P(w|lm state) +
//    α_BT·max_w delta(bt state) + rounding margin). Anything below is pruned by Alg. 1 anyway or
//    cannot enter the top K, so the live beam is bit-identical to the dense [K, V'] evaluation;
//  * survivors go to a shared-memory buffer of 64-bit keys (orderable fp32 score | ~flat index);
//    when it fills, a block radix-select keeps the top K and raises the threshold (threshold
//    algorithm): any candidate count (θ = ∞, flat frames) works in bounded memory;
//  * selection = radix-select of the K-th key + rank sort of <= K keys; ties go to the lower
//    flat index (reading R9) because the index is in the key;
//  * per-slot LM records (whole backoff chain, cumulative backoffs, bound, LM.Final) and boost
//    values are cached in shared memory and carried with the slot, so an LM query is one round of
//    parallel arc searches (all chain levels at once) plus one dense level-1 load;
//  * recombination on (64-bit prefix hash, last label) (R12), log-sum-exp in the canonical order
//    (R14) with exp/log1p evaluated in fp64 and rounded once;
//  * backpointers u8 parent + u16 label per (t, k) plus per-32-frame chunk ancestors, so the
//    backtrace walks chunks in parallel (T/32 + 32 dependent loads, not T).
//  * K <= 32 ("solo"): warp 0 runs the slot-serial phases alone with warp-level sync; warps 1-7
//    stream the rows and precompute each frame's summary one frame ahead, and join only for
//    frames with many listed tokens;
//  * compile-time variants for the paper's shape (V' = 1025, K = 16, 4-gram records, LM +
//    boosting, "plain" options): the frame step is a chain of short dependent steps, so folding
//    runtime bounds and branches out of it shortens every frame (A/B log in DESIGN.md §7).
// All score arithmetic uses __fadd_rn/__fmaf_rn in the canonical order of reading R19 (no
// contraction, no fast-math), so max-mode scores are bit-identical to the fp32 oracle.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <string>

#include "device_common.cuh"
#include "flexctc_internal.h"

namespace flexctc {
namespace {

using namespace dev;

// Per-phase SM-cycle counters (device stats words 10-22) cost ~100 instructions per frame on the
// beam warp; they are compiled in only with -DFLEXCTC_PHASE_TIMERS (build.py --timers).
#ifdef FLEXCTC_PHASE_TIMERS
#define TCLK() clock64()
#else
#define TCLK() 0ll
#endif

constexpr int kDenseMinTokens = 24;  // listed tokens per frame that switch to LM rows (when enabled)


// one bank of per-slot state (two banks, swapped every frame)
struct Bank {
    float* acc; int* last; uint64_t* hash; int* lms; int* bts; uint8_t* anc;
    int* rec;     // [K][RWS] cached LM record of lms
    float* btm;   // [K][2]  {maxd, U} of bts
};

struct Shared {
    float* ring;
    unsigned char* rring;  // [R][kCmpBytes] frame records (use_cmp)
    Bank bk;  // bank 0; bank 1 of every field starts `K` (or K*stride) elements later
    uint64_t* ckey; int* clm; int* cbt;   // candidate buffer [cap]
    uint64_t* skey; int* slm; int* sbt;   // selection [K]
    uint16_t* toks;
    int* alive_idx;
    uint32_t* hist;
    int* endslot;
};

struct Scalars {
    int nbuf, m, nalive, nsel, u, npair, excl, scan, fast;
    float thr, ubvmax, dthr;
    uint64_t kth;
    float rf[4][32];
    uint64_t rk[32];
    int ri[32];
};

// Group-level primitives. A group is either the whole CTA (G = blockDim) or warp 0 alone
// (G = 32, the beam warp of the K <= 32 kernel mode); gsync is the matching barrier.
__device__ __forceinline__ void gsync(int G) {
    if (G == 32) __syncwarp(); else __syncthreads();
}

__device__ __forceinline__ float block_max(float v, Scalars& sc, int G) {
    const int NW = G >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (NW == 1) return v;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sc.rf[0][wid] = v;
    __syncthreads();
    float r = sc.rf[0][0];
    for (int i = 1; i < NW; ++i) r = fmaxf(r, sc.rf[0][i]);
    return r;
}

// Phase-1 reduction in one round: max of three floats, max of a u64 key, exclusive scan of a
// 0/1 flag (slot order). Returns via references.
// k_uniform: k is already the same on every lane (the helpers' frame summary): not reduced.
__device__ __forceinline__ void block_reduce_p1(float& a, float& b, float& c, uint64_t& k, bool flag, int& off,
                                                int& tot, Scalars& sc, int G, bool k_uniform = false) {
    const int NW = G >> 5;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
        b = fmaxf(b, __shfl_xor_sync(0xffffffffu, b, o));
        c = fmaxf(c, __shfl_xor_sync(0xffffffffu, c, o));
        if (!k_uniform) k = umax64(k, __shfl_xor_sync(0xffffffffu, k, o));
    }
    const unsigned bal = __ballot_sync(0xffffffffu, flag);
    const int in_warp = __popc(bal & ((1u << lane) - 1u));
    if (NW == 1) {
        off = in_warp;
        tot = __popc(bal);
        return;
    }
    __syncthreads();
    if (lane == 0) {
        sc.rf[0][wid] = a; sc.rf[1][wid] = b; sc.rf[2][wid] = c; sc.rk[wid] = k;
        sc.ri[wid] = __popc(bal);
    }
    __syncthreads();
    a = sc.rf[0][0]; b = sc.rf[1][0]; c = sc.rf[2][0]; k = sc.rk[0];
    int base = 0, all = 0;
    for (int i = 0; i < NW; ++i) {
        if (i) { a = fmaxf(a, sc.rf[0][i]); b = fmaxf(b, sc.rf[1][i]); c = fmaxf(c, sc.rf[2][i]); k = umax64(k, sc.rk[i]); }
        if (i < wid) base += sc.ri[i];
        all += sc.ri[i];
    }
    off = base + in_warp;
    tot = all;
}

// exclusive prefix over the group of per-thread counts; returns the offset, total in *tot
__device__ __forceinline__ int block_exscan(int v, int* tot, Scalars& sc, int G) {
    const int NW = G >> 5;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (NW == 1) {
        *tot = __shfl_sync(0xffffffffu, x, 31);
        return x - v;
    }
    __syncthreads();
    if (lane == 31) sc.ri[wid] = x;
    __syncthreads();
    int base = 0, all = 0;
    for (int i = 0; i < NW; ++i) {
        if (i < wid) base += sc.ri[i];
        all += sc.ri[i];
    }
    *tot = all;
    return base + x - v;
}

// Radix select over n unique 64-bit keys in smem: returns kth such that exactly K keys are
// >= kth (requires n > K). MSB-first 8-bit digits; stops as soon as the boundary bin is exact.
__device__ uint64_t radix_kth(const uint64_t* keys, int n, int K, Shared& sm, Scalars& sc, int G) {
    uint64_t prefix = 0, mask = 0;
    int remaining = K;
    for (int shift = 56; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += G) sm.hist[i] = 0;
        gsync(G);
        for (int i = threadIdx.x; i < n; i += G) {
            const uint64_t k = keys[i];
            if ((k & mask) == prefix) atomicAdd(&sm.hist[(k >> shift) & 255u], 1u);
        }
        gsync(G);
        if (threadIdx.x < 32) {
            const int lane = threadIdx.x;  // lane l owns digits 255-8l .. 248-8l (descending)
            uint32_t c[8];
            uint32_t s = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) { c[j] = sm.hist[255 - 8 * lane - j]; s += c[j]; }
            uint32_t incl = s;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const uint32_t above = incl - s;
            if (above < (uint32_t)remaining && (uint32_t)remaining <= incl) {
                uint32_t a = above;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (a < (uint32_t)remaining && (uint32_t)remaining <= a + c[j]) {
                        sc.kth = (uint64_t)(255 - 8 * lane - j);
                        sc.ri[0] = (int)((uint32_t)remaining - a);
                        sc.ri[1] = (int)c[j];
                    }
                    a += c[j];
                }
            }
        }
        gsync(G);
        const uint64_t d = sc.kth;
        const int need = sc.ri[0], inbin = sc.ri[1];
        gsync(G);
        prefix |= d << shift;
        mask |= 255ull << shift;
        remaining = need;
        if (need == inbin) return prefix;
    }
    return prefix;
}

// K-th largest of n unique keys (n >= K) by rank counting: every key's rank is the number of
// larger keys; the key of rank K-1 is the answer. O(n^2 / G) shared loads, used for small n.
__device__ __forceinline__ uint64_t kth_by_rank(const uint64_t* keys, int n, int K, Scalars& sc, int G) {
    uint64_t res = 0;
    for (int i = threadIdx.x; i < n; i += G) {
        const uint64_t ki = keys[i];
        int r = 0;
        for (int j = 0; j < n; ++j) r += keys[j] > ki ? 1 : 0;
        if (r == K - 1) res = ki;
    }
    if (G == 32) {
#pragma unroll
        for (int o = 16; o; o >>= 1) res = umax64(res, __shfl_xor_sync(0xffffffffu, res, o));
        return res;
    }
    if (res) sc.kth = res;  // exactly one thread holds it (keys are unique and never 0)
    __syncthreads();
    res = sc.kth;
    __syncthreads();
    return res;
}

// Move the keys >= kth (exactly K of them) from the candidate buffer into the selection arrays.
__device__ void gather_selected(int n, uint64_t kth, Shared& sm, Scalars& sc, int G) {
    if (threadIdx.x == 0) sc.nsel = 0;
    gsync(G);
    for (int i = threadIdx.x; i < n; i += G) {
        const uint64_t k = sm.ckey[i];
        if (k >= kth) {
            const int j = atomicAdd(&sc.nsel, 1);
            sm.skey[j] = k; sm.slm[j] = sm.clm[i]; sm.sbt[j] = sm.cbt[i];
        }
    }
    gsync(G);
}

__device__ __forceinline__ void push_cand(Shared& sm, Scalars& sc, uint64_t key, int lmn, int btn) {
    const int j = atomicAdd(&sc.nbuf, 1);
    sm.ckey[j] = key; sm.clm[j] = lmn; sm.cbt[j] = btn;
}

// Pull the LM record and boost values of a candidate's next state into L1 when the candidate is
// pushed, so that beams.update (phase 6) finds them there if the candidate is selected.
__device__ __forceinline__ void prefetch_state(const DecodeParams& p, int ln, int bn) {
    if (p.use_lm && ln >= 0)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(p.lm.rec + (size_t)ln * (p.lm.RW / 4)));
    if (p.use_bt) {
        asm volatile("prefetch.global.L1 [%0];" ::"l"(p.bt.maxd + bn));
        asm volatile("prefetch.global.L1 [%0];" ::"l"(p.bt.U + bn));
    }
}

// barrier among the helper warps only (named barrier 2)
__device__ __forceinline__ void helpers_sync(int n) { asm volatile("bar.sync 2, %0;" ::"r"(n) : "memory"); }

// Fill an LM row: row[w] = log P(w | state) for every decoder token w, in exactly the fp32
// arithmetic of lm_query (dense level-1 path first, then arc levels from the shortest context to
// the longest so the longest listed context wins). Coalesced reads of the level-1 table.
template <int NT>
__device__ void build_lm_row(const LmDev& lm, int state, float* row, int V) {
    const int4* r4 = lm.rec + (size_t)state * (lm.RW / 4);
    const int4 h0 = __ldg(&r4[0]);
    const int n = h0.x, u = h0.y;
    const float cum_u = __int_as_float(h0.z), cum_root = __int_as_float(h0.w);
    if (u >= 0) {
        const int2* d = lm.dense + (size_t)u * V;
        for (int w = threadIdx.x; w < V; w += NT) {
            const int2 e = __ldg(&d[w]);
            row[w] = __fadd_rn((e.y & 0x80000000) ? cum_u : cum_root, __int_as_float(e.x));
        }
    } else {
        for (int w = threadIdx.x; w < V; w += NT) row[w] = __fadd_rn(cum_root, __ldg(&lm.uni_lp[w]));
    }
    const int* ri = (const int*)r4;
    for (int j = n - 1; j >= 0; --j) {
        __syncthreads();
        const int off = __ldg(&ri[8 + 3 * j]), deg = __ldg(&ri[8 + 3 * j + 1]);
        const float cum = __int_as_float(__ldg(&ri[8 + 3 * j + 2]));
        for (int a = threadIdx.x; a < deg; a += NT) {
            const int4 arc = __ldg(&lm.arcs[off + a]);
            row[arc.x] = __fadd_rn(cum, __int_as_float(arc.y));
        }
    }
}

// SOLO (K <= 32, NT >= 128, 4-row ring; chosen on the host): warp 0 is the beam warp, the other
// warps are helpers. A template parameter so the group size of the slot-parallel phases is a
// compile-time constant.
// compile-time V', K, LM record width (0 = runtime); FUS (0 = runtime): bit 0 LM, bit 1 boosting,
// bit 2 "plain" = no LM-row cache (nrow 0), log-sum-exp merges, non-negative fusion weights; bit 3 =
// read the compaction records (FLEXCTC_CMP=1)
template <int NT, int LMV, bool SOLO, int VPC = 0, int KC = 0, int RWC = 0, int FUS = 0>
__global__ void __launch_bounds__(NT, 1) ctc_beam_kernel(const DecodeParams p, const int ring_rows, const int cap,
                                                      int nrow, const int dense_min) {
    constexpr int kRec = (8 + 3 * LMV + 3) & ~3;  // ints per cached LM record
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ Scalars sc;
    __shared__ int s_line[kMaxBeam];       // per alive position: row-cache line (-1 = sparse path)
    __shared__ float4 s_pos[kMaxBeam];     // per alive position: {acc, ub, |ub terms|, last}
    __shared__ float s_ubnl[kMaxBeam];     // per alive position: ub without the LM term
    __shared__ float2 s_suf[kMaxBeam];     // suffix max over positions of {acc, |ub terms|}
    constexpr int kPairCap = 2 * NT;       // viable (position, token) pairs per evaluation batch
    __shared__ uint32_t s_pairs[kPairCap];
    constexpr int kTab = NT > 32 ? 2 * NT : 1;  // recombination table (NT > 32)
    constexpr int kTabMem = 3;
    __shared__ int s_tocc[kTab];  // slot + 1 of the entry's first member (0 = empty)
    __shared__ int s_tcnt[kTab];
    __shared__ int s_tmem[kTab * kTabMem];
    __shared__ int s_build[2 * 32];        // rows to build: (line, state)
    __shared__ int s_nbuild;
    // solo mode (K <= 32, NT > 32): warp 0 runs the slot-serial phases with warp-level sync;
    // warps 1.. ("helpers") stream the rows and precompute each frame's summary one frame ahead
    // (best non-blank token + every token within kListDelta of it, up to kListCap), and join the
    // beam warp only for frames whose candidate list the summary cannot provide.
    constexpr int kListCap = 32;
    constexpr float kListDelta = 16.0f;
    constexpr int kRing = 4;  // frame rows in flight (cp.async ring; R = kRing for V' <= 2048)
    __shared__ unsigned long long s_sum_key[kRing];
    __shared__ float s_sum_floor[kRing];
    __shared__ int s_sum_cnt[kRing];
    __shared__ int s_list_tok[kRing * kListCap];
    __shared__ float s_list_d[kRing * kListCap];
    __shared__ unsigned long long s_hkey[32];
    const int tid = threadIdx.x;
    const int K = KC ? KC : p.K, Vp1 = VPC ? VPC : p.Vp1, blank = Vp1 - 1, V = Vp1 - 1;
    const int VP = (Vp1 + 3) & ~3;
    const int R = ring_rows;
    const bool lm_on = FUS ? (FUS & 1) != 0 : p.use_lm != 0, bt_on = FUS ? (FUS & 2) != 0 : p.use_bt != 0;
    const int RWS = RWC ? RWC : lm_on ? ((p.lm.RW + 3) & ~3) : 4;  // ints per cached record (int4 aligned)
    constexpr bool plain = (FUS & 4) != 0;
    // FUS bit 4: bf16 logits read straight into the ring (2 B per logit from HBM) and normalised in
    // shared memory with the lse of the frame's compaction record (R25); the specialised north-star
    // variant only (solo, V' = 1025, 8 warps: 224 helper threads convert <= 5 elements each)
    constexpr bool lgt = (FUS & 16) != 0;
    static_assert(!lgt || (SOLO && VPC == 1025 && NT == 256 && (FUS & 8)), "bf16 rows: the records variant only");
    constexpr int kConv = lgt ? (VPC + NT - 33) / (NT - 32) : 1;  // elements per helper thread
    const int RS = VP + (lgt ? 20 : 4);  // ring slot stride (floats); bf16 rows are staged at byte kStage
    const int kStage = (2 * VP + 32 + 15) & ~15;
    const bool ub_inf = plain ? false : (lm_on && p.alpha_lm < 0.0f) || (bt_on && p.alpha_bt < 0.0f);
    // compaction records: the generic variants follow p.use_cmp; specialised ones compile them in
    // (FUS bit 3) or out
    const bool use_cmp = FUS ? (FUS & 8) != 0 : p.use_cmp != 0;
    const int merge_mode = plain ? 0 : p.merge_mode;
    if (plain) nrow = 0;
    constexpr bool solo = SOLO;  // host: K <= 32 && NT >= 128 && R == kRing && !solo_off (>= 3 helper warps)
    constexpr int kPfSolo = kRing - 2;  // solo mode: helpers copy row t + 2 while the beam warp reads row t
    const bool helper = solo && tid >= 32;
    const bool bw = !solo || tid < 32;               // takes part in the slot-serial phases
    const int ltid = helper ? tid - 32 : tid;        // row loader index / count
    const int lnt = solo ? NT - 32 : NT;
    uint32_t st[kNumStats] = {};
    int ready = 0;  // streamed input: frames known to have landed (wait_ready)
    // bf16 logits (lgt): the tensor's byte range (rows whose covering 16-B blocks leave it are
    // copied element by element)
    const char* lg_lo = lgt ? (const char*)p.logits : nullptr;
    const char* lg_hi = lgt ? lg_lo + 2 * ((size_t)(p.B - 1) * p.stride_b + (size_t)(p.T - 1) * p.stride_t + Vp1) : nullptr;

    Shared sm;
    float* rowval = nullptr;  // [nrow][VP] LM rows (row cache)
    int* rowtag = nullptr;    // [nrow] LM state of each line (-1 = empty)
    int2* btroot = nullptr;   // [V] boost transition row of the root {next, delta}
    {
        unsigned char* q = smem_raw;
        auto take = [&](size_t bytes) { unsigned char* r = q; q += (bytes + 15) & ~size_t(15); return r; };
        sm.ring = (float*)take(sizeof(float) * (size_t)R * RS);
        sm.rring = (unsigned char*)take(p.use_cmp ? (size_t)R * kCmpBytes : 0);
        {
            Bank& B = sm.bk;  // both banks of each field, contiguous
            B.acc = (float*)take(8 * K); B.last = (int*)take(8 * K); B.hash = (uint64_t*)take(16 * K);
            B.lms = (int*)take(8 * K); B.bts = (int*)take(8 * K); B.anc = (uint8_t*)take(2 * K);
            B.rec = (int*)take(8 * (size_t)K * RWS); B.btm = (float*)take(16 * K);
        }
        sm.ckey = (uint64_t*)take(8 * (size_t)cap); sm.clm = (int*)take(4 * (size_t)cap); sm.cbt = (int*)take(4 * (size_t)cap);
        sm.skey = (uint64_t*)take(8 * K); sm.slm = (int*)take(4 * K); sm.sbt = (int*)take(4 * K);
        sm.toks = (uint16_t*)take(2 * (size_t)Vp1);
        sm.alive_idx = (int*)take(4 * K);
        sm.hist = (uint32_t*)take(4 * 256);
        sm.endslot = (int*)take(4 * (size_t)p.nch);
        if (nrow > 0) {
            rowval = (float*)take(4 * (size_t)nrow * VP);
            rowtag = (int*)take(4 * (size_t)nrow);
        }
        if (bt_on) btroot = (int2*)take(8 * (size_t)V);
    }
    for (int i = tid; i < nrow; i += NT) rowtag[i] = -1;
    if (bt_on)
        for (int w = tid; w < V; w += NT) btroot[w] = __ldg(&p.bt.tab[w]);
    auto bank = [&](int z) {
        Bank B;
        B.acc = sm.bk.acc + z * K; B.last = sm.bk.last + z * K; B.hash = sm.bk.hash + z * K;
        B.lms = sm.bk.lms + z * K; B.bts = sm.bk.bts + z * K; B.anc = sm.bk.anc + z * K;
        B.rec = sm.bk.rec + (size_t)z * K * RWS; B.btm = sm.bk.btm + z * 2 * K;
        return B;
    };

    auto recof = [&](const Bank& B, int k) -> int* { return B.rec + (size_t)k * RWS; };  // slot k's LM record
    // exact candidate score of a non-blank, non-repeat token w from slot k (Eq. (1), R19 order)
    // With `row` (a cached LM row of the slot's state) the LM value comes from shared memory and
    // the next LM state is deferred (ln = -1) until the candidate is selected.
    auto eval = [&](const Bank& cur, int k, float s0, int w, int& ln, int& bn, const float* row) -> float {
        float s = __fadd_rn(s0, p.beta);
        ln = cur.lms[k];
        bn = cur.bts[k];
        int2 e = make_int2(0, 0);
        if (bt_on) e = bn == 0 ? btroot[w] : __ldg(&p.bt.tab[(size_t)bn * V + w]);  // issued first
        if (lm_on) {
            float lp;
            if (row) { lp = row[w]; ln = -1; }
            else lp = lm_query<LMV>(p.lm, recof(cur, k), w, ln);
            s = __fmaf_rn(p.alpha_lm, lp, s);
        }
        if (bt_on) { bn = e.x; s = __fmaf_rn(p.alpha_bt, __int_as_float(e.y), s); }
        return s;
    };

    for (;;) {
        // ------------------------------------------------------------ next utterance (LPT queue)
        __syncthreads();
        if (tid == 0) sc.u = (int)atomicAdd(&p.flags[1], 1u);
        __syncthreads();
        const int u = sc.u;
        if (u >= p.B) break;
        const int b = p.order[u];
        const int L = p.len_c[b];
        const float* Db = p.log_probs + (int64_t)b * p.stride_b;
        const uint16_t* Lb = lgt ? p.logits + (int64_t)b * p.stride_b : nullptr;
        if (tid == 0) sc.fast = 0;
        ready = 0;  // streamed input: what this thread has seen landed, per utterance
        const int64_t bp_base = (int64_t)b * p.T * K;  // backpointers of this utterance

        // ------------------------------------------------------------ init (Alg. 1)
        {
            const Bank c0 = bank(0);
            for (int k = tid; k < K; k += NT) {
                c0.acc[k] = k == 0 ? 0.0f : kNeg;  // acc_scores[:,0] = 0, else -inf
                c0.last[k] = blank;                 // R6
                c0.hash[k] = 0ull;
                c0.lms[k] = p.lm.start;             // LM(<SOS>)
                c0.bts[k] = 0;                      // BT(<0>) = root
                c0.anc[k] = 0;
            }
            if (lm_on)
                for (int i = tid; i < RWS / 4; i += NT)
                    ((int4*)c0.rec)[i] = __ldg(&p.lm.rec[(size_t)p.lm.start * (p.lm.RW / 4) + i]);
            if (tid == 0) {
                c0.btm[0] = bt_on ? __ldg(&p.bt.maxd[0]) : 0.0f;
                c0.btm[1] = bt_on ? __ldg(&p.bt.U[0]) : 0.0f;
            }
        }
        // Row prefetch: in solo mode the helper warps own the ring (distance R - 2, so the beam warp
        // can still read rows t - 1 and t while helpers fill row t + 2); otherwise all threads (distance R - 1).
        const int pf = solo ? kPfSolo : R - 1;
        if (!solo || helper)
            for (int r = 0; r < pf; ++r) {  // prologue
                if (r < L) {
                    wait_ready(p, u, r, ready);
                    if (lgt) load_row_bf16((char*)(sm.ring + (size_t)(r & (R - 1)) * RS) + kStage, Lb + (int64_t)r * p.stride_t, Vp1, ltid, lnt, lg_lo, lg_hi);
                    else load_row(sm.ring + (size_t)(r & (R - 1)) * RS, Db + (int64_t)r * p.stride_t, Vp1, ltid, lnt, p.overread);
                    if (use_cmp && ltid < kCmpBytes / 16)
                        cp_async16(sm.rring + (size_t)(r & (R - 1)) * kCmpBytes + 16 * ltid,
                                   p.cmp + ((int64_t)b * p.T + r) * kCmpBytes + 16 * ltid);
                }
                cp_commit();
            }

        int cbank = 0;      // current bank (every thread tracks it, helpers included)
        bool flip = false;  // the previous frame wrote the other bank (a fast-path frame updates in place)
        for (int t = 0; t < L; ++t) {
            if (flip) cbank ^= 1;
            flip = true;
            const int cb = cbank;
            const Bank cur = bank(cb);
            const Bank nxt = bank(cb ^ 1);
            const long long ctop = TCLK();
            const int slot = t & (R - 1);  // R is 4 or 2
            float* ring_t = sm.ring + (size_t)slot * RS;
            const float* row = lgt ? ring_t : ring_t + row_off(Db + (int64_t)t * p.stride_t);
            if (!solo || helper) {
                const int r = t + pf;
                if (r < L) {
                    wait_ready(p, u, r, ready);
                    if (lgt) load_row_bf16((char*)(sm.ring + (size_t)(r & (R - 1)) * RS) + kStage, Lb + (int64_t)r * p.stride_t, Vp1, ltid, lnt, lg_lo, lg_hi);
                    else load_row(sm.ring + (size_t)(r & (R - 1)) * RS, Db + (int64_t)r * p.stride_t, Vp1, ltid, lnt, p.overread);
                    if (use_cmp && ltid < kCmpBytes / 16)
                        cp_async16(sm.rring + (size_t)(r & (R - 1)) * kCmpBytes + 16 * ltid,
                                   p.cmp + ((int64_t)b * p.T + r) * kCmpBytes + 16 * ltid);
                }
                cp_commit();
                if (solo) cp_wait<kPfSolo>(); else if (R == 4) cp_wait<3>(); else cp_wait<1>();
            }
            // the compaction pass's record of frame t (use_cmp): D[blank], the listed tokens sorted by
            // (D desc, token asc) and floor >= every unlisted D; n = 0 with floor = +inf: no usable list
            const unsigned char* rc_t = sm.rring + (size_t)slot * kCmpBytes;
            if (helper) {
                // frame summary for the beam warp: best non-blank token and the complete list of
                // tokens within kListDelta of it (capped at 32; the count says when it overflowed)
                // or, with records, the record's list (band <= 16 nats, <= 32 tokens) and floor
                const int h = ltid;
                helpers_sync(lnt);  // every helper's cp.async of row t (and record) has landed
                if constexpr (lgt) {
                    // D = (float)(x - lse) (R25) into the slot's float row: read every staged logit
                    // first (the float row overlaps the staging bytes), then write
                    const double lse = *(const double*)(rc_t + 16);
                    const char* sb = (const char*)ring_t + kStage + ((uintptr_t)(Lb + (int64_t)t * p.stride_t) & 15);
                    float xv[kConv];
#pragma unroll
                    for (int i = 0; i < kConv; ++i) {
                        const int w = h + i * (NT - 32);
                        xv[i] = w < Vp1 ? bf16f(*(const uint16_t*)(sb + 2 * w)) : 0.0f;
                    }
                    helpers_sync(lnt);
#pragma unroll
                    for (int i = 0; i < kConv; ++i) {
                        const int w = h + i * (NT - 32);
                        if (w < Vp1) ring_t[w] = (float)((double)xv[i] - lse);
                    }
                    helpers_sync(lnt);
                }
                const int rn = use_cmp ? ((const int*)rc_t)[2] : 0;
                const float rfl = use_cmp ? ((const float*)rc_t)[1] : INFINITY;
                if (use_cmp && !(rn == 0 && rfl == INFINITY)) {
                    const float* rv = (const float*)(rc_t + 32);
                    const uint16_t* rt = (const uint16_t*)(rc_t + 160);
                    if (h < rn) { s_list_tok[slot * kListCap + h] = rt[h]; s_list_d[slot * kListCap + h] = rv[h]; }
                    if (h == 0) {
                        s_sum_cnt[slot] = rn;
                        s_sum_floor[slot] = rfl;
                        s_sum_key[slot] = rn > 0 ? make_key(rv[0], (uint32_t)rt[0]) : make_key(kNeg, 0u);
                    }
                } else {
                float bv = kNeg;
                int bi = -1;
                for (int w = h; w < blank; w += lnt) {
                    const float v = row[w];
                    if (v > bv || bi < 0) { bv = v; bi = w; }
                }
                uint64_t key = bi >= 0 ? make_key(bv, (uint32_t)bi) : 0ull;
#pragma unroll
                for (int o = 16; o; o >>= 1) key = umax64(key, __shfl_xor_sync(0xffffffffu, key, o));
                if ((tid & 31) == 0) s_hkey[(tid >> 5) - 1] = key;
                if (h == 0) s_sum_cnt[slot] = 0;  // ordered before the list atomics by the barrier
                helpers_sync(lnt);
                uint64_t best = s_hkey[0];
                for (int i = 1; i < (lnt >> 5); ++i) best = umax64(best, s_hkey[i]);
                const float dmax = score_of(best);
                const float floor_ = __fsub_rn(dmax, kListDelta);
                for (int w0 = 0; w0 < blank; w0 += lnt) {
                    const int w = w0 + h;
                    const bool hit = w < blank && row[w] >= floor_;
                    const unsigned bal = __ballot_sync(0xffffffffu, hit);
                    if (bal) {
                        int base = 0;
                        if ((tid & 31) == 0) base = atomicAdd(&s_sum_cnt[slot], __popc(bal));
                        base = __shfl_sync(0xffffffffu, base, 0);
                        const int q = base + __popc(bal & ((1u << (tid & 31)) - 1u));
                        if (hit && q < kListCap) { s_list_tok[slot * kListCap + q] = w; s_list_d[slot * kListCap + q] = row[w]; }
                        // the list overflowed: the beam warp only tests count > kListCap, so this
                        // warp's further hits change nothing
                        if (base + __popc(bal) > kListCap) break;
                    }
                }
                if (h == 0) { s_sum_key[slot] = best; s_sum_floor[slot] = floor_; }
                }  // no usable record
            }
            if (tid == 0) { sc.nbuf = 0; sc.m = 0; sc.npair = 0; }
            __syncthreads();  // B0: row t and its summary are ready
            const long long c0 = TCLK();
            if (tid == 0) st[kCycTop] += (uint32_t)(c0 - ctop);

            const int G = solo ? 32 : NT;  // group of the slot-parallel phases
            long long tp1 = c0, tp2 = c0, tp3 = c0;  // phase boundaries (timers build, thread 0)
            bool stage_a = false;
            int wstar = -1;
            // Settled-beam fast path (K <= 32, beam warp): every live slot's last label is blank, the
            // live slots are a prefix in (score desc, slot asc) order after adding D[blank], and no
            // non-blank token can reach fl(max - θ) (the token filter of phase 3 with thr = τ0). Then
            // Alg. 1 reduces to acc_k += D[blank] for every slot (no repeat candidates, no emission,
            // TopK = the slots in their own order, no recombination: the (hash, blank) keys are
            // distinct) and the θ-prune; the bank is updated in place.
            bool fast = false;
            if (solo && bw && !p.fast_off) {
                const float a = tid < K ? cur.acc[tid] : kNeg;
                const bool al = a > kNeg;
                const int lk = tid < K ? cur.last[tid] : blank;
                const unsigned am = __ballot_sync(0xffffffffu, al);
                const int na = __popc(am);
                const float nw = al ? __fadd_rn(a, row[blank]) : kNeg;
                const float nx = __shfl_down_sync(0xffffffffu, nw, 1);
                bool ok = (!al || lk == blank) && (tid + 1 >= na || nw >= nx);
                ok = __all_sync(0xffffffffu, ok) && na > 0 && am == (na == 32 ? 0xffffffffu : (1u << na) - 1u);
                if (ok) {
                    float ub = kNeg;
                    if (al) {
                        ub = p.beta;
                        if (lm_on) ub += p.alpha_lm * __int_as_float(recof(cur, tid)[4]);
                        if (bt_on) ub += p.alpha_bt * cur.btm[2 * tid];
                        if (ub_inf) ub = INFINITY;
                    }
                    const float accmax = score_of((uint64_t)__reduce_max_sync(0xffffffffu, ord_of(al ? a : kNeg)) << 32);
                    const float ubvmax = score_of((uint64_t)__reduce_max_sync(0xffffffffu, ord_of(ub)) << 32);
                    const float mx = __shfl_sync(0xffffffffu, nw, 0);
                    const float tau0 = __fsub_rn(mx, p.theta);
                    const float dstar = score_of(s_sum_key[slot]);
                    const float mg = 1e-4f * (1.0f + fabsf(tau0) + fabsf(accmax) + fabsf(ubvmax));
                    const float dthr = __fsub_rn(__fsub_rn(__fsub_rn(tau0, accmax), ubvmax), mg);
                    fast = mx > kNeg && !(dstar >= dthr);
                    if (fast && tid < K) {
                        const int64_t bpo = bp_base + (int64_t)(t * K);
                        uint8_t my_anc = 0;
                        if (al && nw >= tau0) {  // survives the θ-prune: parent = itself, label = blank
                            cur.acc[tid] = nw;
                            my_anc = (t % kChunk == 0) ? (uint8_t)tid : cur.anc[tid];
                            cur.anc[tid] = my_anc;
                            p.bp_parent[bpo + tid] = (uint8_t)tid;
                            p.bp_label[bpo + tid] = (uint16_t)blank;
                        } else if (al) {
                            cur.acc[tid] = kNeg; cur.last[tid] = blank; cur.hash[tid] = 0ull;
                            cur.lms[tid] = 0; cur.bts[tid] = 0; cur.anc[tid] = 0;
                        }
                        if ((t % kChunk) == kChunk - 1 || t == L - 1)
                            p.chunk_anc[((int64_t)b * p.nch + t / kChunk) * K + tid] = my_anc;
                    }
                }
                if (tid == 0) {
                    sc.fast = fast ? 1 : 0;
                    if (fast) { sc.scan = 0; sc.m = 0; st[kFastFrames] += 1; st[kFrames] += 1; }
                }
            }
            if (bw && !fast) {
                // ------------------------------------------------ phase 1: exact blank/repeat candidates,
                // per-slot bounds, frame argmax over non-blank tokens, alive list
                float a = kNeg, sbk = kNeg, srk = kNeg, ubk = kNeg;
                int lk = blank;
                bool al = false;
                if (tid < K) {
                    a = cur.acc[tid];
                    al = a > kNeg;
                    lk = cur.last[tid];
                    if (al) {
                        sbk = __fadd_rn(a, row[blank]);                 // blank: no β / fusion
                        if (lk != blank) srk = __fadd_rn(a, row[lk]);    // repeat: no β / fusion
                        if (lk != blank && p.fuse_rep) {
                            // P:167 variant: the repeated emission is scored by the LM / BT at every
                            // occurrence (R19 order, no β; the states do not advance)
                            if (bt_on) {
                                const int2 e = cur.bts[tid] == 0 ? btroot[lk] : __ldg(&p.bt.tab[(size_t)cur.bts[tid] * V + lk]);
                                if (lm_on) {
                                    int nx;
                                    srk = __fmaf_rn(p.alpha_lm, lm_query<LMV>(p.lm, recof(cur, tid), lk, nx), srk);
                                }
                                srk = __fmaf_rn(p.alpha_bt, __int_as_float(e.y), srk);
                            } else if (lm_on) {
                                int nx;
                                srk = __fmaf_rn(p.alpha_lm, lm_query<LMV>(p.lm, recof(cur, tid), lk, nx), srk);
                            }
                        }
                        float ub = p.beta;
                        if (lm_on) ub += p.alpha_lm * __int_as_float(recof(cur, tid)[4]);
                        if (bt_on) ub += p.alpha_bt * cur.btm[2 * tid];
                        ubk = ub_inf ? INFINITY : ub;
                    }
                }
                uint64_t best_tok = 0;
                if (solo) {
                    best_tok = s_sum_key[slot];
                } else if (use_cmp && !(((const int*)rc_t)[2] == 0 && ((const float*)rc_t)[1] == INFINITY)) {
                    // the record's best listed token (every unlisted one is <= floor <= it)
                    const int rn = ((const int*)rc_t)[2];
                    best_tok = rn > 0 ? make_key(((const float*)(rc_t + 32))[0], (uint32_t)((const uint16_t*)(rc_t + 160))[0])
                                      : make_key(kNeg, 0u);
                } else {
                    float bv = kNeg;
                    int bi = -1;
                    for (int w = tid; w < blank; w += NT) {  // blank is the last index (R1)
                        const float v = row[w];
                        if (v > bv || bi < 0) { bv = v; bi = w; }
                    }
                    if (bi >= 0) best_tok = make_key(bv, (uint32_t)bi);
                }
                float mxrb = fmaxf(sbk, srk), accmax = a, ubvmax = ubk;
                int aoff, nalive;
                block_reduce_p1(mxrb, accmax, ubvmax, best_tok, al, aoff, nalive, sc, G, solo);
                if (al) sm.alive_idx[aoff] = tid;
                wstar = (int)flat_of(best_tok);
                const float dstar = score_of(best_tok);
                gsync(G);

                // ------------------------------------------------ phase 2: exact candidates of the frame's
                // best non-blank token (tightens the lower bound of the frame max on emission frames)
                const long long cp2 = TCLK();
                tp1 = cp2;
                float tau0 = __fsub_rn(mxrb, p.theta);
                if (nalive > 0 && mxrb > kNeg) {
                    const float reach = __fadd_rn(__fadd_rn(accmax, dstar), ubvmax) +
                                        1e-4f * (1.0f + fabsf(accmax) + fabsf(dstar) + fabsf(ubvmax));
                    stage_a = reach >= mxrb;
                }
                float sA = kNeg;
                int lnA = 0, bnA = 0, kA = -1;
                if (stage_a) {
                    if (tid < nalive) {
                        kA = sm.alive_idx[tid];
                        if (wstar != cur.last[kA]) sA = eval(cur, kA, __fadd_rn(cur.acc[kA], dstar), wstar, lnA, bnA, nullptr);
                    }
                    const float mxA = block_max(sA, sc, G);
                    tau0 = __fsub_rn(fmaxf(mxrb, mxA), p.theta);  // lower bound of fl(max - θ)
                }
                if (al) {
                    if (sbk > kNeg && sbk >= tau0) push_cand(sm, sc, make_key(sbk, flat_idx(tid, blank)), cur.lms[tid], cur.bts[tid]);
                    if (srk > kNeg && srk >= tau0) push_cand(sm, sc, make_key(srk, flat_idx(tid, lk)), cur.lms[tid], cur.bts[tid]);
                }
                if (sA > kNeg && sA >= tau0) {
                    push_cand(sm, sc, make_key(sA, flat_idx(kA, wstar)), lnA, bnA);
                    prefetch_state(p, lnA, bnA);
                }

                // ------------------------------------------------ phase 3 (decision): token filter
                // a non-rb candidate reaching tau0 needs D[w] >= tau0 - accmax - ubvmax (- margin)
                const long long cp3 = TCLK();
                tp2 = cp3;
                if (tid == 0) st[kCycP2] += (uint32_t)(cp3 - cp2);
                // running threshold: the K-th best exact candidate pushed so far (blank / repeat /
                // best-token candidates). A candidate below the K-th of any K candidates cannot
                // enter the flat TopK, so it need not be scored; on blank-dominated
                // frames this bound is far above fl(max - θ).
                float thr = tau0;
                // a frame whose best non-blank token cannot reach even tau0 <= thr needs no token
                // filter: the K-th key (below) only tightens the filter of frames that scan
                bool need_kth = true;
                if (!stage_a && nalive > 0 && mxrb > kNeg) {
                    const float mg0 = 1e-4f * (1.0f + fabsf(tau0) + fabsf(accmax) + fabsf(ubvmax));
                    need_kth = dstar >= __fsub_rn(__fsub_rn(__fsub_rn(tau0, accmax), ubvmax), mg0);
                }
                gsync(G);
                if (need_kth) {
                    const int nb = sc.nbuf;
                    if (nb >= K && nb <= 2 * G) thr = fmaxf(thr, score_of(kth_by_rank(sm.ckey, nb, K, sc, G)));
                }
                bool scan = false;
                float dthr = INFINITY;
                if (nalive > 0 && mxrb > kNeg) {
                    const float mg = 1e-4f * (1.0f + fabsf(thr) + fabsf(accmax) + fabsf(ubvmax));
                    dthr = __fsub_rn(__fsub_rn(__fsub_rn(thr, accmax), ubvmax), mg);
                    scan = stage_a ? true : (dstar >= dthr);
                }
                bool heavy = false;
                if (solo && scan) {
                    // the summary's list holds every token >= floor: usable when dthr >= floor
                    const int cnt = s_sum_cnt[slot];
                    if (cnt <= kListCap && dthr >= s_sum_floor[slot]) {
                        const int j = tid;
                        const int w = j < cnt ? s_list_tok[slot * kListCap + j] : -1;
                        const bool hit = w >= 0 && w != blank && !(stage_a && w == wstar) &&
                                         s_list_d[slot * kListCap + j] >= dthr;
                        const unsigned bal = __ballot_sync(0xffffffffu, hit);
                        if (hit) sm.toks[__popc(bal & ((1u << tid) - 1u))] = (uint16_t)w;
                        if (tid == 0) sc.m = __popc(bal);
                    } else {
                        heavy = true;
                    }
                }
                if (tid == 0) {
                    sc.thr = thr; sc.nalive = nalive; sc.ubvmax = ubvmax; sc.dthr = dthr;
                    sc.excl = stage_a ? wstar : -1; sc.scan = (!solo && scan) || heavy;
                    st[kStageA] += stage_a ? 1 : 0;
                }
            }
            tp3 = TCLK();
            if (solo) __syncthreads();  // B1: the helpers learn whether this frame needs them
            gsync(G);
            if (solo && sc.fast) {  // fast-path frame: updated in place, nothing more to do
                if (tid == 0) st[kCycFast] += (uint32_t)(TCLK() - c0);
                flip = false;
                continue;
            }
            const bool scan_all = sc.scan;
            const int nalive = sc.nalive;
            const float ubvmax = sc.ubvmax;
            if (scan_all && use_cmp && sc.dthr >= ((const float*)rc_t)[1]) {
                // the record lists every token with D >= floor <= dthr: filter its list
                const float dthr = sc.dthr;
                const int excl = sc.excl;
                const int rn = ((const int*)rc_t)[2];
                if (tid < 32) {
                    const int w = tid < rn ? (int)((const uint16_t*)(rc_t + 160))[tid] : -1;
                    const bool hit = w >= 0 && w != excl && ((const float*)(rc_t + 32))[tid] >= dthr;
                    const unsigned bal = __ballot_sync(0xffffffffu, hit);
                    if (hit) sm.toks[__popc(bal & ((1u << tid) - 1u))] = (uint16_t)w;
                    if (tid == 0) sc.m = __popc(bal);
                }
                __syncthreads();
            } else if (scan_all) {  // full filter scan of the row by the whole CTA
                const float dthr = sc.dthr;
                const int excl = sc.excl;
                for (int w0 = 0; w0 < Vp1; w0 += NT) {
                    const int w = w0 + tid;
                    const bool hit = w < Vp1 && w != blank && w != excl && row[w] >= dthr;
                    const unsigned bal = __ballot_sync(0xffffffffu, hit);
                    if (bal) {
                        int base = 0;
                        if ((tid & 31) == 0) base = atomicAdd(&sc.m, __popc(bal));
                        base = __shfl_sync(0xffffffffu, base, 0);
                        if (hit) sm.toks[base + __popc(bal & ((1u << (tid & 31)) - 1u))] = (uint16_t)w;
                    }
                }
                __syncthreads();
            }
            if (tid == 0) st[kCycP3] += (uint32_t)(TCLK() - c0);
            // group of phase 4: the whole CTA when it scanned, else the beam warp alone (solo)
            const int G4 = (solo && !scan_all) ? 32 : NT;
            if (solo && helper && !scan_all) continue;  // helpers go on to the next row + summary

            // ------------------------------------------------ phase 4: exact non-rb candidates
            const long long c1 = TCLK();
            const int m_frame = sc.m;
            {
                const int m = m_frame;
                if (tid == 0) { st[kFrames] += 1; st[kAlive] += nalive; st[kListed] += m; }
                // dense frame: many listed tokens. Score them from LM rows cached in shared memory
                // (the paper's full-vocabulary NGPU-LM query) instead of per-pair arc searches.
                const bool dense = lm_on && nrow > 0 && m >= dense_min && G4 == NT;
                if (dense) {
                    if (tid == 0) {
                        int nb = 0;
                        unsigned used = 0;  // lines referenced this frame (nrow <= 32)
                        for (int a2 = 0; a2 < nalive; ++a2) {
                            const int st_ = cur.lms[sm.alive_idx[a2]];
                            int line = -1;
                            for (int l = 0; l < nrow; ++l)
                                if (rowtag[l] == st_) { line = l; break; }
                            if (line < 0) {
                                for (int l = 0; l < nrow; ++l)
                                    if (!(used >> l & 1u)) { line = l; break; }
                                if (line >= 0) { rowtag[line] = st_; s_build[2 * nb] = line; s_build[2 * nb + 1] = st_; ++nb; }
                            }
                            if (line >= 0) used |= 1u << line;
                            s_line[a2] = line;
                        }
                        s_nbuild = nb;
                        st[kDenseFrames] += 1;
                        st[kRowsBuilt] += nb;
                    }
                    __syncthreads();
                    const long long cr = TCLK();
                    for (int i = 0; i < s_nbuild; ++i)
                        build_lm_row<NT>(p.lm, s_build[2 * i + 1], rowval + (size_t)s_build[2 * i] * VP, V);
                    __syncthreads();
                    if (tid == 0) st[kCycRows] += (uint32_t)(TCLK() - cr);
                } else if (m > 0 && nrow > 0) {
                    for (int a2 = tid; a2 < nalive; a2 += G4) s_line[a2] = -1;
                }
                if (m > 0) {
                    const long long c4s = TCLK();
                    // per live position: {acc, ub (β + α_LM·max P + α_BT·max Δ), |terms|, last}
                    for (int a2 = tid; a2 < nalive; a2 += G4) {
                        const int k = sm.alive_idx[a2];
                        float ub = p.beta, ua = fabsf(p.beta), ubnl = p.beta;
                        if (lm_on) { const float x = p.alpha_lm * __int_as_float(recof(cur, k)[4]); ub += x; ua += fabsf(x); }
                        if (bt_on) { const float x = p.alpha_bt * cur.btm[2 * k]; ub += x; ua += fabsf(x); ubnl += x; }
                        if (ub_inf) { ub = INFINITY; ubnl = INFINITY; }
                        s_pos[a2] = make_float4(cur.acc[k], ub, ua, __int_as_float(cur.last[k]));
                        s_ubnl[a2] = ubnl;
                    }
                    gsync(G4);
                    // suffix maxima of acc and |ub terms| over live positions (early exit below)
                    if (solo) {  // nalive <= 32: one warp-level suffix scan in warp 0
                        if (tid < 32) {
                            float am = tid < nalive ? s_pos[tid].x : kNeg, um = tid < nalive ? s_pos[tid].z : 0.0f;
#pragma unroll
                            for (int o = 1; o < 32; o <<= 1) {
                                const float a_ = __shfl_down_sync(0xffffffffu, am, o);
                                const float u_ = __shfl_down_sync(0xffffffffu, um, o);
                                if (tid + o < 32) { am = fmaxf(am, a_); um = fmaxf(um, u_); }
                            }
                            if (tid < nalive) s_suf[tid] = make_float2(am, um);
                        }
                    } else {
                        for (int a2 = tid; a2 < nalive; a2 += G4) {
                            float am = kNeg, um = 0.0f;
                            for (int q = a2; q < nalive; ++q) { am = fmaxf(am, s_pos[q].x); um = fmaxf(um, s_pos[q].z); }
                            s_suf[a2] = make_float2(am, um);
                        }
                    }
                    gsync(G4);
                    long long c4c = TCLK();
                    if (tid == 0) st[kCycP4Setup] += (uint32_t)(c4c - c4s);
                    // Token-major collection (lane = listed token, loop over the live slots with an
                    // early exit) of the (position, token) pairs that pass the bounds, then one
                    // parallel evaluation of the batch (one round of LM arc searches for up to
                    // kPairCap pairs). A lane whose pair list is full records where it stopped and
                    // resumes after the batch (no pair is collected twice).
                    // With few listed tokens, LT = 2..32 threads share a token, each taking every
                    // LT-th live slot from its own offset (shorter serial chains; the early exit
                    // stays valid per thread: the suffix maxima cover every later slot).
                    int lt_sh = 0;
                    while (lt_sh < 5 && (m << (lt_sh + 1)) <= G4) ++lt_sh;
                    const int LT = 1 << lt_sh;
                    for (int base = 0; base < (m << lt_sh); base += G4) {
                        const int jj = base + tid;
                        const int j = jj >> lt_sh;
                        const int w = jj < (m << lt_sh) ? (int)sm.toks[j] : -1;
                        const float dw = w >= 0 ? row[w] : 0.0f;
                        int a_from = w >= 0 ? (jj & (LT - 1)) : nalive;
                        for (;;) {
                            const float thr = sc.thr;
                            bool full = false;
                            for (int a2 = a_from; a2 < nalive; a2 += LT) {
                                {   // no later live slot can reach thr with this token: stop
                                    const float2 sf = s_suf[a2];
                                    const float reach = __fadd_rn(__fadd_rn(sf.x, dw), ubvmax);
                                    if (reach + 2e-4f * (1.0f + fabsf(sf.x) + fabsf(dw) + fabsf(ubvmax) + sf.y) < thr) break;
                                }
                                const float4 ps = s_pos[a2];
                                if (w == __float_as_int(ps.w)) continue;  // repeat: scored in phase 1
                                const float s0 = __fadd_rn(ps.x, dw);
                                if (__fadd_rn(s0, ps.y) + 1e-5f * (1.0f + fabsf(s0) + ps.z) < thr) continue;
                                const int line = nrow > 0 ? s_line[a2] : -1;
                                if (line >= 0) {  // exact LM value from the cached row tightens the bound
                                    const float x = p.alpha_lm * rowval[(size_t)line * VP + w];
                                    const float ub = __fadd_rn(s_ubnl[a2], x);
                                    if (__fadd_rn(s0, ub) + 1e-5f * (1.0f + fabsf(s0) + ps.z) < thr) continue;
                                }
                                const int q = atomicAdd(&sc.npair, 1);
                                if (q >= kPairCap) { full = true; a_from = a2; break; }
                                s_pairs[q] = ((uint32_t)a2 << 16) | (uint32_t)j;
                            }
                            if (!full) a_from = nalive;
                            const int any_full = G4 == 32 ? (int)__any_sync(0xffffffffu, full) : __syncthreads_or(full);
                            const long long c4e = TCLK();
                            if (tid == 0) st[kCycP4Collect] += (uint32_t)(c4e - c4c);
                            const int np = min(sc.npair, kPairCap);
                            if (sc.nbuf > cap - np) {
                                // buffer full: keep the top K, raise the threshold (threshold algorithm)
                                const int n = sc.nbuf;
                                const uint64_t kth = radix_kth(sm.ckey, n, K, sm, sc, G4);
                                gather_selected(n, kth, sm, sc, G4);
                                for (int i = tid; i < K; i += G4) { sm.ckey[i] = sm.skey[i]; sm.clm[i] = sm.slm[i]; sm.cbt[i] = sm.sbt[i]; }
                                if (tid == 0) { sc.nbuf = K; sc.thr = fmaxf(sc.thr, score_of(kth)); st[kCompactions] += 1; }
                                gsync(G4);
                            }
                            const float thr2 = sc.thr;
                            for (int q = tid; q < np; q += G4) {
                                const uint32_t pq = s_pairs[q];
                                const int a2 = (int)(pq >> 16), jq = (int)(pq & 0xffffu);
                                const int k = sm.alive_idx[a2];
                                const int wq = sm.toks[jq];
                                const int line = nrow > 0 ? s_line[a2] : -1;
                                const float s0 = __fadd_rn(s_pos[a2].x, row[wq]);
                                int ln, bn;
                                const float s = eval(cur, k, s0, wq, ln, bn, line >= 0 ? rowval + (size_t)line * VP : nullptr);
                                st[line >= 0 ? kEvalDense : kEvalSparse] += 1;
                                if (s > kNeg && s >= thr2) {
                                    push_cand(sm, sc, make_key(s, flat_idx(k, wq)), ln, bn);
                                    prefetch_state(p, ln, bn);
                                }
                            }
                            gsync(G4);
                            c4c = TCLK();
                            if (tid == 0) { sc.npair = 0; st[kCycP4Eval] += (uint32_t)(c4c - c4e); }
                            gsync(G4);
                            if (!any_full) break;
                        }
                    }
                }
            }
            if (solo && helper) continue;  // heavy frame done for the helpers

            // ------------------------------------------------ phase 5: flat TopK + θ-prune
            const long long c2 = TCLK();
            const int n = sc.nbuf;
            const uint64_t* kk;
            const int* kl;
            const int* kb;
            int nsel;
            if (n > G) {
                const uint64_t kth = radix_kth(sm.ckey, n, K, sm, sc, G);
                gather_selected(n, kth, sm, sc, G);
                kk = sm.skey; kl = sm.slm; kb = sm.sbt; nsel = K;
            } else {
                kk = sm.ckey; kl = sm.clm; kb = sm.cbt; nsel = n;
            }
            uint64_t myk = 0;
            int rank = 0, myl = 0, myb = 0;
            if (tid < nsel) {
                myk = kk[tid]; myl = kl[tid]; myb = kb[tid];
                for (int j = 0; j < nsel; ++j) rank += kk[j] > myk ? 1 : 0;
            }
            gsync(G);
            if (tid < nsel && rank < K) { sm.skey[rank] = myk; sm.slm[rank] = myl; sm.sbt[rank] = myb; }
            gsync(G);
            const int nkeep = nsel < K ? nsel : K;
            const float mx = nkeep > 0 ? score_of(sm.skey[0]) : kNeg;  // max_score
            const float tau = __fsub_rn(mx, p.theta);

            const long long c3 = TCLK();
            // ------------------------------------------------ phase 6: beams.update into nxt
            const int64_t bpo = bp_base + (int64_t)(t * K);
            bool live = false, emit = false;
            float my_acc = kNeg;  // this lane's new slot (phase 7 reads it from registers)
            int my_last = blank;
            uint8_t my_anc = 0;
            uint64_t my_hash = 0ull;
            int par = 0;
            int4 rec_ld[kRec / 4];
            float2 bt_ld = make_float2(0.0f, 0.0f);
            if (tid < K) {
                const int i = tid;
                if (i < nkeep) {
                    const uint64_t key = sm.skey[i];
                    const float s = score_of(key);
                    if (s >= tau) {
                        live = true;
                        const uint32_t f = flat_of(key);
                        par = (int)(f >> 16);
                        const int w = (int)(f & 0xffffu);
                        emit = w != blank && w != cur.last[par];
                        int ln = sm.slm[i];
                        const int bn = sm.sbt[i];
                        if (emit && ln < 0) {  // scored from a cached row: resolve the next LM state now
                            lm_query<LMV>(p.lm, recof(cur, par), w, ln);
                            st[kDeferredNext] += 1;
                        }
                        if (emit) {  // new LM / BT states: fetch their records (latency overlaps phase 7)
                            if (lm_on)
#pragma unroll
                                for (int q = 0; q < kRec / 4; ++q)
                                    if (4 * q < RWS) rec_ld[q] = __ldg(&p.lm.rec[(size_t)ln * (p.lm.RW / 4) + q]);
                            if (bt_on) bt_ld = make_float2(__ldg(&p.bt.maxd[bn]), __ldg(&p.bt.U[bn]));
                        }
                        my_acc = s;
                        my_last = w;
                        my_hash = emit ? hash_extend(cur.hash[par], w) : cur.hash[par];
                        nxt.acc[i] = my_acc;
                        nxt.last[i] = my_last;
                        nxt.hash[i] = my_hash;
                        nxt.lms[i] = ln;  // rb candidates carry the parent's states
                        nxt.bts[i] = bn;
                        my_anc = (t % kChunk == 0) ? (uint8_t)par : cur.anc[par];
                        nxt.anc[i] = my_anc;
                        p.bp_parent[bpo + i] = (uint8_t)par;
                        p.bp_label[bpo + i] = (uint16_t)w;
                    }
                }
                if (!live) {
                    nxt.acc[i] = kNeg;
                    nxt.last[i] = blank;
                    nxt.hash[i] = 0ull;
                    nxt.lms[i] = 0; nxt.bts[i] = 0; nxt.anc[i] = 0;
                    // dead slots need no backpointer: the backtrace only follows live ancestors
                }
            }
            // the live slots are a prefix of the (score desc) selection; count them with the barrier
            int nlive_all = 0;
            if (G == 32) gsync(G); else nlive_all = __syncthreads_count(live ? 1 : 0);
            const long long c6 = TCLK();
            // ------------------------------------------------ phase 7: RecombineHypotheses
            unsigned grp = 0;
            // all live slots in warp 0: K <= 32, or (K > 32) at most 32 of them live this frame (the
            // common case at c5), where match.any replaces the shared hash table
            const bool small_beam = K <= 32 || (G != 32 && nlive_all <= 32);
            if (small_beam && tid < 32) {
                // one warp holds the beam: group lanes by (hash, last) with match.any
                const bool lv = tid < K && my_acc > kNeg;
                const uint64_t hk = lv ? my_hash : (0xfedcba9800000000ull | (uint64_t)tid);
                const int lkey = lv ? my_last : -1 - tid;
                const unsigned livemask = __ballot_sync(0xffffffffu, lv);
                // only the live lanes take part: match.any costs ~14 cycles per distinct value
                // (444 cycles for 32 distinct 64-bit keys, tools/micro/lat.cu), and dead lanes
                // would each add one
                if (lv) grp = __match_any_sync(livemask, hk) & __match_any_sync(livemask, lkey);
            }
            const long long t7a = TCLK();
            int tent = -1;  // K > 32: this slot's entry in the (hash, last) table
            if (NT > 32 && !small_beam) {
                // groups have <= 3 members (reading R14): a shared hash table keyed on (hash, last)
                // with member lists replaces the O(K) scan per slot
                for (int e = tid; e < kTab; e += NT) { s_tocc[e] = 0; s_tcnt[e] = 0; }
                __syncthreads();
                if (tid < K && nxt.acc[tid] > kNeg) {
                    // bucket from a fold of (hash, last); an entry belongs to the exact pair of its first
                    // member (compared in full, so two groups whose folds collide never merge)
                    const uint64_t h = nxt.hash[tid];
                    const int l = nxt.last[tid];
                    const uint64_t k2 = h ^ ((uint64_t)(l + 1) * 0x9E3779B97F4A7C15ull);
                    int e = (int)((k2 >> 20) & (uint64_t)(kTab - 1));
                    for (;;) {
                        const int old = atomicCAS(&s_tocc[e], 0, tid + 1);
                        if (old == 0) break;
                        if (nxt.hash[old - 1] == h && nxt.last[old - 1] == l) break;
                        e = (e + 1) & (kTab - 1);
                    }
                    const int q = atomicAdd(&s_tcnt[e], 1);
                    if (q < kTabMem) s_tmem[e * kTabMem + q] = tid;
                    tent = e;
                }
                __syncthreads();
            }
            long long t7b = t7a, t7c = t7a;
            if (tid < K) {
                const int i = tid;
                float s = my_acc;
                if (small_beam && s > kNeg) {
                    if (grp & ((1u << i) - 1u)) {
                        s = kNeg;  // a better (lower) slot of the group survives
                    } else {
                        unsigned others = grp & ~((2u << i) - 1u);  // higher slots, ascending order
                        if (others && merge_mode == 0) {
                            float sum = 0.0f;
                            while (others) {
                                const int j = __ffs(others) - 1;
                                others &= others - 1u;
                                sum = __fadd_rn(sum, (float)exp((double)__fsub_rn(nxt.acc[j], s)));
                            }
                            s = __fadd_rn(s, (float)log1p((double)sum));
                        }
                    }
                } else if (s > kNeg && s_tcnt[tent] <= kTabMem) {
                    const int cnt = s_tcnt[tent];
                    if (cnt > 1) {
                        int mem[kTabMem];
#pragma unroll
                        for (int q = 0; q < kTabMem; ++q) mem[q] = q < cnt ? s_tmem[tent * kTabMem + q] : 0x7fffffff;
#pragma unroll
                        for (int q = 1; q < kTabMem; ++q)  // ascending slot order
#pragma unroll
                            for (int r = q; r > 0; --r)
                                if (mem[r] < mem[r - 1]) { const int x = mem[r]; mem[r] = mem[r - 1]; mem[r - 1] = x; }
                        if (mem[0] != i) {
                            s = kNeg;
                        } else if (merge_mode == 0) {
                            float sum = 0.0f;
#pragma unroll
                            for (int q = 1; q < kTabMem; ++q)
                                if (q < cnt) sum = __fadd_rn(sum, (float)exp((double)__fsub_rn(nxt.acc[mem[q]], s)));
                            s = __fadd_rn(s, (float)log1p((double)sum));
                        }
                    }
                } else if (s > kNeg) {  // oversized group (not expected): plain scan
                    const uint64_t h = nxt.hash[i];
                    const int l = nxt.last[i];
                    bool dead = false;
                    for (int j = 0; j < i; ++j)
                        if (nxt.acc[j] > kNeg && nxt.hash[j] == h && nxt.last[j] == l) { dead = true; break; }
                    if (dead) {
                        s = kNeg;
                    } else {
                        // slots are in (score desc, flat asc) order, so group order == slot order
                        float sum = 0.0f;
                        bool any = false;
                        for (int j = i + 1; j < K; ++j) {
                            const float sj = nxt.acc[j];
                            if (sj > kNeg && nxt.hash[j] == h && nxt.last[j] == l) {
                                any = true;
                                if (merge_mode == 0) sum = __fadd_rn(sum, (float)exp((double)__fsub_rn(sj, s)));
                            }
                        }
                        if (any && merge_mode == 0) s = __fadd_rn(s, (float)log1p((double)sum));
                    }
                }
                t7b = TCLK();
                if ((t % kChunk) == kChunk - 1 || t == L - 1)
                    p.chunk_anc[((int64_t)b * p.nch + t / kChunk) * K + i] = my_anc;
                // cached records of the new slot states
                if (live) {
                    if (emit) {
                        if (lm_on)
#pragma unroll
                            for (int q = 0; q < kRec / 4; ++q)
                                if (4 * q < RWS) ((int4*)(nxt.rec + i * RWS))[q] = rec_ld[q];
                        nxt.btm[2 * i] = bt_ld.x;
                        nxt.btm[2 * i + 1] = bt_ld.y;
                    } else {
                        if (lm_on)
                            for (int q = 0; q < RWS / 4; ++q)
                                ((int4*)(nxt.rec + i * RWS))[q] = ((const int4*)(cur.rec + par * RWS))[q];
                        nxt.btm[2 * i] = cur.btm[2 * par];
                        nxt.btm[2 * i + 1] = cur.btm[2 * par + 1];
                    }
                }
                sm.skey[i] = (uint64_t)__float_as_uint(s);  // stash merged score
                t7c = TCLK();
            }
            gsync(G);
            if (tid < K) nxt.acc[tid] = __uint_as_float((uint32_t)sm.skey[tid]);
            if (tid == 0) {
                const long long c4 = TCLK();
                if (m_frame == 0) {  // frames without listed tokens: phase split
                    st[kLightFrames] += 1;
                    st[kLP1] += (uint32_t)(tp1 - c0); st[kLP2] += (uint32_t)(tp2 - tp1);
                    st[kLP3] += (uint32_t)(tp3 - tp2); st[kLB1] += (uint32_t)(c1 - tp3);
                    st[kLP5] += (uint32_t)(c3 - c2); st[kLP6] += (uint32_t)(c6 - c3);
                    st[kLP7] += (uint32_t)(c4 - c6);
                    st[kLP7a] += (uint32_t)(t7a - c6); st[kLP7b] += (uint32_t)(t7b - t7a);
                    st[kLP7c] += (uint32_t)(t7c - t7b); st[kLP7d] += (uint32_t)(c4 - t7c);
                }
                st[kCycP13] += (uint32_t)(c1 - c0); st[kCycP4] += (uint32_t)(c2 - c1);
                st[kCycP5] += (uint32_t)(c3 - c2); st[kCycP67] += (uint32_t)(c4 - c3);
                if (m_frame > 0) { st[kHeavyFrames] += 1; st[kCycHeavy] += (uint32_t)(c4 - c0); }
            }
            gsync(G);
        }
        cp_wait<0>();
        __syncthreads();  // join the beam warp and the helpers (solo mode)
        const Bank cur = bank(flip ? cbank ^ 1 : cbank);

        // ------------------------------------------------------------ EOS + final merge (R15)
        float fs = kNeg;
        if (tid < K) {
            fs = cur.acc[tid];
            if (fs > kNeg) {
                if (lm_on) fs = __fmaf_rn(p.alpha_lm, __int_as_float(recof(cur, tid)[5]), fs);
                if (bt_on && p.retract) fs = __fmaf_rn(-p.alpha_bt, cur.btm[2 * tid + 1], fs);
            }
            sm.skey[tid] = (uint64_t)__float_as_uint(fs);
        }
        __syncthreads();
        uint64_t mykey = 0;  // final-merge survivor key: (merged score, ~slot); 0 = not a survivor
        if (tid < K && fs > kNeg) {
            const int i = tid;
            float s = fs;
            const uint64_t h = cur.hash[i];
            auto sc_of = [&](int j) { return __uint_as_float((uint32_t)sm.skey[j]); };
            bool dead = false;
            for (int j = 0; j < K; ++j) {
                const float sj = sc_of(j);
                if (j != i && sj > kNeg && cur.hash[j] == h && (sj > s || (sj == s && j < i))) { dead = true; break; }
            }
            if (!dead) {
                float sum = 0.0f;
                bool any = false;
                float prev_s = INFINITY;
                int prev_j = -1;
                for (;;) {  // other members in (score desc, slot asc) order
                    int bj = -1;
                    float bs = kNeg;
                    for (int j = 0; j < K; ++j) {
                        const float sj = sc_of(j);
                        if (j == i || !(sj > kNeg) || cur.hash[j] != h) continue;
                        if (!(sj < prev_s || (sj == prev_s && j > prev_j))) continue;
                        if (bj < 0 || sj > bs || (sj == bs && j < bj)) { bj = j; bs = sj; }
                    }
                    if (bj < 0) break;
                    any = true;
                    if (merge_mode == 0) sum = __fadd_rn(sum, (float)exp((double)__fsub_rn(bs, s)));
                    prev_s = bs;
                    prev_j = bj;
                }
                if (any && merge_mode == 0) s = __fadd_rn(s, (float)log1p((double)sum));
                mykey = ((uint64_t)ord_of(s) << 32) | (uint64_t)(0xffffffffu - (uint32_t)i);
            }
        }
        // rank the survivors by (score desc, slot asc): rank r -> slot, merged score
        const int NB = p.nbest > 1 ? p.nbest : 1;
        __syncthreads();
        if (tid < K) sm.ckey[tid] = mykey;
        int nsurv;
        block_exscan(mykey ? 1 : 0, &nsurv, sc, NT);
        __syncthreads();
        if (mykey) {
            int rank = 0;
            for (int j = 0; j < K; ++j) rank += sm.ckey[j] > mykey ? 1 : 0;
            if (rank < NB) { sm.alive_idx[rank] = tid; sm.slm[rank] = __float_as_int(score_of(mykey)); }
        }
        __syncthreads();

        for (int r = 0; r < NB; ++r) {  // the 1-best (NB = 1) or the n best merged hypotheses
            const bool has_best = r < nsurv;
            const int best = has_best ? sm.alive_idx[r] : -1;
            const float best_score = has_best ? __int_as_float(sm.slm[r]) : kNeg;
            const int64_t orow = (int64_t)b * NB + r;  // output row
            // ------------------------------------------------------------ backtrace ("reconstruction on demand")
            int32_t* align = (p.out_align && r == 0 ? p.out_align : p.align_ws) + (int64_t)b * p.T;
            const int nchk = (L + kChunk - 1) / kChunk;
            if (has_best && L > 0) {
                if (tid == 0) {
                    int s = best;
                    sm.endslot[nchk - 1] = s;
                    for (int c = nchk - 1; c >= 1; --c) {
                        s = p.chunk_anc[((int64_t)b * p.nch + c) * K + s];
                        sm.endslot[c - 1] = s;
                    }
                }
                __syncthreads();
                for (int c = tid; c < nchk; c += NT) {
                    int s = sm.endslot[c];
                    const int t_hi = min(c * kChunk + kChunk - 1, L - 1);
                    for (int t = t_hi; t >= c * kChunk; --t) {
                        const int64_t o = ((int64_t)b * p.T + t) * K + s;
                        align[t] = p.bp_label[o];
                        s = p.bp_parent[o];
                    }
                }
            }
            __syncthreads();
            // collapse to tokens + timestamps (R20): emitted at t iff a_t != blank and a_t != a_{t-1}
            const int per = (L + NT - 1) / NT;
            const int t0 = min(L, tid * per), t1 = min(L, t0 + per);
            int cnt = 0;
            if (has_best)
                for (int t = t0; t < t1; ++t) {
                    const int at = align[t], ap = t ? align[t - 1] : blank;
                    cnt += (at != blank && at != ap) ? 1 : 0;
                }
            int ntok;
            int off = block_exscan(cnt, &ntok, sc, NT);
            int32_t* otok = p.out_tokens + orow * p.T;
            int32_t* ots = p.out_ts ? p.out_ts + orow * p.T : nullptr;
            if (has_best)
                for (int t = t0; t < t1; ++t) {
                    const int at = align[t], ap = t ? align[t - 1] : blank;
                    if (at != blank && at != ap) {
                        otok[off] = at;
                        if (ots) ots[off] = t;
                        ++off;
                    }
                }
            if (!has_best) ntok = 0;
            for (int i = ntok + tid; i < p.T; i += NT) { otok[i] = -1; if (ots) ots[i] = -1; }
            if (p.out_align && r == 0)
                for (int i = (has_best ? L : 0) + tid; i < p.T; i += NT) p.out_align[(int64_t)b * p.T + i] = -1;
            if (tid == 0) {
                p.out_num[orow] = ntok;
                p.out_scores[orow] = best_score;
            }
            __syncthreads();
        }
    }
#pragma unroll
    for (int i = 0; i < kNumStats; ++i)
        if (st[i]) atomicAdd(&p.stats[i], (unsigned long long)st[i]);
}

// L2 warm-up of the fusion tables the frame loop looks up at random (LM level-1 dense rows and
// sorted arcs, the boost transition table): one streaming pass (prefetch.global.L2::evict_last
// per 128-B line) at HBM rate before the frame loop, so the dependent lookups of the recurrence
// hit L2 instead of paying HBM latency after every cold start (the bench flushes L2 per step).
__global__ void l2_warm_kernel(const char* a, int64_t na, const char* b, int64_t nb, const char* c, int64_t nc,
                               const char* d, int64_t nd) {
    const int64_t la = (na + 127) >> 7, lb = (nb + 127) >> 7, lc = (nc + 127) >> 7, ld = (nd + 127) >> 7;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < la + lb + lc + ld;
         i += (int64_t)gridDim.x * blockDim.x) {
        const char* q = i < la ? a + (i << 7)
                        : i < la + lb ? b + ((i - la) << 7)
                        : i < la + lb + lc ? c + ((i - la - lb) << 7) : d + ((i - la - lb - lc) << 7);
        asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(q));
    }
}

// Clamp lengths, flag anomalies, and order utterances longest-first (LPT) for the work queue.
__global__ void order_kernel(const int32_t* __restrict__ lengths, int B, int T, int32_t* order, int32_t* len_c,
                             uint32_t* flags, int sort) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    int L = lengths[b];
    uint32_t fl = 0;
    if (L > T) { L = T; fl |= FLEXCTC_FLAG_LENGTH_CLAMPED_HIGH; }
    if (L < 0) { L = 0; fl |= FLEXCTC_FLAG_LENGTH_CLAMPED_LOW; }
    len_c[b] = L;
    if (fl) atomicOr(flags, fl);
    if (!sort) { order[b] = b; return; }
    int rank = 0;
    for (int j = 0; j < B; ++j) {
        const int Lj = min(max(lengths[j], 0), T);
        rank += (Lj > L || (Lj == L && j < b)) ? 1 : 0;
    }
    order[rank] = b;
}

size_t smem_bytes(int K, int Vp1, int R, int cap, int nch, int RWS, bool lgt) {
    const int VP = (Vp1 + 3) & ~3;
    auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
    size_t s = al(sizeof(float) * (size_t)R * (VP + (lgt ? 20 : 4))) + (size_t)R * kCmpBytes;
    s += al(8 * K) + al(8 * K) + al(16 * K) + al(8 * K) + al(8 * K) + al(2 * K) + al(8 * (size_t)K * RWS) + al(16 * K);
    s += al(8 * (size_t)cap) + 2 * al(4 * (size_t)cap);
    s += al(8 * K) + 2 * al(4 * K);
    s += al(2 * (size_t)Vp1) + al(4 * K) + al(4 * 256) + al(4 * (size_t)nch);
    return s;
}

struct Plan {
    size_t sm = 0;
    int nrow = 0, occ = 0, R = 4, cap = 0, dense_min = kDenseMinTokens;
};

// Shared-memory layout, row-cache lines and occupancy of the NT-thread kernel for this decode.
template <int NT, int LMV>
int plan_nt(const DecodeParams& p, Plan& pl, std::string& err) {
    const int VP = (p.Vp1 + 3) & ~3;
    pl.R = VP <= 2048 ? 4 : 2;
    pl.cap = 4 * NT;  // >= 3K phase-1/2 pushes, and >= kPairCap + K for phase 4
    const int RWS = p.use_lm ? ((p.lm.RW + 3) & ~3) : 4;
    pl.sm = smem_bytes(p.K, p.Vp1, pl.R, pl.cap, p.nch, RWS, p.logits != nullptr) + (p.use_bt ? 8 * (size_t)(p.Vp1 - 1) + 16 : 0);
    if (pl.sm > 200 * 1024) { err = "shared memory requirement too large (V+1 or T)"; return 2; }
    auto kern = ctc_beam_kernel<NT, LMV, false>;
    cudaFuncAttributes fattr{};
    cudaFuncGetAttributes(&fattr, kern);
    // The dense-frame LM row cache is off by default: with 8 warps per utterance the batched
    // sparse evaluation is faster on c3-c5 (measured); FLEXCTC_DENSE_MIN=<tokens> enables it, with
    // as many lines as fit the shared memory left at the register-limited occupancy (<= min(K, 32)).
    const char* e_dm = getenv("FLEXCTC_DENSE_MIN");
    if (e_dm) pl.dense_min = std::max(1, atoi(e_dm));
    pl.nrow = 0;
    if (p.use_lm && e_dm) {
        const size_t line = 4 * (size_t)VP + 4;
        const int occ_regs = std::max(1, 65536 / std::max(1, fattr.numRegs * NT));
        const size_t per_cta = std::min<size_t>(200 * 1024, (size_t)(224 * 1024) / (size_t)occ_regs);
        const size_t budget = per_cta - std::min<size_t>(fattr.sharedSizeBytes, per_cta / 2);
        if (pl.sm + 16 < budget) pl.nrow = (int)std::min<size_t>((budget - pl.sm - 16) / line, (size_t)std::min(p.K, 32));
        pl.sm += pl.nrow ? 4 * (size_t)pl.nrow * VP + ((4 * (size_t)pl.nrow + 15) & ~size_t(15)) : 0;
    }
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.sm);
    if constexpr (NT >= 128)
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(ctc_beam_kernel<NT, LMV, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)pl.sm);
    if constexpr (NT == 64 && LMV == 2)
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(ctc_beam_kernel<NT, LMV, false, 1025, 16, 16, 7>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.sm);
    if constexpr (NT == 256 && LMV == 2) {
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(ctc_beam_kernel<NT, LMV, true, 1025>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)pl.sm);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(ctc_beam_kernel<NT, LMV, false, 1025>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)pl.sm);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(ctc_beam_kernel<NT, LMV, true, 1025, 16, 16>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.sm);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(ctc_beam_kernel<NT, LMV, true, 1025, 16, 16, 3>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.sm);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(ctc_beam_kernel<NT, LMV, true, 1025, 16, 16, 7>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.sm);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(ctc_beam_kernel<NT, LMV, true, 1025, 16, 16, 15>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.sm);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(ctc_beam_kernel<NT, LMV, true, 1025, 16, 16, 31>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.sm);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(ctc_beam_kernel<NT, LMV, true, 1025, 16, 16, 5>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.sm);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(ctc_beam_kernel<NT, LMV, false, 1025, 0, 16, 7>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.sm);
    }
    if (e != cudaSuccess) { err = cudaGetErrorString(e); return 1; }
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pl.occ, kern, NT, pl.sm);
    if (e != cudaSuccess || pl.occ < 1) { err = "occupancy query failed"; return 1; }
    return 0;
}

template <int NT, int LMV>
int run_nt(const DecodeParams& p, const Plan& pl, int nsm, cudaStream_t st, void* ev0, void* ev1, std::string& err) {
    const int grid = std::min(p.B, nsm * pl.occ);
    if (p.logits && !(NT == 256 && LMV == 2 && p.Vp1 == 1025)) {
        err = "bf16 logits: no kernel variant for this configuration";
        return 2;
    }
    DecodeParams q = p;
    const char* e_solo = getenv("FLEXCTC_SOLO");  // "0": every phase uses the whole CTA (test switch)
    q.solo_off = (e_solo && e_solo[0] == '0') ? 1 : 0;
    const char* e_fast = getenv("FLEXCTC_FAST");  // "0": no settled-beam fast path (A/B switch)
    q.fast_off = (e_fast && e_fast[0] == '0') ? 1 : 0;
    const bool solo = p.K <= 32 && NT >= 128 && pl.R == 4 && !q.solo_off;  // 4 = the kernel's kRing
    if (ev0 && ev1) cudaEventRecord((cudaEvent_t)ev0, st);
    if constexpr (NT >= 128) {
        bool done = false;
        if constexpr (NT == 256 && LMV == 2)  // the paper's vocabulary (1024 BPE tokens + blank)
            if (p.Vp1 == 1025) {
                const bool plain = pl.nrow == 0 && p.merge_mode == 0 && !p.retract && p.alpha_lm >= 0.0f &&
                                   p.alpha_bt >= 0.0f;
                if (p.logits) {  // bf16 logits read by the kernel itself (cta_logits_direct)
                    if (solo && p.use_cmp && p.K == 16 && p.use_lm && p.lm.RW == 16 && p.use_bt && plain)
                        ctc_beam_kernel<NT, LMV, true, 1025, 16, 16, 31><<<grid, NT, pl.sm, st>>>(q, pl.R, pl.cap, pl.nrow, pl.dense_min);
                    else { err = "bf16 logits: no kernel variant for this configuration"; return 2; }
                } else if (solo && !p.use_cmp && p.K == 16 && p.use_lm && p.lm.RW == 16 && p.use_bt && plain)  // the north-star decode
                    ctc_beam_kernel<NT, LMV, true, 1025, 16, 16, 7><<<grid, NT, pl.sm, st>>>(q, pl.R, pl.cap, pl.nrow, pl.dense_min);
                else if (solo && p.use_cmp && p.K == 16 && p.use_lm && p.lm.RW == 16 && p.use_bt && plain)  // ... reading records
                    ctc_beam_kernel<NT, LMV, true, 1025, 16, 16, 15><<<grid, NT, pl.sm, st>>>(q, pl.R, pl.cap, pl.nrow, pl.dense_min);
                else if (solo && !p.use_cmp && p.K == 16 && p.use_lm && p.lm.RW == 16 && !p.use_bt && plain)  // LM only (c3)
                    ctc_beam_kernel<NT, LMV, true, 1025, 16, 16, 5><<<grid, NT, pl.sm, st>>>(q, pl.R, pl.cap, pl.nrow, pl.dense_min);
                else if (solo && !p.use_cmp && p.K == 16 && p.use_lm && p.lm.RW == 16 && p.use_bt)  // beam 16, 4-gram LM, boosting
                    ctc_beam_kernel<NT, LMV, true, 1025, 16, 16, 3><<<grid, NT, pl.sm, st>>>(q, pl.R, pl.cap, pl.nrow, pl.dense_min);
                else if (solo && !p.use_cmp && p.K == 16 && p.use_lm && p.lm.RW == 16)  // beam 16 + 4-gram LM
                    ctc_beam_kernel<NT, LMV, true, 1025, 16, 16><<<grid, NT, pl.sm, st>>>(q, pl.R, pl.cap, pl.nrow, pl.dense_min);
                else if (solo) ctc_beam_kernel<NT, LMV, true, 1025><<<grid, NT, pl.sm, st>>>(q, pl.R, pl.cap, pl.nrow, pl.dense_min);
                else if (!p.use_cmp && p.use_lm && p.lm.RW == 16 && p.use_bt && plain)  // K > 32, 4-gram LM, boosting (c5)
                    ctc_beam_kernel<NT, LMV, false, 1025, 0, 16, 7><<<grid, NT, pl.sm, st>>>(q, pl.R, pl.cap, pl.nrow, pl.dense_min);
                else ctc_beam_kernel<NT, LMV, false, 1025><<<grid, NT, pl.sm, st>>>(q, pl.R, pl.cap, pl.nrow, pl.dense_min);
                done = true;
            }
        if (done) {
        } else if (solo) ctc_beam_kernel<NT, LMV, true><<<grid, NT, pl.sm, st>>>(q, pl.R, pl.cap, pl.nrow, pl.dense_min);
        else ctc_beam_kernel<NT, LMV, false><<<grid, NT, pl.sm, st>>>(q, pl.R, pl.cap, pl.nrow, pl.dense_min);
    } else {
        (void)solo;
        bool done = false;
        if constexpr (NT == 64 && LMV == 2)  // throughput mode (B > 4 x #SMs) on the north-star decode
            if (p.Vp1 == 1025 && !p.use_cmp && p.K == 16 && p.use_lm && p.lm.RW == 16 && p.use_bt && pl.nrow == 0 &&
                p.merge_mode == 0 && !p.retract && p.alpha_lm >= 0.0f && p.alpha_bt >= 0.0f) {
                ctc_beam_kernel<NT, LMV, false, 1025, 16, 16, 7><<<grid, NT, pl.sm, st>>>(q, pl.R, pl.cap, pl.nrow, pl.dense_min);
                done = true;
            }
        if (!done) ctc_beam_kernel<NT, LMV, false><<<grid, NT, pl.sm, st>>>(q, pl.R, pl.cap, pl.nrow, pl.dense_min);
    }
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess && ev0 && ev1) cudaEventRecord((cudaEvent_t)ev1, st);
    if (e != cudaSuccess) { err = cudaGetErrorString(e); return 1; }
    set_kernel_name(p.logits ? "ctc_beam_kernel+records+bf16" : p.use_cmp ? "ctc_beam_kernel+records" : "ctc_beam_kernel");
    return 0;
}

template <int LMV>
int plan_any(int nt, const DecodeParams& p, Plan& pl, std::string& err) {
    switch (nt) {
        case 32: return plan_nt<32, LMV>(p, pl, err);
        case 64: return plan_nt<64, LMV>(p, pl, err);
        case 128: return plan_nt<128, LMV>(p, pl, err);
        default: return plan_nt<256, LMV>(p, pl, err);
    }
}
template <int LMV>
int run_any(int nt, const DecodeParams& p, const Plan& pl, int nsm, cudaStream_t st, void* ev0, void* ev1, std::string& err) {
    switch (nt) {
        case 32: return run_nt<32, LMV>(p, pl, nsm, st, ev0, ev1, err);
        case 64: return run_nt<64, LMV>(p, pl, nsm, st, ev0, ev1, err);
        case 128: return run_nt<128, LMV>(p, pl, nsm, st, ev0, ev1, err);
        default: return run_nt<256, LMV>(p, pl, nsm, st, ev0, ev1, err);
    }
}

// Relative per-utterance latency of the NT-thread kernel (measured on c4 / c5, round 1): more
// warps shorten each frame step; fewer warps fit more utterances per SM.
// K <= 32, c4-shaped, one wave each (round 2, profiles/r2_policy.jsonl): NT = 256 1.59 ms at
// B = 148; NT = 128 2.59 ms at B = 256; NT = 64 2.68 / 2.74 / 2.85 ms at B = 256 / 384 / 512.
double latency_factor(int nt, int K) {
    if (K <= 32) return nt == 32 ? 2.2 : nt == 64 ? 1.8 : nt == 128 ? 1.65 : 1.0;
    return nt == 64 ? 1.6 : nt == 128 ? 1.3 : 1.0;
}

template <int LMV>
int launch_lmv(const DecodeParams& p, cudaStream_t st, void* ev0, void* ev1, std::string& err) {
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int need = p.K <= 32 ? 32 : p.K <= 64 ? 64 : p.K <= 128 ? 128 : 256;
    int forced = 0;
    if (const char* e_nt = getenv("FLEXCTC_NT")) {  // tuning override (never below the beam)
        const int want = atoi(e_nt);
        if ((want == 32 || want == 64 || want == 128 || want == 256) && want >= need) forced = want;
    }
    // Threads per utterance: 8 warps (shortest frame step) unless the batch is much larger than
    // the GPU (B > 4 x #SMs), where (waves of utterances) x (per-utterance latency) is minimised.
    // Below that, the longest utterance dominates (LPT queue), so latency wins (c5: B = 512).
    int best_nt = 256;
    Plan best;
    double best_cost = 1e300;
    const bool throughput = p.B > 4 * nsm;
    for (int nt = need; nt <= 256; nt *= 2) {
        if (forced && nt != forced) continue;
        // K > 32: latency mode (one utterance per CTA of 256 threads) unless B > 4 x #SMs
        if (!forced && !throughput && nt != 256 && p.K > 32) continue;
        Plan pl;
        const int rc = plan_any<LMV>(nt, p, pl, err);
        if (rc) { if (forced || nt == 256) return rc; continue; }
        const double waves = std::ceil((double)p.B / ((double)nsm * pl.occ));
        const double cost = waves * latency_factor(nt, p.K);
        if (cost < best_cost - 1e-9 || (cost < best_cost + 1e-9 && nt > best_nt)) { best_cost = cost; best_nt = nt; best = pl; }
    }
    if (best_cost >= 1e299) return 2;
    return run_any<LMV>(best_nt, p, best, nsm, st, ev0, ev1, err);
}

}  // namespace

// The warp-per-utterance path (compaction pass + warp_beam_kernel) serves 2 <= K <= 32 with
// 1-best output and device-resident input; FLEXCTC_WARP=0 keeps the persistent CTA kernel (test
// switch: both paths are parity-tested).
bool use_warp_path(const DecodeParams& p) {
    if (p.K < 2 || p.K > 32 || p.nbest > 1 || p.ready || !p.cmp || !p.rowoff || p.fuse_rep) return false;
    const char* e = getenv("FLEXCTC_WARP");
    if (e && e[0] == '0') return false;
    if (!(e && e[0] == '1')) {
        // Up to 4 x #SMs utterances the persistent CTA kernel (2-8 warps per utterance, up to 592
        // in flight) has the shorter frame step; beyond, the warp kernel's one warp per utterance
        // packs more utterances per SM (tools/policy_sweep.py, profiles/r2/policy_*.jsonl)
        int dev = 0, nsm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        if (p.B <= 4 * nsm) return false;
    }
    const size_t per = warp_beam_smem_per_warp(p.Vp1, p.logits != nullptr, p.nch);
    return per + (p.use_bt ? 8 * (size_t)(p.Vp1 - 1) : 0) <= 200 * 1024;
}

// bf16 logits on the CTA path (K <= 32 at B <= #SMs): the north-star shape reads them directly —
// the compaction pass takes the logits (fused log-softmax, records carry the lse) and the specialised
// records variant stages bf16 rows and normalises them in shared memory — so HBM carries 2 B per
// logit twice instead of 2 + 4 + 4 + 4 through a dense fp32 copy. Other shapes keep that copy
// (flexctc_decode_logits_bf16 in api.cu). Every knob that could steer the launch elsewhere
// (FLEXCTC_CMP / SOLO / NT / DENSE_MIN, FLEXCTC_LOGITS_DIRECT=0) turns it off.
bool cta_logits_direct(const DecodeParams& p) {
    if (!p.logits || !p.cmp || !p.rowoff || p.ready || p.nbest > 1 || p.fuse_rep || p.merge_first) return false;
    for (const char* e : {"FLEXCTC_CMP", "FLEXCTC_SOLO", "FLEXCTC_NT", "FLEXCTC_DENSE_MIN"})
        if (getenv(e)) return false;
    const char* e_ld = getenv("FLEXCTC_LOGITS_DIRECT");
    if (e_ld && e_ld[0] == '0') return false;
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    return p.K == 16 && p.Vp1 == 1025 && p.use_lm && p.lm.RW == 16 && p.lm.NL <= 2 && p.use_bt && p.merge_mode == 0 &&
           !p.retract && p.alpha_lm >= 0.0f && p.alpha_bt >= 0.0f && p.B <= nsm;
}

int launch_decode(const DecodeParams& p, void* stream, void* ev0, void* ev1, std::string& err, void* ev2, void* ev3) {
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(p.flags, 0, 64 + 8 * kStatsWords, st);
    if (e != cudaSuccess) { err = cudaGetErrorString(e); return 1; }
    if (p.B == 0) return 0;
    // K = 1 runs the greedy kernels (greedy_kernel.cu); FLEXCTC_GREEDY=0 keeps the beam kernel
    // (test switch: the two must agree)
    const char* e_gr = getenv("FLEXCTC_GREEDY");
    const bool greedy = p.K == 1 && p.greedy_sum && !(e_gr && e_gr[0] == '0') && !p.fuse_rep && !p.merge_first;
    const bool plain = greedy && !p.use_lm && !p.use_bt && p.beta == 0.0f;
    if (!plain) {  // the plain greedy path clamps lengths itself and needs no order
        order_kernel<<<(p.B + 255) / 256, 256, 0, st>>>(p.lengths, p.B, p.T, p.order, p.len_c, p.flags, p.B <= 16384);
        e = cudaGetLastError();
        if (e != cudaSuccess) { err = cudaGetErrorString(e); return 1; }
    }
    // which kernels run: merge-first, greedy, the warp path, or the CTA kernel (with or without the
    // compaction records). The CTA kernel reads the frame records of the compaction pass (the best
    // token, the listed band and its floor) instead of computing per-frame summaries from the rows
    // when the log-probs are resident and the decode has the north-star shape at B <= #SMs (beam
    // 16, V' = 1025, 4-gram LM + boosting: its specialised variant reads records, and with the
    // settled-beam fast path the helper warps' summaries are on the critical path: c4 1.542 ->
    // 1.535 ms per decode including the pass, profiles/r2/ab_records_fastpath.jsonl). Elsewhere the
    // pass costs more than it saves (c5 5.873 -> 5.961 ms, profiles/r2/cta_records_ab.jsonl).
    // FLEXCTC_CMP=0 / 1 forces it off / on (A/B and test switch).
    const bool warp = !p.merge_first && !greedy && use_warp_path(p);
    DecodeParams q = p;
    if (!p.merge_first && !greedy && !warp) {
        const char* e_cmp = getenv("FLEXCTC_CMP");
        int dev = 0, nsm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        bool want_cmp = p.K == 16 && p.Vp1 == 1025 && p.use_lm && p.lm.RW == 16 && p.use_bt && p.merge_mode == 0 &&
                        !p.retract && p.alpha_lm >= 0.0f && p.alpha_bt >= 0.0f && !p.fuse_rep && p.B <= nsm;
        if (e_cmp) want_cmp = e_cmp[0] == '1';
        q.use_cmp = p.cmp && p.rowoff && !p.ready && (!p.logits || cta_logits_direct(p)) && want_cmp ? 1 : 0;
        if (p.logits && !q.use_cmp) { err = "bf16 logits: the CTA kernel reads them only with records"; return 2; }
    }
    const bool compacts = warp || q.use_cmp;

    // L2 warm-up of the fusion tables the frame loop looks up at random: interleaved with the
    // compaction pass's rows when the decode runs one (no separate launch), else its own launch
    const char* e_w = getenv("FLEXCTC_L2_WARM");  // "0": no warm-up (A/B switch)
    WarmRanges wr;
    bool warm_in_pass = false;
    if ((p.use_lm || p.use_bt) && !(e_w && e_w[0] == '0') && !plain) {
        const char* e_wr = getenv("FLEXCTC_L2_WARM_REC");  // "1": also the LM state records (A/B)
        const bool warm_rec = e_wr && e_wr[0] == '1';
        wr.a[0] = (const char*)p.lm.dense; wr.n[0] = p.use_lm ? p.lm.dense_bytes : 0;
        wr.a[1] = (const char*)p.lm.arcs;  wr.n[1] = p.use_lm ? p.lm.arcs_bytes : 0;
        wr.a[2] = (const char*)p.bt.tab;   wr.n[2] = p.use_bt ? p.bt.tab_bytes : 0;
        wr.a[3] = (const char*)p.lm.rec;   wr.n[3] = p.use_lm && warm_rec ? p.lm.rec_bytes : 0;
        // "1": the pass issues the warm-up (c4 -0.3 %, but the pass's own time then carries 54 MB of
        // table prefetches its roofline does not count); default: the separate launch
        const char* e_wf = getenv("FLEXCTC_WARM_IN_PASS");
        warm_in_pass = compacts && compact_fuses_warm(p.Vp1, p.logits != nullptr) && (e_wf && e_wf[0] == '1');
        if (!warm_in_pass) {
            int dev = 0, nsm = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
            l2_warm_kernel<<<4 * nsm, 256, 0, st>>>(wr.a[0], wr.n[0], wr.a[1], wr.n[1], wr.a[2], wr.n[2], wr.a[3], wr.n[3]);
            e = cudaGetLastError();
            if (e != cudaSuccess) { err = cudaGetErrorString(e); return 1; }
        }
    }
    if (p.merge_first) return launch_merge_first(p, stream, ev0, ev1, err);  // reading R27
    if (greedy) return launch_greedy(p, stream, ev0, ev1, err);
    if (compacts) {
        // the bandwidth-bound compaction pass over every valid row, then the warp kernel (K <= 32,
        // one warp per utterance, warp_beam_kernel.cu) or the CTA kernel reading the records
        int rc = launch_rowoff(p.len_c, p.B, p.rowoff, stream, err);
        if (!rc && ev2 && ev3) cudaEventRecord((cudaEvent_t)ev2, st);
        if (!rc) rc = launch_compact(p.logits ? (const void*)p.logits : (const void*)p.log_probs, p.logits != nullptr,
                                     p.stride_b, p.stride_t, p.rowoff, p.B, p.T, p.Vp1, p.cmp, stream, err,
                                     warm_in_pass ? &wr : nullptr);
        if (!rc && ev2 && ev3) cudaEventRecord((cudaEvent_t)ev3, st);
        if (rc) return rc;
        if (warp) return launch_warp_beam(p, p.logits != nullptr, stream, ev0, ev1, err);
    }
    const bool small_lm = !p.use_lm || p.lm.NL <= 2;  // order <= 4: two arc levels
    return small_lm ? launch_lmv<2>(q, st, ev0, ev1, err) : launch_lmv<kMaxLmLevels>(q, st, ev0, ev1, err);
}

}  // namespace flexctc
