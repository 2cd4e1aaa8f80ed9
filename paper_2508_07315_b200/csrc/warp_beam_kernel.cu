// Warp-per-utterance CTC beam search for beams K <= 32: the latency-bound half of the frame step
// (§III-C Algorithm 1, score of Eq. (1)), after the bandwidth-bound
// frame compaction pass (compact_kernel.cu) has reduced every frame to a 256-B record.
//
// One warp owns one utterance at a time (LPT work queue); lane k holds beam slot k in registers
// (score, last label, 64-bit prefix hash, LM / boost states, bound terms). There are no CTA
// barriers and no helper warps: every step of a frame is warp-synchronous, so several utterances
// share an SM without interfering. Per frame t < L_b:
//  1. the ring (one TMA bulk copy of the frame row and one of its record, issued by lane 0
//     kWRing - 1 frames ahead, completion on an mbarrier) already holds D[b, t, :];
//  2. exact blank and repeat candidates per live slot (no β / fusion terms);
//  3. running threshold thr = max(fl(mx - θ), K-th best key so far): a candidate below the K-th
//     of any K candidates cannot enter the flat TopK, one below fl(max - θ) is pruned
//     (P:138-139);
//  4. non-blank, non-repeat candidates: token w can reach thr only if
//     D[w] >= thr - max acc - max ub (ub = β + α_LM·max_w P(w|s) + α_BT·max Δ); the record lists
//     the best tokens with an upper bound (floor) of the rest, so the row is scanned only when
//     the filter reaches below floor. Pairs (slot, token) whose bound reaches thr are scored
//     exactly (LM arc query + boost table, R19 order), 32 per round, thr raised between rounds;
//  5. flat TopK by rank counting over the candidate keys (score | ~flat index: ties to the lower
//     flat index, R9), θ-prune;
//  6. beams.update: parent state by warp shuffles, hash extension / LM / BT advance only on
//     emission (R5), u8 parent + u16 label backpointers, chunk ancestors;
//  7. recombination on (hash, last) with __match_any_sync (R12), log-sum-exp over the group in
//     (score desc, slot asc) order = slot order (R14), exp / log1p in fp64 rounded once.
// Then LM.Final, the final merge by transcript (R15) and the chunk-parallel
// backtrace. All score arithmetic is __fadd_rn / __fmaf_rn in the canonical order of R19.
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

#ifdef FLEXCTC_PHASE_TIMERS
#define WCLK() clock64()
#else
#define WCLK() 0ll
#endif

constexpr int kWBMax = 8;      // warps (utterances in flight) per CTA, at most
constexpr int kWRing = 4;      // frames in flight per warp (power of two)
constexpr int kCandCap = 128;  // candidate keys per warp
constexpr int kPairCap = 512;  // gathered (slot, token) pairs per chunk

struct WLayout {
    size_t rowslot, ring_rows, ring_recs, bars, ckey, cln, cbn, slots, pairs, tlist, endslot, rmeta, rows, total;
};

// nrow: NGPU-LM dense level-1 rows cached per warp (tag = row index u, loaded by TMA)
__host__ __device__ inline WLayout wlayout(int Vp1, int esz, int nch, int nrow) {
    auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
    WLayout L{};
    L.rowslot = al((size_t)Vp1 * esz + 30);  // covering 16-B blocks of a row at any alignment
    size_t o = 0;
    L.ring_rows = o; o += kWRing * L.rowslot;
    L.ring_recs = o; o += kWRing * (size_t)kCmpBytes;
    L.bars = o; o += al(8 * kWRing);
    L.ckey = o; o += 8 * (kCandCap + 2);  // + a zero sentinel for the paired loads of rank_pass
    L.cln = o; o += 4 * kCandCap;
    L.cbn = o; o += 4 * kCandCap;
    L.slots = o; o += 20 * 32 * 4;  // acc ub ua last lms bts sel rs ord rsort row cumu cumr sglo sghi bU bsglo bsghi (2 spare)
    L.pairs = o; o += 4 * kPairCap;
    L.tlist = o; o += al(2 * (size_t)Vp1);
    L.endslot = o; o += al(4 * (size_t)nch);
    L.rmeta = o; o += al(16 * (size_t)nrow);  // tag, last use, mbarrier per cached row
    L.rows = o; o += (size_t)nrow * (size_t)(Vp1 - 1) * 8;
    L.total = al(o);
    return L;
}

__device__ __forceinline__ float shf(float v, int s) { return __shfl_sync(0xffffffffu, v, s); }
__device__ __forceinline__ float ord_inv(uint32_t o) {  // inverse of ord_of
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}
__device__ __forceinline__ int shi(int v, int s) { return __shfl_sync(0xffffffffu, v, s); }

template <int LMV, bool BF16>
__global__ void __launch_bounds__(32 * kWBMax) warp_beam_kernel(const DecodeParams p, const int nrow) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int K = p.K, Vp1 = p.Vp1, blank = Vp1 - 1, V = Vp1 - 1;
    constexpr int esz = BF16 ? 2 : 4;
    const WLayout WL = wlayout(Vp1, esz, p.nch, nrow);
    unsigned char* ws = smem_raw + (size_t)wid * WL.total;
    unsigned char* ring_rows = ws + WL.ring_rows;
    unsigned char* ring_recs = ws + WL.ring_recs;
    uint64_t* bar = (uint64_t*)(ws + WL.bars);
    uint64_t* ckey = (uint64_t*)(ws + WL.ckey);
    int* cln = (int*)(ws + WL.cln);
    int* cbn = (int*)(ws + WL.cbn);
    float* s_acc = (float*)(ws + WL.slots);
    float* s_ub = s_acc + 32;
    float* s_ua = s_acc + 64;
    int* s_last = (int*)(s_acc + 96);
    int* s_lms = (int*)(s_acc + 128);
    int* s_bts = (int*)(s_acc + 160);
    int* s_sel = (int*)(s_acc + 192);
    float* s_rs = s_acc + 224;
    int* s_ord = (int*)(s_acc + 256);     // live slots by reach (desc) in pair frames
    float* s_rsort = s_acc + 288;         // their reach
    int* s_row = (int*)(s_acc + 320);
    float* s_cumu = s_acc + 352;
    float* s_cumr = s_acc + 384;
    uint32_t* s_sglo = (uint32_t*)(s_acc + 416);
    uint32_t* s_sghi = (uint32_t*)(s_acc + 448);
    float* s_bU = s_acc + 480;                     // boost: U of the slot's node
    uint32_t* s_bsglo = (uint32_t*)(s_acc + 512);  // boost: exception signature of the slot's node
    uint32_t* s_bsghi = (uint32_t*)(s_acc + 544);
    int* rtag = (int*)(ws + WL.rmeta);
    int* ruse = rtag + nrow;
    uint64_t* rbar = (uint64_t*)(ws + WL.rmeta + 8 * (size_t)nrow);
    const int2* rows = (const int2*)(ws + WL.rows);
    uint32_t* s_pairs = (uint32_t*)(ws + WL.pairs);
    uint16_t* tlist = (uint16_t*)(ws + WL.tlist);
    int* endslot = (int*)(ws + WL.endslot);
    int2* btroot = (int2*)(smem_raw + (size_t)(blockDim.x >> 5) * WL.total);

    const bool lm_on = p.use_lm != 0, bt_on = p.use_bt != 0;
    const bool ub_inf = (lm_on && p.alpha_lm < 0.0f) || (bt_on && p.alpha_bt < 0.0f);
    const int RW4 = lm_on ? p.lm.RW / 4 : 0;
    if (bt_on)
        for (int w = threadIdx.x; w < V; w += blockDim.x) btroot[w] = __ldg(&p.bt.tab[w]);
    if (lane == 0) {
        for (int i = 0; i < kWRing; ++i) mbar_init(&bar[i], 1);
        for (int i = 0; i < nrow; ++i) { mbar_init(&rbar[i], 1); rtag[i] = -1; ruse[i] = -1; }
        fence_mbar_init();
    }
    __syncthreads();
    uint32_t ph = 0;  // expected parity of each ring slot's next completion
    uint32_t rph = 0xffffffffu;  // parity of the latest load of each cached row (uniform over the warp)
    const char* xbase = BF16 ? (const char*)p.logits : (const char*)p.log_probs;
    const char* lo = xbase;
    const char* hi = xbase + (int64_t)esz * ((int64_t)(p.B - 1) * p.stride_b + (int64_t)(p.T - 1) * p.stride_t + Vp1);
#ifdef FLEXCTC_PHASE_TIMERS
    unsigned long long tm[18] = {};  // per frame class: wait, rb+rank, pairs, topk+update, merge, count
    // detail of frames with pairs (overwrites the scan-only class words): phase A, staging, scan,
    // gather loops, global-lookup evaluations, pushes that added keys
    long long tq = 0;
#endif
    unsigned long long st_frames = 0, st_alive = 0, st_listed = 0, st_eval = 0, st_scan = 0, st_pairfr = 0;
    unsigned long long st_batch = 0, st_lmg = 0, st_lmr = 0, st_rowld = 0;

    for (;;) {
        int u = 0;
        if (lane == 0) u = (int)atomicAdd(&p.flags[1], 1u);
        u = __shfl_sync(0xffffffffu, u, 0);
        if (u >= p.B) break;
        const int b = p.order[u];
        const int L = p.len_c[b];
        const int64_t bp_base = (int64_t)b * p.T * K;

        // ring: frame r -> slot r % kWRing (row via its covering 16-B blocks + the 256-B record)
        auto issue = [&](int r) {
            const int sl = r & (kWRing - 1);
            unsigned char* rs = ring_rows + sl * WL.rowslot;
            const char* src = xbase + ((int64_t)b * p.stride_b + (int64_t)r * p.stride_t) * esz;
            const char* g = (const char*)((uintptr_t)src & ~(uintptr_t)15);
            const uint32_t nb = (uint32_t)(((src - g) + (int64_t)Vp1 * esz + 15) & ~(int64_t)15);
            const bool bulk = g >= lo && g + nb <= hi;
            if (lane == 0) {
                fence_proxy_async();
                mbar_arrive_tx(&bar[sl], (bulk ? nb : 0u) + (uint32_t)kCmpBytes);
                bulk_g2s(ring_recs + sl * kCmpBytes, p.cmp + ((int64_t)b * p.T + r) * kCmpBytes, kCmpBytes, &bar[sl]);
                if (bulk) bulk_g2s(rs, g, nb, &bar[sl]);
            }
            if (!bulk) {  // the tensor's first / last row at the buffer edge: plain copy
                unsigned char* d = rs + (src - g);
                if (esz == 4)
                    for (int w = lane; w < Vp1; w += 32) ((float*)d)[w] = __ldg((const float*)src + w);
                else
                    for (int w = lane; w < Vp1; w += 32) ((uint16_t*)d)[w] = __ldg((const uint16_t*)src + w);
            }
        };

        // ------------------------------------------------------------ init (Alg. 1)
        float acc = lane == 0 ? 0.0f : kNeg;  // acc_scores[:,0] = 0, else -inf
        int last = blank;                     // R6
        uint64_t hash = 0ull;
        int lms = lm_on ? p.lm.start : 0;     // LM(<SOS>)
        int bts = 0;                          // BT(<0>) = root
        // the slot's LM record header: dense row u, cum_u, cum_root, bound, arc-level signature
        int lmu = -1, lrow = -1;
        bool fresh = false;                       // the state changed at the last frame step
        int arcn = 0, arco0 = 0, arcd0 = 0, arco1 = 0, arcd1 = 0;  // arc levels of the state
        float cumu = 0.0f, cumr = 0.0f, ublm = 0.0f;
        uint32_t sglo = 0, sghi = 0;
        if (lm_on) {
            const int4 h0 = __ldg(p.lm.rec + (size_t)lms * RW4), h1 = __ldg(p.lm.rec + (size_t)lms * RW4 + 1);
            lmu = h0.y; cumu = __int_as_float(h0.z); cumr = __int_as_float(h0.w);
            ublm = __int_as_float(h1.x); sglo = (uint32_t)h1.z; sghi = (uint32_t)h1.w;
        }
        float bmaxd = bt_on ? __ldg(&p.bt.maxd[0]) : 0.0f, bU = bt_on ? __ldg(&p.bt.U[0]) : 0.0f;
        uint32_t bsglo = 0, bsghi = 0;  // exception signature of the slot's boost node (root: none)
        int anc = 0;
        bool dead = false;
        for (int r = 0; r < kWRing - 1 && r < L; ++r) issue(r);
        int nissued = min(kWRing - 1, L), ncons = 0;

        for (int t = 0; t < L; ++t) {
            {
                const int r = t + kWRing - 1;
                __syncwarp();  // every lane's reads of the previous frame's buffers precede their reuse
                if (r < L) {
                    issue(r);
                    nissued = r + 1;
                }
            }
            [[maybe_unused]] const long long c_a = WCLK();
            const int sl = t & (kWRing - 1);
            mbar_wait(&bar[sl], (ph >> sl) & 1u);
            ph ^= 1u << sl;
            ncons = t + 1;
            const unsigned char* rc = ring_recs + sl * kCmpBytes;
            const unsigned char* rowb =
                ring_rows + sl * WL.rowslot + (((uintptr_t)(xbase + ((int64_t)b * p.stride_b + (int64_t)t * p.stride_t) * esz)) & 15);
            const float Dbl = ((const float*)rc)[0];
            const float floor_ = ((const float*)rc)[1];
            const int nlist = ((const int*)rc)[2];
            const double lse = BF16 ? *(const double*)(rc + 16) : 0.0;
            auto Dv = [&](int w) -> float {
                if constexpr (BF16) return (float)((double)bf16f(((const uint16_t*)rowb)[w]) - lse);
                else return ((const float*)rowb)[w];
            };

            [[maybe_unused]] const long long c_b = WCLK();
            // ------------------------------------------------ exact blank / repeat candidates
            const bool alive = lane < K && acc > kNeg;
            float sb = kNeg, sr = kNeg;
            if (alive) {
                sb = __fadd_rn(acc, Dbl);                          // blank: no β / fusion
                if (last != blank) sr = __fadd_rn(acc, Dv(last));  // repeat: no β / fusion
            }
            float ub = p.beta, ua = fabsf(p.beta);
            if (lm_on) { const float x = p.alpha_lm * ublm; ub += x; ua += fabsf(x); }
            if (bt_on) { const float x = p.alpha_bt * bmaxd; ub += x; ua += fabsf(x); }
            if (ub_inf) ub = INFINITY;
            const unsigned alivemask = __ballot_sync(0xffffffffu, alive);
            const int nalive = __popc(alivemask);
            // warp maxima in one redux.sync each (order-preserving integer images of the floats)
            const float accmax = ord_inv(__reduce_max_sync(0xffffffffu, ord_of(alive ? acc : kNeg)));
            const float reachmax = ord_inv(__reduce_max_sync(0xffffffffu, ord_of(alive ? __fadd_rn(acc, ub) : kNeg)));
            const float uamax = __uint_as_float(__reduce_max_sync(0xffffffffu, alive ? __float_as_uint(ua) : 0u));
            const float mxrb = ord_inv(__reduce_max_sync(0xffffffffu, ord_of(fmaxf(sb, sr))));
            // the candidate buffer holds only keys >= fl(max_rb - θ) (anything lower is pruned,
            // P:139, since the frame max is >= max_rb), compacted, never a zero key
            const float tau0 = __fsub_rn(mxrb, p.theta);
            int nc;
            {
                const bool okb = sb > kNeg && sb >= tau0, okr = sr > kNeg && sr >= tau0;
                const unsigned bb = __ballot_sync(0xffffffffu, okb), br = __ballot_sync(0xffffffffu, okr);
                const unsigned lt = (1u << lane) - 1u;
                if (okb) {
                    const int e = __popc(bb & lt);
                    ckey[e] = make_key(sb, flat_idx(lane, blank)); cln[e] = lms; cbn[e] = bts;
                }
                if (okr) {
                    const int e = __popc(bb) + __popc(br & lt);
                    ckey[e] = make_key(sr, flat_idx(lane, last)); cln[e] = lms; cbn[e] = bts;
                }
                nc = __popc(bb) + __popc(br);
            }
            __syncwarp();

            // ranks of the buffer keys (unique): s_sel[r] = entry of rank r < K
            auto rank_pass = [&](int n) {
                if (lane < K) s_sel[lane] = -1;
                if (lane == 0) ckey[n] = 0ull;  // sentinel: keys are read in pairs
                __syncwarp();
                const ulonglong2* k2 = (const ulonglong2*)ckey;
                const int n2 = (n + 1) >> 1;
                for (int e = lane; e < n; e += 32) {
                    const uint64_t me = ckey[e];
                    int r = 0;
#pragma unroll 4
                    for (int j = 0; j < n2; ++j) {
                        const ulonglong2 q = k2[j];
                        r += (q.x > me ? 1 : 0) + (q.y > me ? 1 : 0);
                    }
                    if (r < K) s_sel[r] = e;
                }
                __syncwarp();
            };
            rank_pass(nc);
            float thr = tau0;
            if (nc >= K) thr = fmaxf(thr, score_of(ckey[s_sel[K - 1]]));

            [[maybe_unused]] const long long c_c = WCLK();
            // dense-row cache (acquired lazily, on the first frame step that scores a pair): mark the
            // rows of the live slots used at t, load the missing ones (one TMA bulk copy each into
            // the least recently used row no live slot needs)
            bool rows_ready = nrow == 0;
            // want: the lanes that need their row now (every live slot on the first pair frame
            // step; only the slots whose state changed at t - 1 in the eager call below)
            auto acquire_rows = [&](bool want) {
                    // dense-row cache: mark the rows of the live slots used at t; load the missing ones
                    // (one TMA bulk copy each into the least recently used row no live slot needs)
                    if (alive && lrow >= 0) ruse[lrow] = t;
                    if (want && alive && lrow < 0 && lmu >= 0)
                        for (int r = 0; r < nrow; ++r)
                            if (rtag[r] == lmu) { lrow = r; ruse[r] = t; }
                    const bool miss = want && alive && lrow < 0 && lmu >= 0;
                    const unsigned mm = __ballot_sync(0xffffffffu, miss);
                    __syncwarp();
                    if (mm) {
                        const unsigned g = miss ? __match_any_sync(mm, lmu) : 0u;
                        unsigned leaders = __ballot_sync(0xffffffffu, miss && (g & ((1u << lane) - 1u)) == 0u);
                        while (leaders) {
                            const int src = __ffs(leaders) - 1;
                            leaders &= leaders - 1u;
                            const int uu = __shfl_sync(0xffffffffu, lmu, src);
                            const unsigned vk = lane < nrow && ruse[lane] < t ? (((unsigned)(ruse[lane] + 1)) << 5) | (unsigned)lane
                                                                              : 0xffffffffu;
                            const unsigned best = __reduce_min_sync(0xffffffffu, vk);
                            if (best == 0xffffffffu) break;  // every row serves a live slot: global path
                            const int v = (int)(best & 31u);
                            if (lane == 0) {
                                mbar_wait(&rbar[v], (rph >> v) & 1u);  // the row's previous load has landed
                                rtag[v] = uu;
                                ruse[v] = t;
                                fence_proxy_async();
                                mbar_arrive_tx(&rbar[v], (uint32_t)(V * 8));
                                bulk_g2s((void*)(rows + (size_t)v * V), p.lm.dense + (size_t)uu * V, (uint32_t)(V * 8), &rbar[v]);
                            }
                            rph ^= 1u << v;
                            ++st_rowld;
                            if (miss && lmu == uu) lrow = v;
                            __syncwarp();
                        }
                    }
                    __syncwarp();  // the reads of ruse / rtag above precede the next call's writes
            };
            // slots whose state changed at t - 1: get their dense rows now (TMA, lands while the
            // frame runs) and pull the arc lines of their LM state into L1 (the global lookups of
            // later frames then hit L1)
            if (__ballot_sync(0xffffffffu, fresh && alive)) {
                if (nrow > 0) acquire_rows(fresh);
                if (fresh && alive && lm_on) {
                    const int na = min(arcn, 2);
                    for (int j = 0; j < na; ++j) {
                        const int off = j ? arco1 : arco0, deg = j ? arcd1 : arcd0;
                        for (int i = 0; i < deg && i < 64; i += 8)
                            asm volatile("prefetch.global.L1 [%0];" ::"l"(p.lm.arcs + off + i));
                    }
                }
            }
            fresh = false;
            // ------------------------------------------------ non-blank, non-repeat candidates
            // Tokens best first: the record's sorted list, then (only if the filter still reaches
            // below its floor) the unlisted tokens from a scan of the row. The first few listed
            // tokens are scored with lane = slot (spike frames: one or two tokens, every slot);
            // the rest with lane = token, slot by slot, until no slot can reach thr. A pair is
            // scored exactly (Eq. (1), R19 order) only if its bound reaches thr; thr rises with
            // every push (fl(max - θ) and the K-th best key).
            const uint16_t* ltok = (const uint16_t*)(rc + 160);
            const float* lval = (const float*)(rc + 32);
            const float xthr = ((const float*)rc)[3];  // listed iff the raw value >= xthr
            auto dthr_of = [&](float th) -> float {     // a token reaching th has D >= dthr_of(th)
                if (ub_inf || !(th > kNeg)) return kNeg;
                const float mg = 1e-4f * (1.0f + fabsf(th) + fabsf(reachmax) + uamax);
                return __fsub_rn(__fsub_rn(th, reachmax), mg);
            };
            bool scanned = false, paired = false;
            int ntok = 0;
            // exact score of token w (log-prob d) from a slot given by its fields; key 0 if < thr
            // boost: from a non-root node u, a token outside u's exception signature has δ(u, w) =
            // δ(root, w) and delta = fl(delta(root, w) - U(u)) exactly (boost_build.cpp): the root
            // row in shared memory serves it; signature hits read the transition table
            auto eval = [&](float acc_k, float d, int w, int lms_k, int bts_k, int lrow_k, float cumu_k, float cumr_k,
                            uint32_t sglo_k, uint32_t sghi_k, float bU_k, uint32_t bsglo_k, uint32_t bsghi_k, int k,
                            int& ln, int& bn) -> uint64_t {
                float sx = __fadd_rn(__fadd_rn(acc_k, d), p.beta);
                ln = lms_k;
                bn = bts_k;
                int2 e = make_int2(0, 0);
                if (bt_on) {
                    const int bbit = lm_sig_bit(w);
                    if (bn == 0) {
                        e = btroot[w];
                    } else if (((bbit < 32 ? bsglo_k : bsghi_k) >> (bbit & 31)) & 1u) {
                        e = __ldg(&p.bt.tab[(size_t)bn * V + w]);
                    } else {
                        const int2 r = btroot[w];
                        e = make_int2(r.x, __float_as_int(__fsub_rn(__int_as_float(r.y), bU_k)));
                    }
                }
                if (lm_on) {
                    float lp;
                    const int sbit = lm_sig_bit(w);
                    const uint32_t sg = (sbit < 32 ? sglo_k : sghi_k) >> (sbit & 31);
                    if (lrow_k >= 0 && !(sg & 1u)) {
                        // no arc level holds w: the cached dense row decides (lm_query's dense
                        // path, the same fp32 operation)
                        mbar_wait(&rbar[lrow_k], (rph >> lrow_k) & 1u);
                        const int2 de = rows[(size_t)lrow_k * V + w];
                        lp = __fadd_rn((de.y & 0x80000000) ? cumu_k : cumr_k, __int_as_float(de.x));
                        ln = de.y & 0x7fffffff;
                        ++st_lmr;
                    } else {
                        lp = lm_query<LMV>(p.lm, (const int*)(p.lm.rec + (size_t)ln * RW4), w, ln);
                        ++st_lmg;
                    }
                    sx = __fmaf_rn(p.alpha_lm, lp, sx);
                }
                if (bt_on) { bn = e.x; sx = __fmaf_rn(p.alpha_bt, __int_as_float(e.y), sx); }
                return (sx > kNeg && sx >= thr) ? make_key(sx, flat_idx(k, w)) : 0ull;
            };
            // append the non-zero keys of the lanes, then re-rank and raise thr
            auto push = [&](uint64_t key, int ln, int bn) {
                ++st_batch;
                const unsigned kb = __ballot_sync(0xffffffffu, key != 0ull);
                if (!kb) return;
#ifdef FLEXCTC_PHASE_TIMERS
                tm[11] += 1;
#endif
                if (nc + __popc(kb) > kCandCap) {  // keep the top K keys first
                    const int ke = lane < K && lane < nc ? s_sel[lane] : -1;
                    const uint64_t k1 = ke >= 0 ? ckey[ke] : 0ull;
                    const int l1 = ke >= 0 ? cln[ke] : 0, b1 = ke >= 0 ? cbn[ke] : 0;
                    __syncwarp();
                    if (ke >= 0) { ckey[lane] = k1; cln[lane] = l1; cbn[lane] = b1; }
                    nc = min(nc, K);
                }
                if (key) {
                    const int dd = nc + __popc(kb & ((1u << lane) - 1u));
                    ckey[dd] = key; cln[dd] = ln; cbn[dd] = bn;
                    if (lm_on) asm volatile("prefetch.global.L1 [%0];" ::"l"(p.lm.rec + (size_t)ln * RW4));
                }
                nc += __popc(kb);
                __syncwarp();
                rank_pass(nc);
                thr = fmaxf(thr, __fsub_rn(score_of(ckey[s_sel[0]]), p.theta));
                if (nc >= K) thr = fmaxf(thr, score_of(ckey[s_sel[K - 1]]));
            };
            if (nalive > 0) {
#ifdef FLEXCTC_PHASE_TIMERS
                tq = clock64();
#define TQ(i) do { const long long _n = clock64(); tm[6 + (i)] += _n - tq; tq = _n; } while (0)
#else
#define TQ(i) do { } while (0)
#endif
                // (A) the best listed token, lane = slot (own registers): on emission frames it
                // lifts thr to about fl(max - θ) before the other tokens are looked at
                if (nlist > 0) {
                    const float d = lval[0];
                    if (d >= dthr_of(thr)) {
                        const int w = ltok[0];
                        ++ntok;
                        bool pass = false;
                        if (alive && w != last) {
                            const float s0 = __fadd_rn(acc, d);
                            pass = __fadd_rn(s0, ub) + 1e-5f * (1.0f + fabsf(s0) + ua) >= thr;
                        }
                        const unsigned pb = __ballot_sync(0xffffffffu, pass);
                        if (pb) {
                            paired = true;
                            if (!rows_ready) { acquire_rows(alive); rows_ready = true; }
                            st_eval += __popc(pb);
                            int ln = 0, bn = 0;
                            const uint64_t key = pass ? eval(acc, d, w, lms, bts, lrow, cumu, cumr, sglo, sghi, bU, bsglo, bsghi, lane, ln, bn) : 0ull;
                            push(key, ln, bn);
                        }
                    }
                }
                TQ(0);
                const int jA = nlist > 0 ? 1 : 0;  // token 0 was scored in (A), or no listed token passes
                // (B) the rest, lane = token: listed tokens [jA, m0), then the scanned ones. Per chunk
                // of 32 tokens: gather every (slot, token) pair whose bound reaches thr (slots in
                // index order, until the suffix maximum of the reach fails), then score them: the
                // cheap ones (cached dense row, boost at the root) 32 per round, then the ones that
                // need the global arc search / boost table together, then one re-rank.
                bool staged = false;
                auto process_B = [&](bool scan, int j_begin, int m) {
                    if (!staged) {  // per-slot values for the token lanes; live slots by reach (desc)
                        if (!rows_ready) { acquire_rows(alive); rows_ready = true; }
                        const float myr = alive ? __fadd_rn(acc, ub) : kNeg;
                        if (lane < K) {
                            s_acc[lane] = alive ? acc : kNeg; s_ub[lane] = ub; s_ua[lane] = ua;
                            s_last[lane] = last; s_lms[lane] = lms; s_bts[lane] = bts;
                            s_row[lane] = lrow; s_cumu[lane] = cumu; s_cumr[lane] = cumr;
                            s_sglo[lane] = sglo; s_sghi[lane] = sghi; s_rs[lane] = myr;
                            s_bU[lane] = bU; s_bsglo[lane] = bsglo; s_bsghi[lane] = bsghi;
                        }
                        __syncwarp();
                        if (alive) {
                            int r = 0;
#pragma unroll 4
                            for (int j = 0; j < K; ++j) {
                                const float rj = s_rs[j];
                                r += (rj > myr || (rj == myr && j < lane)) ? 1 : 0;
                            }
                            s_ord[r] = lane;
                            s_rsort[r] = myr;
                        }
                        __syncwarp();
                        staged = true;
                        TQ(1);
                    }
                    for (int j0 = j_begin; j0 < m; j0 += 32) {
                        const int j = j0 + lane;
                        const int w = j < m ? (scan ? (int)tlist[j] : (int)ltok[j]) : -1;
                        const float d = w >= 0 ? (scan ? Dv(w) : lval[j]) : kNeg;
                        const float dmx = ord_inv(__reduce_max_sync(0xffffffffu, ord_of(d)));
                        bool any_slot = false;
                        int kk = 0;
                        for (;;) {
                            int nexp = 0;
                            bool stop = false;
                            for (; kk < nalive; ++kk) {
                                const int k = s_ord[kk];
                                const float sfk = s_rsort[kk];
                                if (__fadd_rn(dmx, sfk) + 1e-4f * (1.0f + fabsf(dmx) + fabsf(sfk) + uamax) < thr) {
                                    stop = true;  // slots by reach: no later slot reaches thr with these tokens
                                    break;
                                }
                                any_slot = true;
                                // a pair whose LM value is in a cached dense row and whose boost state is
                                // the root is scored exactly right here (shared-memory loads only); the
                                // others that pass the bound are gathered for the global lookups
                                bool pass = false, cheap = false;
                                uint64_t keyc = 0;
                                int lnc = 0, bnc = 0;
                                if (w >= 0 && w != s_last[k]) {
                                    const float s0 = __fadd_rn(s_acc[k], d);
                                    pass = __fadd_rn(s0, s_ub[k]) + 1e-5f * (1.0f + fabsf(s0) + s_ua[k]) >= thr;
                                    if (pass) {
                                        const int sbit = lm_sig_bit(w);
                                        const uint32_t sg = (sbit < 32 ? s_sglo[k] : s_sghi[k]) >> (sbit & 31);
                                        const uint32_t bsg = (sbit < 32 ? s_bsglo[k] : s_bsghi[k]) >> (sbit & 31);
                                        cheap = (!lm_on || (s_row[k] >= 0 && !(sg & 1u))) &&
                                                (!bt_on || s_bts[k] == 0 || !(bsg & 1u));
                                        if (cheap)
                                            keyc = eval(s_acc[k], d, w, s_lms[k], s_bts[k], s_row[k], s_cumu[k], s_cumr[k],
                                                        s_sglo[k], s_sghi[k], s_bU[k], s_bsglo[k], s_bsghi[k], k, lnc, bnc);
                                    }
                                }
                                const unsigned pc = __ballot_sync(0xffffffffu, pass && cheap);
                                if (pc) {
                                    paired = true;
                                    st_eval += __popc(pc);
                                    push(keyc, lnc, bnc);
                                }
                                const unsigned pe = __ballot_sync(0xffffffffu, pass && !cheap);
                                const unsigned lt = (1u << lane) - 1u;
                                const uint32_t pq = ((uint32_t)k << 8) | (uint32_t)lane;
                                if (pass && !cheap) s_pairs[nexp + __popc(pe & lt)] = pq;
                                nexp += __popc(pe);
                                if (nexp > kPairCap - 32) { ++kk; break; }  // full: score, then go on
                            }
                            __syncwarp();
                            TQ(3);
                            const int np = nexp;
                            if (np) {
                                paired = true;
                                st_eval += np;
                                for (int q0 = 0; q0 < np; q0 += 32) {
                                    const int q = q0 + lane;
                                    uint64_t key = 0;
                                    int ln = 0, bn = 0;
                                    if (q < np) {
                                        const uint32_t pq = s_pairs[q];
                                        const int kq = (int)(pq >> 8), jl = (int)(pq & 255u);
                                        const int wq = scan ? (int)tlist[j0 + jl] : (int)ltok[j0 + jl];
                                        const float dq = scan ? Dv(wq) : lval[j0 + jl];
                                        key = eval(s_acc[kq], dq, wq, s_lms[kq], s_bts[kq], s_row[kq], s_cumu[kq], s_cumr[kq],
                                                   s_sglo[kq], s_sghi[kq], s_bU[kq], s_bsglo[kq], s_bsghi[kq], kq, ln, bn);
                                    }
                                    push(key, ln, bn);
                                }
                            }
                            __syncwarp();  // the batch's reads of s_pairs precede the next gather
                            TQ(4);
                            if (stop || kk >= nalive) break;
                        }
                        if (!any_slot && !scan) break;  // sorted list: later chunks are lower still
                    }
                };
                const float dt0 = dthr_of(thr);
                const int m0 = __popc(__ballot_sync(0xffffffffu, lane < nlist && lval[lane < nlist ? lane : 0] >= dt0));
                if (m0 > jA) { ntok += m0 - jA; process_B(false, jA, m0); }
                const float dt1 = dthr_of(thr);
#ifdef FLEXCTC_PHASE_TIMERS
                tq = clock64();
#endif
                if (floor_ >= dt1) {
                    // the filter reaches below the listed band: scan the row for the rest
                    scanned = true;
                    int m1 = 0;
                    for (int w0 = 0; w0 < blank; w0 += 32) {
                        const int w = w0 + lane;
                        bool hit = false;
                        if (w < blank) {
                            const float x = BF16 ? bf16f(((const uint16_t*)rowb)[w]) : ((const float*)rowb)[w];
                            hit = x < xthr && Dv(w) >= dt1;
                        }
                        const unsigned bal = __ballot_sync(0xffffffffu, hit);
                        if (hit) tlist[m1 + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)w;
                        m1 += __popc(bal);
                    }
                    __syncwarp();
                    TQ(2);
                    ntok += m1;
                    if (m1) process_B(true, 0, m1);
                }
            }
            st_frames += 1;
            st_alive += nalive;
            st_listed += ntok;
            st_scan += scanned ? 1 : 0;
            st_pairfr += paired ? 1 : 0;

            [[maybe_unused]] const long long c_d = WCLK();
            // ------------------------------------------------ flat TopK + θ-prune
            // s_sel holds the entries of ranks 0..K-1 from the last rank_pass (the buffer has not
            // changed since); ties are impossible: the flat index is part of the key (R9)
            const int myent = lane < K && lane < nc ? s_sel[lane] : -1;
            const uint64_t mykey = myent >= 0 ? ckey[myent] : 0ull;
            const int myln = myent >= 0 ? cln[myent] : 0, mybn = myent >= 0 ? cbn[myent] : 0;
            const uint64_t topk = __shfl_sync(0xffffffffu, mykey, 0);
            if (!topk) { dead = true; break; }  // no finite candidate: every hypothesis dies
            const float tau = __fsub_rn(score_of(topk), p.theta);
            const float s_new = mykey ? score_of(mykey) : kNeg;
            const bool live = mykey && s_new >= tau;

            // ------------------------------------------------ beams.update
            const uint32_t f = flat_of(mykey);
            const int par = live ? (int)(f >> 16) : lane;
            const int w = (int)(f & 0xffffu);
            const int p_last = shi(last, par);
            const uint32_t ph_lo = (uint32_t)__shfl_sync(0xffffffffu, (uint32_t)hash, par);
            const uint32_t ph_hi = (uint32_t)__shfl_sync(0xffffffffu, (uint32_t)(hash >> 32), par);
            const uint64_t p_hash = ((uint64_t)ph_hi << 32) | ph_lo;
            const float p_ublm = shf(ublm, par), p_maxd = shf(bmaxd, par), p_U = shf(bU, par);
            const uint32_t p_bsglo = (uint32_t)shi((int)bsglo, par), p_bsghi = (uint32_t)shi((int)bsghi, par);
            const float p_cumu = shf(cumu, par), p_cumr = shf(cumr, par);
            const int p_lmu = shi(lmu, par), p_lrow = shi(lrow, par);
            const uint32_t p_sglo = (uint32_t)shi((int)sglo, par), p_sghi = (uint32_t)shi((int)sghi, par);
            const int p_anc = shi(anc, par);
            const bool emit = live && w != blank && w != p_last;
            float n_acc = kNeg;
            int n_last = blank, n_lms = 0, n_bts = 0, n_anc = 0;
            uint64_t n_hash = 0ull;
            float n_ublm = 0.0f, n_maxd = 0.0f, n_U = 0.0f, n_cumu = 0.0f, n_cumr = 0.0f;
            uint32_t n_bsglo = 0, n_bsghi = 0;
            int n_lmu = -1, n_lrow = -1, n_arcn = 0, n_arco0 = 0, n_arcd0 = 0, n_arco1 = 0, n_arcd1 = 0;
            uint32_t n_sglo = 0, n_sghi = 0;
            if (live) {
                n_acc = s_new;
                n_last = w;
                n_hash = emit ? hash_extend(p_hash, w) : p_hash;
                n_lms = myln;  // rb candidates carry the parent's states (buffer entries)
                n_bts = mybn;
                n_anc = (t % kChunk == 0) ? par : p_anc;
                if (emit) {  // new LM / BT states: their record headers (latency overlaps the merge)
                    if (lm_on) {
                        const int4 h0 = __ldg(p.lm.rec + (size_t)n_lms * RW4), h1 = __ldg(p.lm.rec + (size_t)n_lms * RW4 + 1);
                        n_lmu = h0.y; n_cumu = __int_as_float(h0.z); n_cumr = __int_as_float(h0.w);
                        n_ublm = __int_as_float(h1.x); n_sglo = (uint32_t)h1.z; n_sghi = (uint32_t)h1.w;
                        if (RW4 >= 4) {  // arc levels 0 and 1 (same 64-B record line)
                            const int4 h2 = __ldg(p.lm.rec + (size_t)n_lms * RW4 + 2), h3 = __ldg(p.lm.rec + (size_t)n_lms * RW4 + 3);
                            n_arcn = h0.x; n_arco0 = h2.x; n_arcd0 = h2.y; n_arco1 = h2.w; n_arcd1 = h3.x;
                        }
                    }
                    n_maxd = bt_on ? __ldg(&p.bt.maxd[n_bts]) : 0.0f;
                    n_U = bt_on ? __ldg(&p.bt.U[n_bts]) : 0.0f;
                    if (bt_on) {
                        const unsigned long long sg = __ldg(&p.bt.sig[n_bts]);
                        n_bsglo = (uint32_t)sg; n_bsghi = (uint32_t)(sg >> 32);
                    }
                } else {
                    n_ublm = p_ublm; n_maxd = p_maxd; n_U = p_U; n_bsglo = p_bsglo; n_bsghi = p_bsghi;
                    n_lmu = p_lmu; n_lrow = p_lrow; n_cumu = p_cumu; n_cumr = p_cumr; n_sglo = p_sglo; n_sghi = p_sghi;
                }
                const int64_t o = bp_base + (int64_t)t * K + lane;
                p.bp_parent[o] = (uint8_t)par;
                p.bp_label[o] = (uint16_t)w;
            }
            if (lane < K && ((t % kChunk) == kChunk - 1 || t == L - 1))
                p.chunk_anc[((int64_t)b * p.nch + t / kChunk) * K + lane] = (uint8_t)n_anc;

            [[maybe_unused]] const long long c_e = WCLK();
            // ------------------------------------------------ RecombineHypotheses
            const unsigned livemask = __ballot_sync(0xffffffffu, live);
            unsigned grp = 0;
            if (live) grp = __match_any_sync(livemask, n_hash) & __match_any_sync(livemask, n_last);
            float s_m = n_acc;
            const bool leader = live && (grp & ((1u << lane) - 1u)) == 0u;
            unsigned oth = leader ? (grp & ~(1u << lane)) : 0u;  // higher slots of the group, ascending
            if (live && !leader) s_m = kNeg;                     // a better (lower) slot survives
            if (p.merge_mode == 0) {
                float sum = 0.0f;
                bool any = false;
                while (__any_sync(0xffffffffu, oth != 0u)) {
                    const int src = oth ? __ffs(oth) - 1 : lane;
                    const float v = shf(n_acc, src);
                    if (oth) {
                        sum = __fadd_rn(sum, (float)exp((double)__fsub_rn(v, n_acc)));
                        any = true;
                        oth &= oth - 1u;
                    }
                }
                if (any) s_m = __fadd_rn(n_acc, (float)log1p((double)sum));
            }
            acc = s_m;
            last = n_last;
            hash = n_hash;
            lms = n_lms;
            bts = n_bts;
            anc = n_anc;
            ublm = n_ublm;
            bmaxd = n_maxd;
            bsglo = n_bsglo; bsghi = n_bsghi;
            bU = n_U;
            lmu = n_lmu; lrow = n_lrow; cumu = n_cumu; cumr = n_cumr; sglo = n_sglo; sghi = n_sghi;
            fresh = emit;
            arcn = n_arcn; arco0 = n_arco0; arcd0 = n_arcd0; arco1 = n_arco1; arcd1 = n_arcd1;
            if (!(acc > kNeg)) {
                acc = kNeg; last = blank; hash = 0ull; lms = 0; bts = 0; ublm = 0.0f; bmaxd = 0.0f; bU = 0.0f;
                bsglo = 0; bsghi = 0;
                lmu = -1; lrow = -1;
            }
#ifdef FLEXCTC_PHASE_TIMERS
            {
                const long long c_f = WCLK();
                if (paired || !scanned) {
                    const int base = paired ? 0 : 12;  // pair frames / light (scan-only frames: not timed)
                    tm[base + 0] += c_b - c_a; tm[base + 1] += c_c - c_b; tm[base + 2] += c_d - c_c;
                    tm[base + 3] += c_e - c_d; tm[base + 4] += c_f - c_e; tm[base + 5] += 1;
                }
            }
#endif
        }
        for (int f2 = ncons; f2 < nissued; ++f2) {  // rows issued past a dead frame: drain the ring
            const int sl = f2 & (kWRing - 1);
            mbar_wait(&bar[sl], (ph >> sl) & 1u);
            ph ^= 1u << sl;
        }
        __syncwarp();

        // ------------------------------------------------------------ EOS + final merge (R15)
        const bool al = !dead && lane < K && acc > kNeg;
        float fs = al ? acc : kNeg;
        if (al) {
            if (lm_on) fs = __fmaf_rn(p.alpha_lm, __int_as_float(__ldg((const int*)(p.lm.rec + (size_t)lms * RW4) + 5)), fs);
            if (bt_on && p.retract) fs = __fmaf_rn(-p.alpha_bt, bU, fs);
        }
        if (lane < K) s_acc[lane] = al ? fs : kNeg;  // the merge below reads the others' EOS scores here
        __syncwarp();
        // group the live slots by transcript (hash); survivor = (score desc, slot asc)
        const unsigned almask = __ballot_sync(0xffffffffu, al);
        unsigned g2 = 0;
        if (al) g2 = __match_any_sync(almask, hash);
        bool surv = al;
        {
            unsigned o2 = al ? (g2 & ~(1u << lane)) : 0u;
            while (__any_sync(0xffffffffu, o2 != 0u)) {
                const int src = o2 ? __ffs(o2) - 1 : lane;
                const float v = shf(fs, src);
                if (o2) {
                    if (v > fs || (v == fs && src < lane)) surv = false;
                    o2 &= o2 - 1u;
                }
            }
        }
        float fm = fs;
        if (surv && p.merge_mode == 0) {
            // other members in (score desc, slot asc) order
            float sum = 0.0f;
            bool any = false;
            float prev_s = INFINITY;
            int prev_j = -1;
            const unsigned mem = g2 & ~(1u << lane);
            for (;;) {
                int bj = -1;
                float bs = kNeg;
                unsigned mm = mem;
                while (mm) {  // divergent per lane: no shuffles, the scores come from shared memory
                    const int j = __ffs(mm) - 1;
                    mm &= mm - 1u;
                    const float sj = s_acc[j];
                    if (!(sj < prev_s || (sj == prev_s && j > prev_j))) continue;
                    if (bj < 0 || sj > bs || (sj == bs && j < bj)) { bj = j; bs = sj; }
                }
                if (bj < 0) break;
                any = true;
                sum = __fadd_rn(sum, (float)exp((double)__fsub_rn(bs, fs)));
                prev_s = bs;
                prev_j = bj;
            }
            if (any) fm = __fadd_rn(fs, (float)log1p((double)sum));
        }
        // best survivor by (merged score desc, slot asc)
        uint64_t bk = surv ? (((uint64_t)ord_of(fm) << 32) | (uint64_t)(0xffffffffu - (uint32_t)lane)) : 0ull;
#pragma unroll
        for (int o = 16; o; o >>= 1) bk = umax64(bk, __shfl_xor_sync(0xffffffffu, bk, o));
        const bool has_best = bk != 0ull;
        const int best = has_best ? (int)(0xffffffffu - (uint32_t)bk) : -1;
        const float best_score = has_best ? score_of(bk) : kNeg;

        // ------------------------------------------------------------ backtrace + collapse (R20)
        int32_t* align = (p.out_align ? p.out_align : p.align_ws) + (int64_t)b * p.T;
        const int nchk = (L + kChunk - 1) / kChunk;
        if (has_best && L > 0) {
            if (lane == 0) {
                int s = best;
                endslot[nchk - 1] = s;
                for (int c = nchk - 1; c >= 1; --c) {
                    s = p.chunk_anc[((int64_t)b * p.nch + c) * K + s];
                    endslot[c - 1] = s;
                }
            }
            __syncwarp();
            for (int c = lane; c < nchk; c += 32) {
                int s = endslot[c];
                const int t_hi = min(c * kChunk + kChunk - 1, L - 1);
                for (int t = t_hi; t >= c * kChunk; --t) {
                    const int64_t o = bp_base + (int64_t)t * K + s;
                    align[t] = p.bp_label[o];
                    s = p.bp_parent[o];
                }
            }
        }
        __syncwarp();
        int32_t* otok = p.out_tokens + (int64_t)b * p.T;
        int32_t* ots = p.out_ts ? p.out_ts + (int64_t)b * p.T : nullptr;
        int ntok = 0;
        if (has_best) {
            for (int t0 = 0; t0 < L; t0 += 32) {
                const int t = t0 + lane;
                const int at = t < L ? align[t] : blank;
                const int ap = t == 0 ? blank : (t < L ? align[t - 1] : blank);
                const bool em = t < L && at != blank && at != ap;
                const unsigned bal = __ballot_sync(0xffffffffu, em);
                if (em) {
                    const int q = ntok + __popc(bal & ((1u << lane) - 1u));
                    otok[q] = at;
                    if (ots) ots[q] = t;
                }
                ntok += __popc(bal);
            }
        }
        for (int i = ntok + lane; i < p.T; i += 32) { otok[i] = -1; if (ots) ots[i] = -1; }
        if (p.out_align)
            for (int i = (has_best ? L : 0) + lane; i < p.T; i += 32) p.out_align[(int64_t)b * p.T + i] = -1;
        if (lane == 0) {
            p.out_num[b] = ntok;
            p.out_scores[b] = best_score;
        }
        __syncwarp();
    }
    if (lane == 0) {
        atomicAdd(&p.stats[kFrames], st_frames);
        atomicAdd(&p.stats[kAlive], st_alive);
        atomicAdd(&p.stats[kListed], st_listed);
        atomicAdd(&p.stats[kEvalSparse], st_eval);
        atomicAdd(&p.stats[kDenseFrames], st_scan);     // frames whose filter needed the row scan
        atomicAdd(&p.stats[kHeavyFrames], st_pairfr);   // frames with candidate pairs
        atomicAdd(&p.stats[24], st_batch);   // scoring batches (one ballot of pairs)
        atomicAdd(&p.stats[25], st_rowld);   // dense rows loaded into the cache
    }
    {  // per-lane counts: LM lookups through the global arc search / the cached dense rows
        const unsigned long long a = st_lmg, c = st_lmr;
        atomicAdd(&p.stats[26], a);
        atomicAdd(&p.stats[27], c);
    }
    if (lane == 0) {
#ifdef FLEXCTC_PHASE_TIMERS
        for (int i = 0; i < 18; ++i) atomicAdd(&p.stats[30 + i], tm[i]);  // words 30..47
#endif
    }
}

}  // namespace

// Warp-per-utterance beam path (K <= 32): frame_compact_kernel (launched by the caller) then
// this kernel. Warps per CTA: 1 while the batch fits the SMs (one utterance per SM: the
// shortest frame step), else up to kWBMax, as shared memory allows.
size_t warp_beam_smem_per_warp(int Vp1, bool bf16, int nch) { return wlayout(Vp1, bf16 ? 2 : 4, nch, 0).total; }

int launch_warp_beam(const DecodeParams& p, bool bf16, void* stream, void* ev0, void* ev1, std::string& err) {
    cudaStream_t st = (cudaStream_t)stream;
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const size_t per = wlayout(p.Vp1, bf16 ? 2 : 4, p.nch, 0).total;
    const size_t root = p.use_bt ? 8 * (size_t)(p.Vp1 - 1) : 0;
    int wpc = std::min(kWBMax, std::max(1, (p.B + nsm - 1) / nsm));
    while (wpc > 1 && wpc * per + root > 200 * 1024) --wpc;
    // dense-row cache: as many rows (<= 16) as the shared memory left per warp holds
    int nrow = 0;
    if (p.use_lm && ((p.Vp1 - 1) & 1) == 0 && wpc * per + root <= 200 * 1024) {  // rows of 16-B multiples
        const size_t rowb = (size_t)(p.Vp1 - 1) * 8 + 16;
        const size_t left = 200 * 1024 - (wpc * per + root);
        nrow = (int)std::min<size_t>(16, left / (wpc * rowb));
        if (const char* e = getenv("FLEXCTC_WARP_ROWS")) nrow = std::min(nrow, std::max(0, atoi(e)));  // A/B switch
    }
    const size_t per2 = wlayout(p.Vp1, bf16 ? 2 : 4, p.nch, nrow).total;
    const size_t smem = wpc * per2 + root;
    if (smem > 200 * 1024) { err = "shared memory requirement too large (V+1 or T)"; return 2; }
    const bool small_lm = !p.use_lm || p.lm.NL <= 2;
    void (*kern)(const DecodeParams, int);
    if (small_lm) kern = bf16 ? warp_beam_kernel<2, true> : warp_beam_kernel<2, false>;
    else kern = bf16 ? warp_beam_kernel<kMaxLmLevels, true> : warp_beam_kernel<kMaxLmLevels, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * wpc, smem);
    if (e != cudaSuccess || occ < 1) { err = e != cudaSuccess ? cudaGetErrorString(e) : "occupancy query failed"; return 1; }
    const int grid = std::min((p.B + wpc - 1) / wpc, nsm * occ);
    if (ev0 && ev1) cudaEventRecord((cudaEvent_t)ev0, st);
    kern<<<grid, 32 * wpc, smem, st>>>(p, nrow);
    set_kernel_name("warp_beam_kernel");
    e = cudaGetLastError();
    if (e == cudaSuccess && ev0 && ev1) cudaEventRecord((cudaEvent_t)ev1, st);
    if (e != cudaSuccess) { err = cudaGetErrorString(e); return 1; }
    return 0;
}

}  // namespace flexctc
