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
//    work queue (LPT), the whole frame loop in-kernel: zero host syncs, one launch per decode;
//  * frame rows D[b,t,:] streamed HBM -> shared memory with cp.async (16 B when aligned) in a
//    ring R frames ahead of the recurrence, so the only O(B·T·V') HBM stream overlaps it;
//  * exact pre-prune: the blank/repeat candidates (no fusion terms) give a lower bound mx0 of the
//    frame max, hence τ0 = fl(mx0 - θ) <= τ; a non-blank candidate is scored exactly (LM arc
//    search in L2 + boost table lookup) only if acc + D + ub(state) can reach τ0 (ub = β +
//    α_LM·max_w P(w|lm) + α_BT·max_w delta(bt) + rounding margin). Everything below τ0 is pruned
//    by Alg. 1 anyway, so the live beam is bit-identical to the dense [K, V'] evaluation;
//  * survivors go to a shared-memory buffer of 64-bit keys (orderable fp32 score | ~flat index);
//    when it fills, a block radix-select keeps the top K and raises the threshold (threshold
//    algorithm), so any candidate count (θ = ∞, flat frames) works in bounded memory;
//  * selection = radix-select of the K-th key + rank sort of K keys; ties go to the lower flat
//    index (reading R9) because the index is in the key;
//  * recombination on (64-bit prefix hash, last label) (R12) over the K slots, log-sum-exp in the
//    canonical order (R14) with exp/log1p evaluated in fp64 and rounded once;
//  * backpointers u8 parent + u16 label per (t, k) in global memory plus per-32-frame chunk
//    ancestors, so the backtrace walks chunks in parallel (T/32 + 32 dependent loads, not T).
// All score arithmetic uses __fadd_rn/__fmaf_rn in the canonical order of reading R19 (no
// contraction, no fast-math), so max-mode scores are bit-identical to the fp32 oracle.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <string>

#include "flexctc_internal.h"

namespace flexctc {
namespace {

constexpr float kNeg = -INFINITY;

__device__ __forceinline__ uint64_t hash_extend(uint64_t h, int w) {  // SPEC S:58 (FNV-64 prime)
    return (h ^ (uint64_t)(w + 1)) * 1099511628211ull;
}

__device__ __forceinline__ uint32_t ord_of(float s) {
    uint32_t u = __float_as_uint(s);
    if (u == 0x80000000u) u = 0u;  // -0 == +0
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float score_of(uint64_t key) {
    uint32_t o = (uint32_t)(key >> 32);
    uint32_t u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
    return __uint_as_float(u);
}
__device__ __forceinline__ uint64_t make_key(float s, uint32_t f) {
    return ((uint64_t)ord_of(s) << 32) | (uint64_t)(0xffffffffu - f);
}
__device__ __forceinline__ uint32_t flat_of(uint64_t key) { return 0xffffffffu - (uint32_t)key; }

__device__ __forceinline__ void cp_async4(void* s, const void* g) {
    uint32_t sa = (uint32_t)__cvta_generic_to_shared(s);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(g));
}
__device__ __forceinline__ void cp_async16(void* s, const void* g) {
    uint32_t sa = (uint32_t)__cvta_generic_to_shared(s);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// NGPU-LM query: log P(w | state) and the next state (walk the backoff chain; arcs are sorted by
// token within a state). Same arithmetic order as lm_query_host and as the oracle (R19).
__device__ __forceinline__ float lm_query(const LmDev& lm, int s, int w, int& next) {
    float acc = 0.0f;
    while (s != 0) {
        const int4 h = __ldg(&lm.st_hdr[s]);
        int lo = h.x, hi = h.x + h.y;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if ((int)__ldg(&lm.arc_tok[mid]) < w) lo = mid + 1; else hi = mid;
        }
        if (lo < h.x + h.y && (int)__ldg(&lm.arc_tok[lo]) == w) {
            const int2 v = __ldg(&lm.arc_val[lo]);
            next = v.y;
            return __fadd_rn(acc, __int_as_float(v.x));
        }
        acc = __fadd_rn(acc, __int_as_float(h.w));
        s = h.z;
    }
    next = __ldg(&lm.uni_next[w]);
    return __fadd_rn(acc, __ldg(&lm.uni_lp[w]));
}

struct Shared {
    float* ring;
    // current slot state
    float* acc; int* last; uint64_t* hash; int* lms; int* bts; uint8_t* anc; float* ubv; float* uba;
    // next slot state
    float* acc2; int* last2; uint64_t* hash2; int* lms2; int* bts2; uint8_t* anc2;
    // candidate buffer + selection
    uint64_t* ckey; int* clm; int* cbt;
    uint64_t* skey; int* slm; int* sbt;
    uint16_t* toks;
    int* alive_idx;
    uint32_t* hist;
    int* endslot;
};

struct Scalars {
    int nbuf, m, nalive, nsel, u;
    float thr;
    uint64_t kth;
    uint32_t prefix_found;
    float red_f[32];
    uint64_t red_k[32];
    int red_i[32];
};

template <int NT>
__device__ __forceinline__ float block_max(float v, Scalars& sc) {
    constexpr int NW = NT / 32;
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (NW == 1) return v;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sc.red_f[wid] = v;
    __syncthreads();
    float r = sc.red_f[0];
#pragma unroll
    for (int i = 1; i < NW; ++i) r = fmaxf(r, sc.red_f[i]);
    return r;
}

template <int NT>
__device__ __forceinline__ uint64_t block_max_u64(uint64_t v, Scalars& sc) {
    constexpr int NW = NT / 32;
    for (int o = 16; o; o >>= 1) {
        uint64_t x = __shfl_xor_sync(0xffffffffu, v, o);
        v = x > v ? x : v;
    }
    if (NW == 1) return v;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) sc.red_k[wid] = v;
    __syncthreads();
    uint64_t r = sc.red_k[0];
#pragma unroll
    for (int i = 1; i < NW; ++i) r = sc.red_k[i] > r ? sc.red_k[i] : r;
    return r;
}

// exclusive prefix over the block of per-thread counts; returns the offset, total in *tot
template <int NT>
__device__ __forceinline__ int block_exscan(int v, int* tot, Scalars& sc) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    __syncthreads();
    if (lane == 31) sc.red_i[wid] = x;
    __syncthreads();
    int base = 0, all = 0;
#pragma unroll
    for (int i = 0; i < NW; ++i) {
        if (i < wid) base += sc.red_i[i];
        all += sc.red_i[i];
    }
    *tot = all;
    return base + x - v;
}

// Radix select over n unique 64-bit keys in smem: returns the key kth such that exactly K keys
// are >= kth (n > K). MSB-first 8-bit digits; stops as soon as the boundary bin is exact.
template <int NT>
__device__ uint64_t radix_kth(const uint64_t* keys, int n, int K, Shared& sm, Scalars& sc) {
    uint64_t prefix = 0, mask = 0;
    int remaining = K;
    for (int shift = 56; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += NT) sm.hist[i] = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += NT) {
            const uint64_t k = keys[i];
            if ((k & mask) == prefix) atomicAdd(&sm.hist[(k >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (threadIdx.x < 32) {
            // lane l owns bins [248-8l .. 255-8l] (descending digits)
            const int lane = threadIdx.x;
            uint32_t c[8];
            uint32_t s = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) { c[j] = sm.hist[255 - 8 * lane - j]; s += c[j]; }
            uint32_t incl = s;
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            uint32_t above = incl - s;  // keys in strictly higher digits than this lane's bins
            if (above < (uint32_t)remaining && (uint32_t)remaining <= incl) {
                uint32_t a = above;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (a < (uint32_t)remaining && (uint32_t)remaining <= a + c[j]) {
                        const uint32_t d = 255 - 8 * lane - j;
                        sc.kth = (uint64_t)d;
                        sc.red_i[0] = (int)((uint32_t)remaining - a);   // still needed inside bin d
                        sc.red_i[1] = (int)c[j];                        // keys in bin d
                    }
                    a += c[j];
                }
            }
        }
        __syncthreads();
        const uint64_t d = sc.kth;
        const int need = sc.red_i[0], inbin = sc.red_i[1];
        __syncthreads();
        prefix |= d << shift;
        mask |= 255ull << shift;
        remaining = need;
        if (need == inbin) return prefix;  // every key with this prefix is in: threshold = prefix
    }
    return prefix;  // unique keys: the last digit pins the K-th key exactly
}

// Move the keys >= kth (exactly K of them) from the candidate buffer into the selection arrays.
template <int NT>
__device__ void gather_selected(int n, uint64_t kth, Shared& sm, Scalars& sc) {
    if (threadIdx.x == 0) sc.nsel = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += NT) {
        const uint64_t k = sm.ckey[i];
        if (k >= kth) {
            const int j = atomicAdd(&sc.nsel, 1);
            sm.skey[j] = k; sm.slm[j] = sm.clm[i]; sm.sbt[j] = sm.cbt[i];
        }
    }
    __syncthreads();
}

template <int NT>
__global__ void __launch_bounds__(NT) ctc_beam_kernel(const DecodeParams p, const int ring_rows, const int cap) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ Scalars sc;
    const int tid = threadIdx.x;
    const int K = p.K, Vp1 = p.Vp1, blank = Vp1 - 1;
    const int VP = (Vp1 + 3) & ~3;
    const int R = ring_rows;

    // ---- carve dynamic shared memory
    Shared sm;
    {
        unsigned char* q = smem_raw;
        auto take = [&](size_t bytes) { unsigned char* r = q; q += (bytes + 15) & ~size_t(15); return r; };
        sm.ring = (float*)take(sizeof(float) * (size_t)R * VP);
        sm.acc = (float*)take(4 * K); sm.last = (int*)take(4 * K); sm.hash = (uint64_t*)take(8 * K);
        sm.lms = (int*)take(4 * K); sm.bts = (int*)take(4 * K); sm.anc = (uint8_t*)take(K);
        sm.ubv = (float*)take(4 * K); sm.uba = (float*)take(4 * K);
        sm.acc2 = (float*)take(4 * K); sm.last2 = (int*)take(4 * K); sm.hash2 = (uint64_t*)take(8 * K);
        sm.lms2 = (int*)take(4 * K); sm.bts2 = (int*)take(4 * K); sm.anc2 = (uint8_t*)take(K);
        sm.ckey = (uint64_t*)take(8 * (size_t)cap); sm.clm = (int*)take(4 * (size_t)cap); sm.cbt = (int*)take(4 * (size_t)cap);
        sm.skey = (uint64_t*)take(8 * K); sm.slm = (int*)take(4 * K); sm.sbt = (int*)take(4 * K);
        sm.toks = (uint16_t*)take(2 * (size_t)Vp1);
        sm.alive_idx = (int*)take(4 * K);
        sm.hist = (uint32_t*)take(4 * 256);
        sm.endslot = (int*)take(4 * (size_t)p.nch);
    }
    const bool lm_on = p.use_lm != 0, bt_on = p.use_bt != 0;
    const bool ub_inf = (lm_on && p.alpha_lm < 0.0f) || (bt_on && p.alpha_bt < 0.0f);

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

        // ------------------------------------------------------------ init (Alg. 1)
        for (int k = tid; k < K; k += NT) {
            sm.acc[k] = k == 0 ? 0.0f : kNeg;   // acc_scores[:,0] = 0, else -inf
            sm.last[k] = blank;                  // R6
            sm.hash[k] = 0ull;
            sm.lms[k] = p.lm.start;              // LM(<SOS>)
            sm.bts[k] = 0;                       // BT(<0>) = root
            sm.anc[k] = 0;
            float ub = p.beta, ua = fabsf(p.beta);
            if (lm_on) { float x = p.alpha_lm * __ldg(&p.lm.ub[p.lm.start]); ub += x; ua += fabsf(x); }
            sm.ubv[k] = ub_inf ? INFINITY : ub;
            sm.uba[k] = ua;
        }
        // prologue: prefetch rows 0..R-2
        for (int r = 0; r < R - 1; ++r) {
            if (r < L) {
                const float* src = Db + (int64_t)r * p.stride_t;
                float* dst = sm.ring + (size_t)(r % R) * VP;
                if ((((uintptr_t)src) & 15) == 0) {
                    const int n4 = Vp1 >> 2;
                    for (int i = tid; i < n4; i += NT) cp_async16(dst + 4 * i, src + 4 * i);
                    for (int i = 4 * n4 + tid; i < Vp1; i += NT) cp_async4(dst + i, src + i);
                } else {
                    for (int i = tid; i < Vp1; i += NT) cp_async4(dst + i, src + i);
                }
            }
            cp_commit();
        }

        for (int t = 0; t < L; ++t) {
            // ---------------------------------------------------- stage row t (issue row t+R-1)
            {
                const int r = t + R - 1;
                if (r < L) {
                    const float* src = Db + (int64_t)r * p.stride_t;
                    float* dst = sm.ring + (size_t)(r % R) * VP;
                    if ((((uintptr_t)src) & 15) == 0) {
                        const int n4 = Vp1 >> 2;
                        for (int i = tid; i < n4; i += NT) cp_async16(dst + 4 * i, src + 4 * i);
                        for (int i = 4 * n4 + tid; i < Vp1; i += NT) cp_async4(dst + i, src + i);
                    } else {
                        for (int i = tid; i < Vp1; i += NT) cp_async4(dst + i, src + i);
                    }
                }
                cp_commit();
            }
            if (R == 4) cp_wait<3>(); else cp_wait<1>();
            if (tid == 0) { sc.nbuf = 0; sc.m = 0; }
            __syncthreads();
            const float* row = sm.ring + (size_t)(t % R) * VP;

            // ---------------------------------------------------- phase 1: exact blank / repeat candidates
            float a = kNeg, sbk = kNeg, srk = kNeg, ubk = kNeg;
            int lk = blank;
            bool al = false;
            if (tid < K) {
                a = sm.acc[tid];
                al = a > kNeg;
                lk = sm.last[tid];
                if (al) {
                    sbk = __fadd_rn(a, row[blank]);            // blank: no β / fusion
                    if (lk != blank) srk = __fadd_rn(a, row[lk]); // repeat: no β / fusion
                    ubk = sm.ubv[tid];
                }
            }
            {
                // alive list (slot order)
                const unsigned bal = __ballot_sync(0xffffffffu, al);
                int tot;
                const int off = block_exscan<NT>(al ? 1 : 0, &tot, sc);
                if (al) sm.alive_idx[off] = tid;
                (void)bal;
                if (tid == 0) sc.nalive = tot;
            }
            const float mx0 = block_max<NT>(fmaxf(sbk, srk), sc);
            const float accmax = block_max<NT>(a, sc);
            const float ubvmax = block_max<NT>(ubk, sc);
            const float tau0 = __fsub_rn(mx0, p.theta);   // lower bound of fl(max - θ)
            if (tid == 0) sc.thr = tau0;
            __syncthreads();
            if (al) {
                if (sbk > kNeg && sbk >= tau0) {
                    const int j = atomicAdd(&sc.nbuf, 1);
                    sm.ckey[j] = make_key(sbk, (uint32_t)(tid * Vp1 + blank));
                    sm.clm[j] = sm.lms[tid]; sm.cbt[j] = sm.bts[tid];
                }
                if (srk > kNeg && srk >= tau0) {
                    const int j = atomicAdd(&sc.nbuf, 1);
                    sm.ckey[j] = make_key(srk, (uint32_t)(tid * Vp1 + lk));
                    sm.clm[j] = sm.lms[tid]; sm.cbt[j] = sm.bts[tid];
                }
            }
            // ---------------------------------------------------- phase 2: frame token filter
            // any non-rb candidate that can reach tau0 has D[w] >= tau0 - accmax - ubvmax - margin
            if (mx0 > kNeg) {
                const float mg = 1e-4f * (1.0f + fabsf(tau0) + fabsf(accmax) + fabsf(ubvmax));
                const float dthr = __fsub_rn(__fsub_rn(__fsub_rn(tau0, accmax), ubvmax), mg);
                for (int w0 = 0; w0 < Vp1; w0 += NT) {
                    const int w = w0 + tid;
                    const bool hit = w < Vp1 && w != blank && row[w] >= dthr;
                    const unsigned bal = __ballot_sync(0xffffffffu, hit);
                    if (bal) {
                        int base = 0;
                        if ((tid & 31) == 0) base = atomicAdd(&sc.m, __popc(bal));
                        base = __shfl_sync(0xffffffffu, base, 0);
                        if (hit) sm.toks[base + __popc(bal & ((1u << (tid & 31)) - 1u))] = (uint16_t)w;
                    }
                }
            }
            __syncthreads();
            // ---------------------------------------------------- phase 3: exact non-rb candidates
            {
                const int m = sc.m;
                const int npairs = sc.nalive * m;
                for (int base = 0; base < npairs; base += NT) {
                    if (sc.nbuf > cap - NT) {
                        // buffer full: keep the top K, raise the threshold (threshold algorithm)
                        const int n = sc.nbuf;
                        const uint64_t kth = radix_kth<NT>(sm.ckey, n, K, sm, sc);
                        gather_selected<NT>(n, kth, sm, sc);
                        for (int i = tid; i < K; i += NT) { sm.ckey[i] = sm.skey[i]; sm.clm[i] = sm.slm[i]; sm.cbt[i] = sm.sbt[i]; }
                        if (tid == 0) { sc.nbuf = K; sc.thr = fmaxf(sc.thr, score_of(kth)); }
                        __syncthreads();
                    }
                    const float thr = sc.thr;
                    const int pi = base + tid;
                    if (pi < npairs) {
                        const int k = sm.alive_idx[pi / m];
                        const int w = sm.toks[pi % m];
                        if (w != sm.last[k]) {
                            const float ak = sm.acc[k];
                            const float s0 = __fadd_rn(ak, row[w]);
                            const float uv = sm.ubv[k];
                            const float bound = __fadd_rn(s0, uv) + 1e-5f * (1.0f + fabsf(s0) + sm.uba[k]);
                            if (bound >= thr) {
                                float s = __fadd_rn(s0, p.beta);
                                int ln = sm.lms[k], bn = sm.bts[k];
                                if (lm_on) {
                                    const float lp = lm_query(p.lm, ln, w, ln);
                                    s = __fmaf_rn(p.alpha_lm, lp, s);
                                }
                                if (bt_on) {
                                    const int2 e = __ldg(&p.bt.tab[(size_t)bn * p.bt.V + w]);
                                    bn = e.x;
                                    s = __fmaf_rn(p.alpha_bt, __int_as_float(e.y), s);
                                }
                                if (s > kNeg && s >= thr) {
                                    const int j = atomicAdd(&sc.nbuf, 1);
                                    sm.ckey[j] = make_key(s, (uint32_t)(k * Vp1 + w));
                                    sm.clm[j] = ln; sm.cbt[j] = bn;
                                }
                            }
                        }
                    }
                    __syncthreads();
                }
            }
            // ---------------------------------------------------- phase 4: flat TopK + θ-prune
            const int n = sc.nbuf;
            const uint64_t* kk;
            const int* kl;
            const int* kb;
            int nsel;
            if (n > NT) {
                const uint64_t kth = radix_kth<NT>(sm.ckey, n, K, sm, sc);
                gather_selected<NT>(n, kth, sm, sc);
                kk = sm.skey; kl = sm.slm; kb = sm.sbt; nsel = K;
            } else {
                kk = sm.ckey; kl = sm.clm; kb = sm.cbt; nsel = n;
            }
            // rank sort (keys are unique); entry -> slot rank when rank < K
            uint64_t myk = 0;
            int rank = 0, myl = 0, myb = 0;
            if (tid < nsel) {
                myk = kk[tid]; myl = kl[tid]; myb = kb[tid];
                for (int j = 0; j < nsel; ++j) rank += kk[j] > myk ? 1 : 0;
            }
            __syncthreads();
            if (tid < nsel && rank < K) { sm.skey[rank] = myk; sm.slm[rank] = myl; sm.sbt[rank] = myb; }
            __syncthreads();
            const int nkeep = nsel < K ? nsel : K;
            const float mx = nkeep > 0 ? score_of(sm.skey[0]) : kNeg;   // max_score
            const float tau = __fsub_rn(mx, p.theta);
            // ---------------------------------------------------- phase 5: beams.update
            const int64_t bpo = ((int64_t)b * p.T + t) * K;
            if (tid < K) {
                const int i = tid;
                bool live = false;
                if (i < nkeep) {
                    const uint64_t key = sm.skey[i];
                    const float s = score_of(key);
                    if (s >= tau) {
                        live = true;
                        const uint32_t f = flat_of(key);
                        const int par = (int)(f / (uint32_t)Vp1), w = (int)(f % (uint32_t)Vp1);
                        const int pl = sm.last[par];
                        const bool emit = w != blank && w != pl;
                        sm.acc2[i] = s;
                        sm.last2[i] = w;
                        sm.hash2[i] = emit ? hash_extend(sm.hash[par], w) : sm.hash[par];
                        sm.lms2[i] = sm.slm[i];   // rb candidates carry the parent's states
                        sm.bts2[i] = sm.sbt[i];
                        sm.anc2[i] = (t % kChunk == 0) ? (uint8_t)par : sm.anc[par];
                        p.bp_parent[bpo + i] = (uint8_t)par;
                        p.bp_label[bpo + i] = (uint16_t)w;
                    }
                }
                if (!live) {
                    sm.acc2[i] = kNeg;
                    sm.last2[i] = blank;
                    sm.hash2[i] = 0ull;
                    sm.lms2[i] = 0; sm.bts2[i] = 0; sm.anc2[i] = 0;
                    p.bp_parent[bpo + i] = 0xff;
                    p.bp_label[bpo + i] = 0xffff;
                }
            }
            __syncthreads();
            // ---------------------------------------------------- phase 6: RecombineHypotheses
            if (tid < K) {
                const int i = tid;
                float s = sm.acc2[i];
                if (s > kNeg) {
                    const uint64_t h = sm.hash2[i];
                    const int l = sm.last2[i];
                    bool dead = false;
                    for (int j = 0; j < i; ++j)
                        if (sm.acc2[j] > kNeg && sm.hash2[j] == h && sm.last2[j] == l) { dead = true; break; }
                    if (dead) {
                        s = kNeg;
                    } else {
                        // slots are in (score desc, flat asc) order, so the group order is slot order
                        float sum = 0.0f;
                        bool any = false;
                        for (int j = i + 1; j < K; ++j) {
                            const float sj = sm.acc2[j];
                            if (sj > kNeg && sm.hash2[j] == h && sm.last2[j] == l) {
                                any = true;
                                if (p.merge_mode == 0) sum = __fadd_rn(sum, (float)exp((double)__fsub_rn(sj, s)));
                            }
                        }
                        if (any && p.merge_mode == 0) s = __fadd_rn(s, (float)log1p((double)sum));
                    }
                }
                sm.acc[i] = s;
                sm.last[i] = sm.last2[i];
                sm.hash[i] = sm.hash2[i];
                sm.lms[i] = sm.lms2[i];
                sm.bts[i] = sm.bts2[i];
                sm.anc[i] = sm.anc2[i];
                if (s > kNeg) {
                    float ub = p.beta, ua = fabsf(p.beta);
                    if (lm_on) { float x = p.alpha_lm * __ldg(&p.lm.ub[sm.lms2[i]]); ub += x; ua += fabsf(x); }
                    if (bt_on) { float x = p.alpha_bt * __ldg(&p.bt.maxd[sm.bts2[i]]); ub += x; ua += fabsf(x); }
                    sm.ubv[i] = ub_inf ? INFINITY : ub;
                    sm.uba[i] = ua;
                }
                if ((t % kChunk) == kChunk - 1 || t == L - 1)
                    p.chunk_anc[((int64_t)b * p.nch + t / kChunk) * K + i] = sm.anc2[i];
            }
            __syncthreads();
        }
        cp_wait<0>();

        // ------------------------------------------------------------ EOS + final merge (R15)
        if (tid < K) {
            float s = sm.acc[tid];
            if (s > kNeg) {
                if (lm_on) s = __fmaf_rn(p.alpha_lm, __ldg(&p.lm.eos[sm.lms[tid]]), s);
                if (bt_on && p.retract) s = __fmaf_rn(-p.alpha_bt, __ldg(&p.bt.U[sm.bts[tid]]), s);
            }
            sm.acc2[tid] = s;
        }
        __syncthreads();
        uint64_t bestkey = 0;
        if (tid < K) {
            const int i = tid;
            float s = sm.acc2[i];
            if (s > kNeg) {
                const uint64_t h = sm.hash[i];
                bool dead = false;
                for (int j = 0; j < K; ++j) {
                    const float sj = sm.acc2[j];
                    if (j != i && sj > kNeg && sm.hash[j] == h && (sj > s || (sj == s && j < i))) { dead = true; break; }
                }
                if (!dead) {
                    // other members in (score desc, slot asc) order
                    float sum = 0.0f;
                    bool any = false;
                    float prev_s = INFINITY;
                    int prev_j = -1;
                    for (;;) {
                        int bj = -1;
                        float bs = kNeg;
                        for (int j = 0; j < K; ++j) {
                            const float sj = sm.acc2[j];
                            if (j == i || !(sj > kNeg) || sm.hash[j] != h) continue;
                            const bool after_prev = sj < prev_s || (sj == prev_s && j > prev_j);
                            if (!after_prev) continue;
                            if (bj < 0 || sj > bs || (sj == bs && j < bj)) { bj = j; bs = sj; }
                        }
                        if (bj < 0) break;
                        any = true;
                        if (p.merge_mode == 0) sum = __fadd_rn(sum, (float)exp((double)__fsub_rn(bs, s)));
                        prev_s = bs; prev_j = bj;
                    }
                    if (any && p.merge_mode == 0) s = __fadd_rn(s, (float)log1p((double)sum));
                    bestkey = ((uint64_t)ord_of(s) << 32) | (uint64_t)(0xffffffffu - (uint32_t)i);
                }
            }
        }
        bestkey = block_max_u64<NT>(bestkey, sc);
        const bool has_best = bestkey != 0ull;
        const int best = has_best ? (int)(0xffffffffu - (uint32_t)bestkey) : -1;
        const float best_score = has_best ? score_of(bestkey) : kNeg;

        // ------------------------------------------------------------ backtrace ("reconstruction on demand")
        int32_t* align = (p.out_align ? p.out_align : p.align_ws) + (int64_t)b * p.T;
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
        int off = block_exscan<NT>(cnt, &ntok, sc);
        int32_t* otok = p.out_tokens + (int64_t)b * p.T;
        int32_t* ots = p.out_ts ? p.out_ts + (int64_t)b * p.T : nullptr;
        if (has_best)
            for (int t = t0; t < t1; ++t) {
                const int at = align[t], ap = t ? align[t - 1] : blank;
                if (at != blank && at != ap) {
                    otok[off] = at;
                    if (ots) ots[off] = t;
                    ++off;
                }
            }
        for (int i = ntok + tid; i < p.T; i += NT) { otok[i] = -1; if (ots) ots[i] = -1; }
        if (p.out_align)
            for (int i = (has_best ? L : 0) + tid; i < p.T; i += NT) p.out_align[(int64_t)b * p.T + i] = -1;
        if (tid == 0) {
            p.out_num[b] = ntok;
            p.out_scores[b] = best_score;
        }
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

size_t smem_bytes(int K, int Vp1, int R, int cap, int nch) {
    const int VP = (Vp1 + 3) & ~3;
    auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
    size_t s = al(sizeof(float) * (size_t)R * VP);
    s += 2 * (al(4 * K) + al(4 * K) + al(8 * K) + al(4 * K) + al(4 * K) + al(K)) + 2 * al(4 * K);
    s += al(8 * (size_t)cap) + 2 * al(4 * (size_t)cap);
    s += al(8 * K) + 2 * al(4 * K);
    s += al(2 * (size_t)Vp1) + al(4 * K) + al(4 * 256) + al(4 * (size_t)nch);
    return s;
}

template <int NT>
int launch_nt(const DecodeParams& p, cudaStream_t st, void* ev0, void* ev1, std::string& err) {
    const int VP = (p.Vp1 + 3) & ~3;
    const int R = VP <= 2048 ? 4 : 2;
    const int cap = 8 * NT;
    const size_t sm = smem_bytes(p.K, p.Vp1, R, cap, p.nch);
    if (sm > 200 * 1024) { err = "shared memory requirement too large (V+1 or T)"; return 2; }
    cudaError_t e = cudaFuncSetAttribute(ctc_beam_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) { err = cudaGetErrorString(e); return 1; }
    int dev = 0, nsm = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ctc_beam_kernel<NT>, NT, sm);
    if (e != cudaSuccess || occ < 1) { err = "occupancy query failed"; return 1; }
    const int grid = std::min(p.B, nsm * occ);
    if (ev0 && ev1) cudaEventRecord((cudaEvent_t)ev0, st);
    ctc_beam_kernel<NT><<<grid, NT, sm, st>>>(p, R, cap);
    e = cudaGetLastError();
    if (e == cudaSuccess && ev0 && ev1) cudaEventRecord((cudaEvent_t)ev1, st);
    if (e != cudaSuccess) { err = cudaGetErrorString(e); return 1; }
    return 0;
}

}  // namespace

int launch_decode(const DecodeParams& p, void* stream, void* ev0, void* ev1, std::string& err) {
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(p.flags, 0, 2 * sizeof(uint32_t), st);
    if (e != cudaSuccess) { err = cudaGetErrorString(e); return 1; }
    if (p.B == 0) return 0;
    order_kernel<<<(p.B + 255) / 256, 256, 0, st>>>(p.lengths, p.B, p.T, p.order, p.len_c, p.flags, p.B <= 16384);
    e = cudaGetLastError();
    if (e != cudaSuccess) { err = cudaGetErrorString(e); return 1; }
    const int nt = p.K <= 32 ? 32 : p.K <= 64 ? 64 : p.K <= 128 ? 128 : 256;
    switch (nt) {
        case 32: return launch_nt<32>(p, st, ev0, ev1, err);
        case 64: return launch_nt<64>(p, st, ev0, ev1, err);
        case 128: return launch_nt<128>(p, st, ev0, ev1, err);
        default: return launch_nt<256>(p, st, ev0, ev1, err);
    }
}

}  // namespace flexctc
