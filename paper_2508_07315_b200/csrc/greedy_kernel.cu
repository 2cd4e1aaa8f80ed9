// Greedy CTC decoding (beam K = 1) with optional N-gram LM / phrase-boosting fusion.
//
// the Table II greedy rows and "NGPU-LM ... during greedy
// decoding". K = 1 is Algorithm 1 with a beam of one hypothesis: per frame it
// takes the best candidate of Eq. (1) over all V' tokens -- blank and the repeat without
// β / fusion terms -- ties to the lower token index (reading R9); the θ-prune
// and the recombination are no-ops for one hypothesis; EOS adds
// α_LM·LM.Final. The outputs are those of the beam kernel at K = 1 (and of the
// oracle), from two much shorter paths:
//
//  * plain (β = 0, no LM, no boosting: c2's greedy leg). Every candidate is fl(acc + D[t, w]),
//    so the frame's choice is the row argmax whatever acc is -- except when rounding makes
//    fl(acc + d2) == fl(acc + d1) for a runner-up d2 < d1 (then the lowest tied index wins).
//    frame_summary_kernel streams D once at HBM rate (one warp per row, 16-B loads, every row of
//    the batch spread over the whole GPU) and writes {d1, d2, D[blank], w1} per frame;
//    greedy_chain_kernel (one warp per utterance) replays the fp32 chain acc = fl(acc + d1) in
//    frame order (bit-identical to the sequential definition), rescans the rare rows where the
//    runner-up ties after rounding, and collapses the labels to tokens + timestamps (R20).
//  * fused (β != 0 or LM or boosting): the hypothesis' LM / boost state couples the frames, so
//    one warp per utterance runs the frame loop (4 utterances per CTA, LPT work queue) after the
//    same summary pass. Rows stream into a per-warp ring 7 frames ahead, one TMA bulk copy
//    (cp.async.bulk, completion on an mbarrier) per row issued by one lane; per frame: the
//    summary gives the best non-blank tokens without a scan, exact blank and repeat
//    candidates, the exact score of the best non-repeat token, then only tokens whose
//    bound D[w] + ub(state) can reach the running best are scored (LM arc query + boost table
//    load, 32 lanes in parallel); the winner advances the LM / boost state on emission (R5, R18).
// Score arithmetic: __fadd_rn / __fmaf_rn in the canonical order of reading R19, as the beam
// kernel.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <string>

#include "device_common.cuh"
#include "flexctc_internal.h"

namespace flexctc {
namespace {

using namespace dev;

// ---------------------------------------------------------------------------------- plain path

constexpr uint32_t kNoTok = 0xffffu;

// Frame summary {d1, d2, D[blank], w1}: the best non-blank value d1 and its lowest index w1
// (kNoTok = none), an upper bound d2 of the best non-blank value at any other index (exact
// unless a value repeats or a NaN is present: the consumers only use it conservatively), and the
// blank value (NaN -> -inf: never a candidate, as in the beam kernel).
// The only O(B·T·V') pass of the greedy paths, bandwidth-bound: one CTA per 8 consecutive frames
// of one utterance (one row per warp), rows t >= L_b skipped before any load, every 16-B load of
// a row (8 per lane at V' = 1025) issued before the first compare, evict-first loads (D is read
// once). Per element: 3 FMNMX for the running (max, second) and 2 ops for the argmax pass.
constexpr int kSumRows = 8;
__device__ __forceinline__ void max2(float x, float& m1, float& m2) {
    m2 = fmaxf(m2, fminf(m1, x));
    m1 = fmaxf(m1, x);
}
__global__ void __launch_bounds__(32 * kSumRows, 4) frame_summary_kernel(const float* __restrict__ D, int64_t sb,
                                                                        int64_t stt,
                                                                        const int32_t* __restrict__ lengths, int B,
                                                                        int T, int Vp1, float4* __restrict__ summ) {
    const int lane = threadIdx.x & 31;
    const int blank = Vp1 - 1;
    const int nchunk = (T + kSumRows - 1) / kSumRows;
    const int b = blockIdx.x / nchunk;
    const int t = (blockIdx.x - b * nchunk) * kSumRows + (threadIdx.x >> 5);
    const int L = min(max(__ldg(&lengths[b]), 0), T);
    if (t >= L) return;
    const float* row = D + (int64_t)b * sb + (int64_t)t * stt;
    const int off = row_off(row);
    const int h = min((4 - off) & 3, Vp1);
    const int n4 = (Vp1 - h) >> 2;
    const int tl = h + 4 * n4;
    const float4* body = (const float4*)(row + h);
    // head / tail scalars (< 4 each) and the blank value, then the body in batches of 8 x 16 B
    float hv = kNeg, tv = kNeg, db = kNeg;
    if (lane < h) hv = __ldcs(row + lane);
    if (tl + lane < Vp1) tv = __ldcs(row + tl + lane);
    if (lane == 0) db = __ldcs(row + blank);
    if (lane >= h || lane >= blank) hv = kNeg;
    if (tl + lane >= blank) tv = kNeg;
    float m1 = kNeg, m2 = kNeg, w1v = kNeg;  // w1: lowest index of value w1v in folded batches
    int w1 = 0x7fffffff;
    max2(hv, m1, m2);
    max2(tv, m1, m2);
    float4 v[8];
    for (int i0 = 0; i0 < n4; i0 += 256) {  // one batch at V' <= 4100
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int i = i0 + lane + 32 * j;
            v[j] = i < n4 ? __ldcs(&body[i]) : make_float4(kNeg, kNeg, kNeg, kNeg);
            const int w = h + 4 * i;
            if (w + 3 >= blank) {  // the blank (or nothing) sits in this vector: mask it out
                if (w >= blank) v[j].x = kNeg;
                if (w + 1 >= blank) v[j].y = kNeg;
                if (w + 2 >= blank) v[j].z = kNeg;
                v[j].w = kNeg;
            }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) { max2(v[j].x, m1, m2); max2(v[j].y, m1, m2); max2(v[j].z, m1, m2); max2(v[j].w, m1, m2); }
        if (i0 + 256 < n4) {  // V' > 4100: fold this batch's argmax candidates now (rare shapes)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (m1 > w1v) { w1v = m1; w1 = 0x7fffffff; }
                const int w = h + 4 * (i0 + lane + 32 * j);
                if (v[j].x == m1) w1 = min(w1, w);
                if (v[j].y == m1) w1 = min(w1, w + 1);
                if (v[j].z == m1) w1 = min(w1, w + 2);
                if (v[j].w == m1) w1 = min(w1, w + 3);
            }
        }
    }
    // warp (max, second): the second is max(every second, every max but the largest)
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const float a1 = __shfl_xor_sync(0xffffffffu, m1, o), a2 = __shfl_xor_sync(0xffffffffu, m2, o);
        m2 = fmaxf(fmaxf(m2, a2), fminf(m1, a1));
        m1 = fmaxf(m1, a1);
    }
    // lowest index holding d1 = m1 (exact fp32 equality with the loaded values)
    int wl = 0x7fffffff;
    if (m1 > kNeg) {
        if (hv == m1) wl = lane;
        const int tail_n = n4 > 256 ? ((n4 - 1) & ~255) : 0;  // start of the last batch still in v[]
#pragma unroll
        for (int j = 7; j >= 0; --j) {
            const int w = h + 4 * (tail_n + lane + 32 * j);
            if (v[j].w == m1) wl = w + 3;
            if (v[j].z == m1) wl = w + 2;
            if (v[j].y == m1) wl = w + 1;
            if (v[j].x == m1) wl = w;
        }
        if (tv == m1) wl = min(wl, tl + lane);
        if (w1v == m1) wl = min(wl, w1);
#pragma unroll
        for (int o = 16; o; o >>= 1) wl = min(wl, __shfl_xor_sync(0xffffffffu, wl, o));
    }
    if (lane == 0) {
        const uint32_t wi = m1 > kNeg ? (uint32_t)wl : kNoTok;
        summ[(int64_t)b * T + t] = make_float4(m1, m2, db > kNeg ? db : kNeg, __uint_as_float(wi));
    }
}

// Finish one utterance: tokens / timestamps padding, alignment padding, count and score.
// dead = no finite candidate at some frame (the hypothesis died, as in the beam kernel).
__device__ void finish_utterance(const DecodeParams& p, int b, int L, int n, float score, bool dead, int lane) {
    int32_t* otok = p.out_tokens + (int64_t)b * p.T;
    int32_t* ots = p.out_ts ? p.out_ts + (int64_t)b * p.T : nullptr;
    const int n0 = dead ? 0 : n;
    for (int i = n0 + lane; i < p.T; i += 32) { otok[i] = -1; if (ots) ots[i] = -1; }
    if (p.out_align)
        for (int i = (dead ? 0 : L) + lane; i < p.T; i += 32) p.out_align[(int64_t)b * p.T + i] = -1;
    if (lane == 0) {
        p.out_num[b] = n0;
        p.out_scores[b] = dead ? kNeg : score;
    }
}

// Collapse labels lab[0..nt) of frames t0.. (prev = label of frame t0-1) into tokens at
// out position n (R20: a token is emitted at t iff a_t != blank and a_t != a_{t-1}).
__device__ __forceinline__ int collapse_tile(const DecodeParams& p, int b, const int* lab, int nt, int t0, int prev,
                                             int n, int blank, int lane) {
    int32_t* otok = p.out_tokens + (int64_t)b * p.T;
    int32_t* ots = p.out_ts ? p.out_ts + (int64_t)b * p.T : nullptr;
    for (int i0 = 0; i0 < nt; i0 += 32) {
        const int i = i0 + lane;
        const int a = i < nt ? lab[i] : blank;
        const int ap = i == 0 ? prev : (i < nt ? lab[i - 1] : blank);
        const bool em = i < nt && a != blank && a != ap;
        const unsigned bal = __ballot_sync(0xffffffffu, em);
        if (em) {
            const int q = n + __popc(bal & ((1u << lane) - 1u));
            otok[q] = a;
            if (ots) ots[q] = t0 + i;
        }
        if (p.out_align && i < nt) p.out_align[(int64_t)b * p.T + t0 + i] = a;
        n += __popc(bal);
    }
    return n;
}

constexpr int kTile = 256;  // frames per chain tile

// One warp per utterance: the fp32 score chain in frame order, tie resolution, collapse.
// Clamps lengths and raises the length flags (the plain path runs no order_kernel).
__global__ void __launch_bounds__(128) greedy_chain_kernel(const DecodeParams p) {
    __shared__ float s_d1[4][kTile], s_d2[4][kTile], s_acc[4][kTile];
    __shared__ int s_lab[4][kTile];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int b = blockIdx.x * 4 + wid;
    if (b >= p.B) return;
    const int blank = p.Vp1 - 1;
    int L = p.lengths[b];
    if (lane == 0) {
        uint32_t fl = 0;
        if (L > p.T) fl |= FLEXCTC_FLAG_LENGTH_CLAMPED_HIGH;
        if (L < 0) fl |= FLEXCTC_FLAG_LENGTH_CLAMPED_LOW;
        if (fl) atomicOr(p.flags, fl);
    }
    L = min(max(L, 0), p.T);
    float* d1 = s_d1[wid];
    float* d2 = s_d2[wid];
    float* ap = s_acc[wid];
    int* lab = s_lab[wid];
    const float4* summ = p.greedy_sum + (int64_t)b * p.T;
    float acc = 0.0f;  // acc_scores[:, 0] = 0
    bool dead = false;
    int n = 0, prev = blank;  // last label starts as blank (R6)
    int ties = 0;
    for (int t0 = 0; t0 < L && !dead; t0 += kTile) {
        const int nt = min(kTile, L - t0);
        // best candidate over all V' tokens (blank has the highest index: it wins only when
        // strictly above the best non-blank) and the runner-up value; all loads issued first
        float4 sv[kTile / 32];
#pragma unroll
        for (int k = 0; k < kTile / 32; ++k)
            if (32 * k + lane < nt) sv[k] = summ[t0 + 32 * k + lane];
#pragma unroll
        for (int k = 0; k < kTile / 32; ++k) {
            const int i = 32 * k + lane;
            if (i < nt) {
                const float4 s = sv[k];
                const uint32_t w1 = __float_as_uint(s.w) & 0xffffu;
                float bv = kNeg, rv = kNeg;
                int bw = -1;
                if (w1 != kNoTok && !(s.z > s.x)) { bv = s.x; bw = (int)w1; rv = fmaxf(s.y, s.z); }
                else if (s.z > kNeg) { bv = s.z; bw = blank; rv = w1 != kNoTok ? s.x : kNeg; }
                d1[i] = bv; lab[i] = bw; d2[i] = rv;
            }
        }
        __syncwarp();
        // the fp32 chain acc = fl(acc + d1) in frame order (lane 0): ap[i] = acc before frame i.
        // A frame without a finite candidate makes acc -inf for good (the hypothesis died).
        if (lane == 0) {
            int i = 0;
            for (; i + 8 <= nt; i += 8) {
                float x[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) x[k] = d1[i + k];
#pragma unroll
                for (int k = 0; k < 8; ++k) { ap[i + k] = acc; acc = __fadd_rn(acc, x[k]); }
            }
            for (; i < nt; ++i) { ap[i] = acc; acc = __fadd_rn(acc, d1[i]); }
        }
        __syncwarp();
        acc = __shfl_sync(0xffffffffu, acc, 0);
        if (!(acc > kNeg)) { dead = true; break; }
        // tie frames (runner-up equal after rounding): lowest w with fl(acc + D[w]) == target
        for (int i0 = 0; i0 < nt; i0 += 32) {
            const int i = i0 + lane;
            bool tie = false;
            if (i < nt) tie = d2[i] > kNeg && __fadd_rn(ap[i], d2[i]) == __fadd_rn(ap[i], d1[i]);
            unsigned tb = __ballot_sync(0xffffffffu, tie);
            ties += __popc(tb);
            while (tb) {
                const int q = i0 + __ffs(tb) - 1;
                tb &= tb - 1u;
                const float a = ap[q], target = __fadd_rn(a, d1[q]);
                const float* row = p.log_probs + (int64_t)b * p.stride_b + (int64_t)(t0 + q) * p.stride_t;
                int wmin = 0x7fffffff;
                for (int w = lane; w < p.Vp1; w += 32)
                    if (__fadd_rn(a, row[w]) == target) { wmin = min(wmin, w); break; }
#pragma unroll
                for (int o = 16; o; o >>= 1) wmin = min(wmin, __shfl_xor_sync(0xffffffffu, wmin, o));
                if (lane == 0) lab[q] = wmin;
            }
        }
        __syncwarp();
        n = collapse_tile(p, b, lab, nt, t0, prev, n, blank, lane);
        prev = lab[nt - 1];
        __syncwarp();
    }
    finish_utterance(p, b, L, n, acc, dead, lane);
    if (lane == 0) {
        atomicAdd(&p.stats[kFrames], (unsigned long long)L);
        if (ties) atomicAdd(&p.stats[kListed], (unsigned long long)ties);
    }
}

// ---------------------------------------------------------------------------------- fused path

constexpr int kGW = 4;     // utterances (warps) per CTA, at most (fewer when V' makes the ring large)
constexpr int kGRing = 8;  // frame rows in flight per warp, at most (covers HBM latency at ~300-cycle frames)

__host__ __device__ __forceinline__ size_t greedy_warp_smem(int Vp1, int RWS, int ring) {
    const int VP = (Vp1 + 3) & ~3;
    const size_t a = (((size_t)ring * (VP + 4) * 4 + (size_t)RWS * 4 + (size_t)Vp1 * 2 + 7) & ~size_t(7));
    return (a + 8 * (size_t)ring + 15) & ~size_t(15);
}

__device__ __forceinline__ float4 shfl4(float4 v, int src) {
    return make_float4(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src),
                       __shfl_sync(0xffffffffu, v.z, src), __shfl_sync(0xffffffffu, v.w, src));
}

template <int LMV>
__global__ void __launch_bounds__(32 * kGW) greedy_fused_kernel(const DecodeParams p, const int ringn /* 2, 4 or 8 */) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int Vp1 = p.Vp1, blank = Vp1 - 1, V = Vp1 - 1;
    const int VP = (Vp1 + 3) & ~3;
    const bool lm_on = p.use_lm != 0, bt_on = p.use_bt != 0;
    const int RWS = lm_on ? ((p.lm.RW + 3) & ~3) : 4;
    const bool ub_inf = (lm_on && p.alpha_lm < 0.0f) || (bt_on && p.alpha_bt < 0.0f);
    // layout: [warps] x {ring[ringn][VP + 4] f32, rec[RWS] i32, list[Vp1] u16, bar[ringn] u64},
    // then btroot[V] int2
    const size_t per_warp = greedy_warp_smem(Vp1, RWS, ringn);
    unsigned char* base = smem_raw + (size_t)wid * per_warp;
    float* ring = (float*)base;
    int* rec = (int*)(base + (size_t)ringn * (VP + 4) * 4);
    uint16_t* list = (uint16_t*)(base + (size_t)ringn * (VP + 4) * 4 + (size_t)RWS * 4);
    uint64_t* bar = (uint64_t*)(base + (((size_t)ringn * (VP + 4) * 4 + (size_t)RWS * 4 + (size_t)Vp1 * 2 + 7) & ~size_t(7)));
    int2* btroot = (int2*)(smem_raw + (size_t)(blockDim.x >> 5) * per_warp);
    if (bt_on)
        for (int w = threadIdx.x; w < V; w += blockDim.x) btroot[w] = __ldg(&p.bt.tab[w]);
    if (lane == 0) {
        for (int i = 0; i < ringn; ++i) mbar_init(&bar[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    uint32_t ph = 0;  // expected parity of each ring slot's next completion
    // the tensor's byte range: bulk copies never read outside it (overread: 16 B of slack after)
    const char* lo = (const char*)p.log_probs;
    const char* hi = lo + 4 * ((int64_t)(p.B - 1) * p.stride_b + (int64_t)(p.T - 1) * p.stride_t + Vp1) +
                     (p.overread ? 16 : 0);
    unsigned long long st_frames = 0, st_listed = 0, st_eval = 0;
    int ready = 0;

    for (;;) {
        int u = 0;
        if (lane == 0) u = (int)atomicAdd(&p.flags[1], 1u);
        u = __shfl_sync(0xffffffffu, u, 0);
        if (u >= p.B) break;
        const int b = p.order[u];
        const int L = p.len_c[b];
        const float* Db = p.log_probs + (int64_t)b * p.stride_b;
        const float4* summ = p.greedy_sum + (int64_t)b * p.T;
        // init (Alg. 1): acc = 0, last = blank (R6), LM(<SOS>), BT root
        float acc = 0.0f;
        int last = blank, lms = p.lm.start, bts = 0, n = 0;
        bool dead = false;
        if (lm_on)
            for (int q = lane; q < RWS / 4; q += 32)
                ((int4*)rec)[q] = __ldg(&p.lm.rec[(size_t)lms * (p.lm.RW / 4) + q]);
        float bt_maxd = bt_on ? __ldg(&p.bt.maxd[0]) : 0.0f, bt_U = bt_on ? __ldg(&p.bt.U[0]) : 0.0f;
        __syncwarp();
        int32_t* otok = p.out_tokens + (int64_t)b * p.T;
        int32_t* ots = p.out_ts ? p.out_ts + (int64_t)b * p.T : nullptr;
        int32_t* oal = p.out_align ? p.out_align + (int64_t)b * p.T : nullptr;

        // exact Eq. (1) score of a non-blank, non-repeat token (R19 order), next states in ln / bn
        auto eval = [&](int w, float d, int& ln, int& bn) -> float {
            float s = __fadd_rn(__fadd_rn(acc, d), p.beta);
            ln = lms;
            bn = bts;
            int2 e = make_int2(0, 0);
            if (bt_on) e = bts == 0 ? btroot[w] : __ldg(&p.bt.tab[(size_t)bts * V + w]);
            if (lm_on) s = __fmaf_rn(p.alpha_lm, lm_query<LMV>(p.lm, rec, w, ln), s);
            if (bt_on) { bn = e.x; s = __fmaf_rn(p.alpha_bt, __int_as_float(e.y), s); }
            return s;
        };

        // frame summaries (frame_summary_kernel): lane l holds frame 32j + l of the current batch;
        // the next batch is loaded one batch ahead
        const float4 none4 = make_float4(kNeg, kNeg, kNeg, __uint_as_float(0xffffffffu));
        float4 sum_c = lane < L ? summ[lane] : none4;
        float4 sum_n = 32 + lane < L ? summ[32 + lane] : none4;
        // frame rows: one TMA bulk copy per row (lane 0), ringn - 1 rows ahead
        int nissued = 0, ncons = 0;
        for (int r = 0; r < ringn - 1 && r < L; ++r) {
            wait_ready(p, 0, r, ready);
            bulk_row(ring + (size_t)r * (VP + 4), Db + (int64_t)r * p.stride_t, Vp1, &bar[r], lo, hi, lane);
        }
        nissued = min(ringn - 1, L);
        for (int t = 0; t < L; ++t) {
            if ((t & 31) == 0 && t) {
                sum_c = sum_n;
                sum_n = t + 32 + lane < L ? summ[t + 32 + lane] : none4;
            }
            {
                const int r = t + ringn - 1;
                if (r < L) {
                    // every lane's reads of this slot (frame t - 1) precede lane 0's proxy fence and the
                    // async-proxy (TMA) write that reuses it
                    __syncwarp();
                    wait_ready(p, 0, r, ready);
                    bulk_row(ring + (size_t)(r & (ringn - 1)) * (VP + 4), Db + (int64_t)r * p.stride_t, Vp1,
                             &bar[r & (ringn - 1)], lo, hi, lane);
                    nissued = r + 1;
                }
            }
            const float4 fs4 = shfl4(sum_c, t & 31);
            const int w1 = (int)(__float_as_uint(fs4.w) & 0xffffu);
            {
                const int sl = t & (ringn - 1);
                mbar_wait(&bar[sl], (ph >> sl) & 1u);
                ph ^= 1u << sl;
                ncons = t + 1;
            }
            const float* row = ring + (size_t)(t & (ringn - 1)) * (VP + 4) + row_off(Db + (int64_t)t * p.stride_t);
            // exact blank / repeat candidates: no β, no fusion
            uint64_t best = 0;
            int best_ln = lms, best_bn = bts;
            {
                const float sb = __fadd_rn(acc, fs4.z);
                if (sb > kNeg) best = make_key(sb, (uint32_t)blank);
                if (last != blank) {
                    const float sr = __fadd_rn(acc, row[last]);
                    if (sr > kNeg) best = umax64(best, make_key(sr, (uint32_t)last));
                }
            }
            // best non-repeat token, then every token whose bound can reach the running best
            int wt = -1;
            float dt = kNeg;
            if (w1 != (int)kNoTok) {
                if (w1 != last) {
                    wt = w1;
                    dt = fs4.x;
                } else if (fs4.y > kNeg) {  // the best token is the repeat: best other one from the row
                    float bv = kNeg;
                    int bi = 0x7fffffff;
                    for (int w = lane; w < blank; w += 32) {
                        const float v = row[w];
                        if (w != last && v > bv) { bv = v; bi = w; }
                    }
                    uint64_t kb = bi != 0x7fffffff ? make_key(bv, (uint32_t)bi) : 0ull;
#pragma unroll
                    for (int o = 16; o; o >>= 1) kb = umax64(kb, __shfl_xor_sync(0xffffffffu, kb, o));
                    if (kb) { wt = (int)flat_of(kb); dt = score_of(kb); }
                }
            }
            if (wt >= 0) {
                float ub = p.beta;
                if (lm_on) ub += p.alpha_lm * __int_as_float(rec[4]);
                if (bt_on) ub += p.alpha_bt * bt_maxd;
                if (ub_inf) ub = INFINITY;
                const float bs0 = best ? score_of(best) : kNeg;
                const float reach = __fadd_rn(__fadd_rn(acc, dt), ub) + 1e-4f * (1.0f + fabsf(acc) + fabsf(dt) + fabsf(ub));
                if (!best || reach >= bs0) {
                    int ln = 0, bn = 0;
                    const float s = eval(wt, dt, ln, bn);  // every lane, same value (broadcast loads)
                    ++st_eval;
                    if (s > kNeg) {
                        const uint64_t kt = make_key(s, (uint32_t)wt);
                        if (kt > best) { best = kt; best_ln = ln; best_bn = bn; }
                    }
                    const float bs = best ? score_of(best) : kNeg;
                    const float mg = 1e-4f * (1.0f + fabsf(bs) + fabsf(acc) + fabsf(ub));
                    const float dthr = best ? __fsub_rn(__fsub_rn(__fsub_rn(bs, acc), ub), mg) : kNeg;
                    int m = 0;
                    // d2 bounds every non-blank value but w1's: no other token can pass the bound
                    const bool none_else = wt == w1 && !(fs4.y >= dthr);
                    for (int w0 = 0; w0 < blank && !none_else; w0 += 32) {
                        const int w = w0 + lane;
                        const float v = w < blank ? row[w] : kNeg;
                        const bool hit = w < blank && w != last && w != wt && v > kNeg && v >= dthr;
                        const unsigned bal = __ballot_sync(0xffffffffu, hit);
                        if (hit) list[m + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)w;
                        m += __popc(bal);
                    }
                    __syncwarp();
                    st_listed += m;
                    for (int j0 = 0; j0 < m; j0 += 32) {
                        uint64_t kk = 0;
                        int ln2 = 0, bn2 = 0;
                        if (j0 + lane < m) {
                            const int w = list[j0 + lane];
                            const float s2 = eval(w, row[w], ln2, bn2);
                            if (s2 > kNeg) kk = make_key(s2, (uint32_t)w);
                        }
                        st_eval += min(32, m - j0);
                        uint64_t km = kk;
#pragma unroll
                        for (int o = 16; o; o >>= 1) km = umax64(km, __shfl_xor_sync(0xffffffffu, km, o));
                        if (km > best) {
                            const int src = __ffs(__ballot_sync(0xffffffffu, kk == km)) - 1;
                            best = km;
                            best_ln = __shfl_sync(0xffffffffu, ln2, src);
                            best_bn = __shfl_sync(0xffffffffu, bn2, src);
                        }
                    }
                }
            }
            ++st_frames;
            if (!best) { dead = true; break; }  // no finite candidate: the hypothesis dies
            // beams.update: advance the LM / BT states only on emission (R5, R18)
            const int ws = (int)flat_of(best);
            const bool emit = ws != blank && ws != last;
            if (emit) {
                lms = best_ln;
                bts = best_bn;
                __syncwarp();
                if (lm_on)
                    for (int q = lane; q < RWS / 4; q += 32)
                        ((int4*)rec)[q] = __ldg(&p.lm.rec[(size_t)lms * (p.lm.RW / 4) + q]);
                if (bt_on) { bt_maxd = __ldg(&p.bt.maxd[bts]); bt_U = __ldg(&p.bt.U[bts]); }
                if (lane == 0) { otok[n] = ws; if (ots) ots[n] = t; }
                ++n;
                __syncwarp();
            }
            if (oal && lane == 0) oal[t] = ws;
            acc = score_of(best);
            last = ws;
        }
        for (int f = ncons; f < nissued; ++f) {  // rows issued past a dead frame: drain the ring
            const int sl = f & (ringn - 1);
            mbar_wait(&bar[sl], (ph >> sl) & 1u);
            ph ^= 1u << sl;
        }
        __syncwarp();
        // EOS: + α_LM·LM.Final(state); optional boost retraction (R17)
        float fs = acc;
        if (!dead) {
            if (lm_on) fs = __fmaf_rn(p.alpha_lm, __int_as_float(rec[5]), fs);
            if (bt_on && p.retract) fs = __fmaf_rn(-p.alpha_bt, bt_U, fs);
        }
        finish_utterance(p, b, L, n, fs, dead, lane);
        __syncwarp();
    }
    if (lane == 0) {
        if (st_frames) atomicAdd(&p.stats[kFrames], st_frames);
        if (st_listed) atomicAdd(&p.stats[kListed], st_listed);
        if (st_eval) atomicAdd(&p.stats[kEvalSparse], st_eval);
    }
}

template <int LMV>
int launch_fused(const DecodeParams& p, cudaStream_t st, void* ev0, void* ev1, std::string& err) {
    const int RWS = p.use_lm ? ((p.lm.RW + 3) & ~3) : 4;
    // ring depth and warps per CTA: the deepest ring (<= 8 rows) and the most warps (<= 4) that fit
    // 200 KB of shared memory (V' up to 8192: 2 rows x 1 warp)
    const size_t root = p.use_bt ? 8 * (size_t)(p.Vp1 - 1) : 0;
    int ringn = kGRing, gw = kGW;
    while (ringn > 2 && greedy_warp_smem(p.Vp1, RWS, ringn) + root > 200 * 1024) ringn >>= 1;
    while (gw > 1 && gw * greedy_warp_smem(p.Vp1, RWS, ringn) + root > 200 * 1024) --gw;
    const size_t smem = gw * greedy_warp_smem(p.Vp1, RWS, ringn) + root;
    if (smem > 200 * 1024) { err = "shared memory requirement too large (V+1)"; return 2; }
    auto kern = greedy_fused_kernel<LMV>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * gw, smem);
    if (e != cudaSuccess || occ < 1) { err = e != cudaSuccess ? cudaGetErrorString(e) : "occupancy query failed"; return 1; }
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int grid = std::min((p.B + gw - 1) / gw, nsm * occ);
    if (ev0 && ev1) cudaEventRecord((cudaEvent_t)ev0, st);
    kern<<<grid, 32 * gw, smem, st>>>(p, ringn);
    set_kernel_name("greedy_fused_kernel");
    e = cudaGetLastError();
    if (e == cudaSuccess && ev0 && ev1) cudaEventRecord((cudaEvent_t)ev1, st);
    if (e != cudaSuccess) { err = cudaGetErrorString(e); return 1; }
    return 0;
}

}  // namespace

// K = 1: frame_summary_kernel over every valid row (HBM stream), then the chain (plain) or the
// fused warp-per-utterance kernel. The plain path needs no length order (launch_decode skips
// order_kernel for it).
int launch_greedy(const DecodeParams& p, void* stream, void* ev0, void* ev1, std::string& err) {
    cudaStream_t st = (cudaStream_t)stream;
    const bool plain = !p.use_lm && !p.use_bt && p.beta == 0.0f;
    const int64_t grid = (int64_t)p.B * ((p.T + kSumRows - 1) / kSumRows);
    if (grid > 0x7fffffff) { err = "B * T too large"; return 2; }
    // the profile events bracket the dominant kernel: the summary stream (plain) or the fused loop
    if (plain && ev0 && ev1) cudaEventRecord((cudaEvent_t)ev0, st);
    if (grid > 0)  // T = 0: no rows; the second kernel still writes counts and scores
        frame_summary_kernel<<<(int)grid, 32 * kSumRows, 0, st>>>(p.log_probs, p.stride_b, p.stride_t, p.lengths, p.B,
                                                                  p.T, p.Vp1, p.greedy_sum);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess && plain && ev0 && ev1) cudaEventRecord((cudaEvent_t)ev1, st);
    if (e != cudaSuccess) { err = cudaGetErrorString(e); return 1; }
    if (plain) {
        greedy_chain_kernel<<<(p.B + 3) / 4, 128, 0, st>>>(p);
        set_kernel_name("greedy_chain_kernel");
        e = cudaGetLastError();
        if (e != cudaSuccess) { err = cudaGetErrorString(e); return 1; }
        return 0;
    }
    const bool small_lm = !p.use_lm || p.lm.NL <= 2;
    return small_lm ? launch_fused<2>(p, st, ev0, ev1, err) : launch_fused<kMaxLmLevels>(p, st, ev0, ev1, err);
}

}  // namespace flexctc
