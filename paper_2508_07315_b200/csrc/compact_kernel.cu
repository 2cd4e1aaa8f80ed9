// Frame compaction pass: the bandwidth-bound half of the frame step (the
// "compact_frames" kernel K14; §III-C Alg. 1 P:120 "for t ... D[:, t, :]").
//
// Every valid frame row (b, t < L_b; padding is never read, reading R16) is streamed from HBM
// exactly once, by one warp, and reduced to a 256-B record (layout in flexctc_internal.h):
// D[blank], the non-blank tokens within a band below the frame's best non-blank value, sorted by
// (D desc, token asc), and `floor`, an upper bound of every unlisted non-blank D. The band is the
// widest of Δ = 16, 8, 4, 2, 1, 0 nats that lists at most 32 tokens. The latency-bound beam
// kernel (warp_beam_kernel.cu) then needs no per-frame scan of V' values: a frame whose
// filter threshold lies above `floor` is served from the record alone.
//
// Input side (reading R25): with bf16 logits the log-softmax is fused into
// this pass: m = max, S = Σ exp(x - m) in fp64, lse = m + log S (fp64), D = (float)(x - lse); the
// record stores lse so the beam kernel can normalise any other logit it reads exactly the same
// way. The logits are read once at 2 B per element.
//
// Rows are addressed through the prefix of the clamped lengths (rowoff, written by
// rowoff_kernel): the grid covers Σ_b L_b rows, not B·T (LibriSpeech-shaped batches are ~80 %
// padding at T_max), 4 consecutive rows per warp, each loaded as 16-B blocks into registers.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <string>

#include "device_common.cuh"
#include "flexctc_internal.h"

namespace flexctc {
namespace {

using namespace dev;

constexpr int kWarps = 8;        // warps per CTA
constexpr int kRowsPerWarp = 4;  // consecutive flattened rows per warp (one utterance lookup each)
// 16-B blocks per lane held in registers: rows of <= 32·kBlk blocks (V' <= 1149 for fp32 log-probs,
// <= 1273 for bf16 logits) stay in registers
template <bool BF16> constexpr int kBlk = BF16 ? 5 : 9;

// 0xffffffff if a >= b else 0 (one FSET: the counting and hit passes sum / mask these with
// IADD3 / LOP3 instead of a predicate + select per element)
__device__ __forceinline__ uint32_t ge_mask(float a, float b) {
    uint32_t m;
    asm("set.ge.u32.f32 %0, %1, %2;" : "=r"(m) : "f"(a), "f"(b));
    return m;
}

template <bool BF16>
__device__ __forceinline__ float elem(const uint4& q, int j) {  // element j of a 16-B block
    if constexpr (BF16) {
        const uint32_t u = j < 2 ? (j == 0 ? q.x : q.x >> 16) : j < 4 ? (j == 2 ? q.y : q.y >> 16)
                         : j < 6 ? (j == 4 ? q.z : q.z >> 16) : (j == 6 ? q.w : q.w >> 16);
        return bf16f((uint16_t)(u & 0xffffu));
    } else {
        return __uint_as_float(j == 0 ? q.x : j == 1 ? q.y : j == 2 ? q.z : q.w);
    }
}

// One row -> one record. The warp loads the row's covering 16-B blocks (LDG.128, evict-first: D
// is read once) into registers, kBlk per lane; a block lying partly outside [lo, hi) (at most
// the tensor's first and last row) is assembled element by element from inside the range.
// Rows longer than 32·kBlk blocks take the generic path (values re-read from L1/L2).
template <bool BF16>
__device__ void compact_row(const void* row, int Vp1, uint8_t* rec, uint64_t* keys, int lane, const char* lo,
                            const char* hi) {
    constexpr int EPB = BF16 ? 8 : 4;  // elements per 16-B block
    constexpr int ESZ = BF16 ? 2 : 4;
    const int blank = Vp1 - 1;
    const char* src = (const char*)row;
    const char* g = (const char*)((uintptr_t)src & ~(uintptr_t)15);
    const int off = (int)(src - g) / ESZ;  // element offset of w = 0 inside block 0
    const int nblk = (off + Vp1 + EPB - 1) / EPB;
    const bool in_regs = nblk <= 32 * kBlk<BF16>;
    uint4 q[kBlk<BF16>];
    if (in_regs) {
        const uint64_t pol = policy_evict_first();
        const bool all_in = g >= lo && g + 16 * (size_t)nblk <= hi;  // every covering block inside the tensor
        const uint32_t ninf = BF16 ? 0xff80ff80u : 0xff800000u;  // -inf in every element
#pragma unroll
        for (int i = 0; i < kBlk<BF16>; ++i) {
            const int bi = lane + 32 * i;
            q[i] = make_uint4(ninf, ninf, ninf, ninf);
            if (bi < nblk) {
                const char* a = g + 16 * (size_t)bi;
                if (all_in || (a >= lo && a + 16 <= hi)) {
                    asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                                 : "=r"(q[i].x), "=r"(q[i].y), "=r"(q[i].z), "=r"(q[i].w) : "l"(a), "l"(pol));
                } else {  // edge block: only the row's own elements
                    uint16_t h[8] = {};
                    float f[4] = {};
                    for (int j = 0; j < EPB; ++j) {
                        const int w = bi * EPB + j - off;
                        if (w >= 0 && w < Vp1) {
                            if constexpr (BF16) h[j] = __ldg((const uint16_t*)src + w);
                            else f[j] = __ldg((const float*)src + w);
                        }
                    }
                    if constexpr (BF16)
                        q[i] = make_uint4(h[0] | ((uint32_t)h[1] << 16), h[2] | ((uint32_t)h[3] << 16),
                                          h[4] | ((uint32_t)h[5] << 16), h[6] | ((uint32_t)h[7] << 16));
                    else
                        q[i] = make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]),
                                          __float_as_uint(f[3]));
                }
            }
        }
    }
    // token index of element slot (i, j) of this lane; v[] = the non-blank values, -inf elsewhere
    auto tok_of = [&](int i, int j) { return (lane + 32 * i) * EPB + j - off; };
    auto ld_w = [&](int w) -> float {  // generic path
        if constexpr (BF16) return bf16f(__ldg((const uint16_t*)src + w));
        else return __ldg((const float*)src + w);
    };
    constexpr int NV = kBlk<BF16> * EPB;
    float v[NV];
    float mn = kNeg;  // max over non-blank tokens (NaN never wins)
    if (in_regs) {
        float m4[4] = {kNeg, kNeg, kNeg, kNeg};  // independent partial maxima
#pragma unroll
        for (int i = 0; i < kBlk<BF16>; ++i) {
            // valid elements j of block bi: [jlo, jhi) (interior blocks: all; the blank, the last
            // element of the row, lies in the last block)
            const int base = (lane + 32 * i) * EPB - off;
            const int jlo = min(max(-base, 0), EPB), jhi = min(max(blank - base, 0), EPB);
#pragma unroll
            for (int j = 0; j < EPB; ++j) {
                const float x = elem<BF16>(q[i], j);
                v[i * EPB + j] = (j >= jlo && j < jhi) ? x : kNeg;
                m4[j & 3] = fmaxf(m4[j & 3], v[i * EPB + j]);
            }
        }
        mn = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
    } else {
        for (int w = lane; w < blank; w += 32) mn = fmaxf(mn, ld_w(w));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mn = fmaxf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    const float xb = ld_w(blank);  // blank value (logit or D): an L1 hit

    double lse = 0.0;
    if constexpr (BF16) {  // R25: m over every logit, S in fp64, lse = m + log S
        const double m = (double)fmaxf(mn, xb);
        double S = 0.0;
        if (in_regs) {
#pragma unroll
            for (int i = 0; i < NV; ++i)
                if (v[i] > kNeg) S += exp((double)v[i] - m);  // exp(-inf) = 0: only finite logits count
            if (lane == 0) S += exp((double)xb - m);
        } else {
            for (int w = lane; w < Vp1; w += 32) S += exp((double)ld_w(w) - m);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) S += __shfl_xor_sync(0xffffffffu, S, o);
        lse = m + log(S);
    }
    auto dval = [&](float x) -> float {
        if constexpr (BF16) return (float)((double)x - lse);
        else return x;
    };
    auto count_ge = [&](float th, int& mine) -> int {  // non-blank values >= th: this lane's, warp total
        int c = 0;
        if (in_regs) {
            int c4[4] = {0, 0, 0, 0};  // independent partial sums (no serial add chain)
#pragma unroll
            for (int i = 0; i < NV; ++i) c4[i & 3] += v[i] >= th ? 1 : 0;
            c = (c4[0] + c4[1]) + (c4[2] + c4[3]);
        } else {
            for (int w = lane; w < blank; w += 32) c += ld_w(w) >= th ? 1 : 0;
        }
        mine = c;
        return __reduce_add_sync(0xffffffffu, c);
    };

    // band: the widest Δ in {16, 8, 4, 2, 1, 0} with at most kCmpList non-blank values >= mn - Δ
    // (counts are monotone in Δ: a binary search over the six, <= 3 counting passes)
    float thr = INFINITY;
    int n = 0, h = 0;  // listed tokens: warp total, this lane's
    if (mn > kNeg) {
        int lo_i = 0, hi_i = 5;  // the smallest index (widest band) whose count fits; Δ = 16 >> index
        while (lo_i <= hi_i) {
            const int mid = (lo_i + hi_i) >> 1;
            const float th = __fsub_rn(mn, mid == 5 ? 0.0f : (float)(16 >> mid));
            int mine;
            const int c = count_ge(th, mine);
            if (c <= kCmpList) { thr = th; n = c; h = mine; hi_i = mid - 1; } else { lo_i = mid + 1; }
        }
    }
    // collect the listed tokens, then rank them by (value desc, token asc)
    if (n > 0) {
        int pos = h;  // exclusive prefix of the hit counts over the lanes
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, pos, o);
            if (lane >= o) pos += y;
        }
        pos -= h;
        if (h) {
            if (in_regs) {
                // hit mask of this lane's elements, then one key per set bit
                uint32_t hlo = 0, hhi = 0;
#pragma unroll
                for (int e = 0; e < NV; ++e) {
                    if (e < 32) hlo |= (v[e] >= thr ? 1u : 0u) << e;
                    else hhi |= (v[e] >= thr ? 1u : 0u) << (e - 32);
                }
                uint64_t hm = ((uint64_t)hhi << 32) | hlo;
                while (hm) {
                    const int e = __ffsll((long long)hm) - 1;
                    hm &= hm - 1;
                    const int w = tok_of(e / EPB, e % EPB);
                    const float x = ld_w(w);  // an L1 hit (the row was just loaded)
                    keys[pos++] = ((uint64_t)ord_of(x) << 32) | (uint64_t)(0xffffffffu - (uint32_t)w);
                }
            } else {
                for (int w = lane; w < blank; w += 32) {
                    const float x = ld_w(w);
                    if (x >= thr) keys[pos++] = ((uint64_t)ord_of(x) << 32) | (uint64_t)(0xffffffffu - (uint32_t)w);
                }
            }
        }
        __syncwarp();
        if (lane < n) {
            const uint64_t mykey = keys[lane];
            int r = 0, r2 = 0;
            int j = 0;
            for (; j + 1 < n; j += 2) { r += keys[j] > mykey ? 1 : 0; r2 += keys[j + 1] > mykey ? 1 : 0; }
            if (j < n) r += keys[j] > mykey ? 1 : 0;
            r += r2;
            const int w = (int)(0xffffffffu - (uint32_t)mykey);
            ((float*)(rec + 32))[r] = dval(score_of(mykey));
            ((uint16_t*)(rec + 160))[r] = (uint16_t)w;
        }
        __syncwarp();
    }
    if (lane == 0) {
        float* f = (float*)rec;
        f[0] = dval(xb);
        // unlisted non-blank values are < thr (log-probs) or their logits are (bf16: the rounding
        // of x - lse is monotone, so D <= fl(thr - lse))
        f[1] = mn > kNeg ? dval(thr) : kNeg;  // thr = +inf: no band fits (no usable list)
        ((int32_t*)rec)[2] = n;
        f[3] = mn > kNeg ? thr : INFINITY;  // listed iff the raw value (log-prob or logit) >= this
        *(double*)(rec + 16) = lse;
    }
}

template <bool BF16>
__global__ void __launch_bounds__(32 * kWarps, 3) frame_compact_kernel(const void* __restrict__ X, int64_t sb, int64_t stt,
                                                                   const int64_t* __restrict__ rowoff, int B, int T,
                                                                   int Vp1, uint8_t* __restrict__ cmp, const char* lo,
                                                                   const char* hi) {
    __shared__ uint64_t s_keys[kWarps][kCmpList];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t nrows = __ldg(&rowoff[B]);
    const int64_t nchunks = (nrows + kRowsPerWarp - 1) / kRowsPerWarp;
    const size_t esz = BF16 ? 2 : 4;
    for (int64_t c = (int64_t)blockIdx.x * kWarps + wid; c < nchunks; c += (int64_t)gridDim.x * kWarps) {
        int64_t r = c * kRowsPerWarp;
        // utterance of row r: the last b with rowoff[b] <= r (binary search, L1-resident)
        int lo_b = 0, hi_b = B - 1;
        while (lo_b < hi_b) {
            const int mid = (lo_b + hi_b + 1) >> 1;
            if (__ldg(&rowoff[mid]) <= r) lo_b = mid; else hi_b = mid - 1;
        }
        int b = lo_b;
        int64_t off = __ldg(&rowoff[b]), end = __ldg(&rowoff[b + 1]);
        const int64_t rend = min(nrows, r + kRowsPerWarp);
        for (; r < rend; ++r) {
            while (r >= end) { ++b; off = end; end = __ldg(&rowoff[b + 1]); }  // skips empty utterances
            const int t = (int)(r - off);
            const char* row = (const char*)X + ((int64_t)b * sb + (int64_t)t * stt) * esz;
            compact_row<BF16>(row, Vp1, cmp + ((int64_t)b * T + t) * kCmpBytes, s_keys[wid], lane, lo, hi);
        }
    }
}

// ---- TMA-staged pass (the default when a row fits the registers) ----------------------------
// Same records as frame_compact_kernel, different data movement: a persistent grid (#SMs x the
// occupancy) in which warp g takes the chunks of 4 consecutive rows g, g + W, g + 2W, ... (W =
// warps in the grid; neighbouring warps read neighbouring chunks). Each warp owns a ring of kStages row slots in shared memory; lane
// 0 stages row k + kStages - 1 with ONE cp.async.bulk (TMA, completion on the slot's mbarrier)
// before the warp ranks row k, so the HBM stream runs ahead of the ranking instead of every warp
// alternating between waiting for its row and computing on it (the register-loading kernel above
// ran at 0.55 IPC per SMSP with most warps stalled on their own loads).
constexpr int kTWarps = 8;   // warps per CTA
constexpr int kTChunk = 4;   // consecutive rows per warp chunk (one utterance search each)

template <bool BF16>
__host__ __device__ constexpr int slot_bytes(int Vp1) {  // covering 16-B blocks of any row alignment
    return ((16 - (BF16 ? 2 : 4)) + Vp1 * (BF16 ? 2 : 4) + 15) & ~15;
}
template <int kStages>  // row slots per warp
__host__ __device__ constexpr int warp_smem(int sbytes) { return kStages * sbytes + 8 * kCmpList + 16 * kStages; }

// Row `src` into `slot` (16-B aligned) at byte offset src mod 16, completing on `bar` (count 1): one
// bulk copy of the covering 16-B blocks when those lie inside [lo, hi) (the tensor's bytes),
// otherwise (at most the tensor's first and last row) a plain copy of the row's own elements.
template <bool BF16>
__device__ __forceinline__ void stage_row(uint8_t* slot, const char* src, int Vp1, uint64_t* bar, const char* lo,
                                          const char* hi, int lane) {
    constexpr int ESZ = BF16 ? 2 : 4;
    const int offb = (int)((uintptr_t)src & 15);
    const char* g = src - offb;
    const uint32_t bytes = (uint32_t)((offb + Vp1 * ESZ + 15) & ~15);
    if (g >= lo && g + bytes <= hi) {
        if (lane == 0) {
            fence_proxy_async();  // the warp's earlier generic accesses of this slot before the async write
            mbar_arrive_tx(bar, bytes);
            bulk_g2s_hint(slot, g, bytes, bar, policy_evict_first());  // D is read once: keep the LM / boost tables in L2
        }
    } else {
        for (int w = lane; w < Vp1; w += 32) {
            if constexpr (BF16) ((uint16_t*)(slot + offb))[w] = __ldg((const uint16_t*)src + w);
            else ((float*)(slot + offb))[w] = __ldg((const float*)src + w);
        }
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
    }
}

// One staged row -> one record (the ranking of compact_row, reading shared memory). Before the
// blocks are loaded, the slot's elements outside the row's non-blank tokens (the head of block 0,
// the blank and the tail of the last block) are overwritten with -inf, so the max / count / hit
// passes need no per-element range test.
template <bool BF16>
__device__ void compact_staged(uint8_t* slot, int offb, int Vp1, uint8_t* rec, uint64_t* keys, int lane,
                               const double* __restrict__ etab) {
    constexpr int EPB = BF16 ? 8 : 4;
    constexpr int ESZ = BF16 ? 2 : 4;
    constexpr int NV = kBlk<BF16> * EPB;
    const int blank = Vp1 - 1;
    const int off = offb / ESZ;
    const int nblk = (offb + Vp1 * ESZ + 15) >> 4;
    auto ld_w = [&](int w) -> float {
        if constexpr (BF16) return bf16f(((const uint16_t*)slot)[off + w]);
        else return ((const float*)slot)[off + w];
    };
    const float xb = ld_w(blank);
    __syncwarp();  // every lane has read the blank before it is masked
    if (lane < EPB) {
        const int e1 = lane, e2 = off + blank + lane;
        if constexpr (BF16) {
            if (e1 < off) ((uint16_t*)slot)[e1] = 0xff80u;
            if (e2 < nblk * EPB) ((uint16_t*)slot)[e2] = 0xff80u;
        } else {
            if (e1 < off) ((float*)slot)[e1] = kNeg;
            if (e2 < nblk * EPB) ((float*)slot)[e2] = kNeg;
        }
    }
    __syncwarp();
    const uint32_t ninf = BF16 ? 0xff80ff80u : 0xff800000u;
    float v[NV];
    float m4[4] = {kNeg, kNeg, kNeg, kNeg};
#pragma unroll
    for (int i = 0; i < kBlk<BF16>; ++i) {
        const int bi = lane + 32 * i;
        const uint4 q = bi < nblk ? ((const uint4*)slot)[bi] : make_uint4(ninf, ninf, ninf, ninf);
#pragma unroll
        for (int j = 0; j < EPB; ++j) {
            v[i * EPB + j] = elem<BF16>(q, j);
            m4[j & 3] = fmaxf(m4[j & 3], v[i * EPB + j]);
        }
    }
    float mn = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
#pragma unroll
    for (int o = 16; o; o >>= 1) mn = fmaxf(mn, __shfl_xor_sync(0xffffffffu, mn, o));

    double lse = 0.0;
    if constexpr (BF16) {  // R25: m over every logit, S in fp64, lse = m + log S
        const double m = (double)fmaxf(mn, xb);
        double S = 0.0;
        if (etab && m >= -700.0 && m <= 700.0) {
            // exp of every bf16 value from a 65536-entry fp64 table (exp_table_kernel): lse =
            // log Σ exp(x) = m + log Σ exp(x - m) with one table load per logit instead of an
            // fp64 exp (|m| <= 700: no term overflows, the largest does not underflow)
#pragma unroll
            for (int i = 0; i < NV; ++i)
                if (v[i] > kNeg) S += __ldg(&etab[__float_as_uint(v[i]) >> 16]);
            if (lane == 0) S += __ldg(&etab[__float_as_uint(xb) >> 16]);
#pragma unroll
            for (int o = 16; o; o >>= 1) S += __shfl_xor_sync(0xffffffffu, S, o);
            lse = log(S);
        } else {
#pragma unroll
            for (int i = 0; i < NV; ++i)
                if (v[i] > kNeg) S += exp((double)v[i] - m);
            if (lane == 0) S += exp((double)xb - m);
#pragma unroll
            for (int o = 16; o; o >>= 1) S += __shfl_xor_sync(0xffffffffu, S, o);
            lse = m + log(S);
        }
    }
    auto dval = [&](float x) -> float {
        if constexpr (BF16) return (float)((double)x - lse);
        else return x;
    };
    auto count_ge = [&](float th, int& mine) -> int {
        // v >= th  <=>  fl(v - th) has a clear sign bit (rounding never flips the sign; v == th
        // gives +0; v = -inf gives -inf): one FADD and one LEA.HI per element count the values below
        uint32_t c2[2] = {0u, 0u};
#pragma unroll
        for (int i = 0; i < NV; ++i) c2[i & 1] += __float_as_uint(__fsub_rn(v[i], th)) >> 31;
        mine = NV - (int)(c2[0] + c2[1]);
        return __reduce_add_sync(0xffffffffu, mine);
    };
    // band: the widest Δ in {16, 8, 4, 2, 1, 0} with at most kCmpList non-blank values >= mn - Δ.
    // The binary search over the six starts at Δ = 2 instead of the middle (Δ = 4): on CTC-peaky
    // rows Δ = 2 holds > 32 tokens on ~70 % of frames and Δ = 1 then fits, so most rows take two
    // counting passes instead of three (same result: the counts are monotone in Δ)
    float thr = INFINITY;
    int n = 0, h = 0;
    if (mn > kNeg) {
        int lo_i = 0, hi_i = 5;
        bool first = true;
        while (lo_i <= hi_i) {
            const int mid = first ? 3 : (lo_i + hi_i) >> 1;
            first = false;
            const float th = __fsub_rn(mn, mid == 5 ? 0.0f : (float)(16 >> mid));
            int mine;
            const int c = count_ge(th, mine);
            if (c <= kCmpList) { thr = th; n = c; h = mine; hi_i = mid - 1; } else { lo_i = mid + 1; }
        }
    }
    if (n > 0) {
        int pos = h;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, pos, o);
            if (lane >= o) pos += y;
        }
        pos -= h;
        if (h) {
            uint32_t hlo = 0, hhi = 0;
#pragma unroll
            for (int e = 0; e < NV; ++e) {
                if (e < 32) hlo |= ge_mask(v[e], thr) & (1u << e);
                else hhi |= ge_mask(v[e], thr) & (1u << (e - 32));
            }
            uint64_t hm = ((uint64_t)hhi << 32) | hlo;
            while (hm) {
                const int e = __ffsll((long long)hm) - 1;
                hm &= hm - 1;
                const int w = (lane + 32 * (e / EPB)) * EPB + e % EPB - off;
                const float x = ld_w(w);
                keys[pos++] = ((uint64_t)ord_of(x) << 32) | (uint64_t)(0xffffffffu - (uint32_t)w);
            }
        }
        __syncwarp();
        if (lane < n) {
            const uint64_t mykey = keys[lane];
            int r = 0, r2 = 0;
            int j = 0;
            for (; j + 1 < n; j += 2) { r += keys[j] > mykey ? 1 : 0; r2 += keys[j + 1] > mykey ? 1 : 0; }
            if (j < n) r += keys[j] > mykey ? 1 : 0;
            r += r2;
            const int w = (int)(0xffffffffu - (uint32_t)mykey);
            ((float*)(rec + 32))[r] = dval(score_of(mykey));
            ((uint16_t*)(rec + 160))[r] = (uint16_t)w;
        }
    }
    if (lane == 0) {
        float* f = (float*)rec;
        f[0] = dval(xb);
        f[1] = mn > kNeg ? dval(thr) : kNeg;
        ((int32_t*)rec)[2] = n;
        f[3] = mn > kNeg ? thr : INFINITY;
        *(double*)(rec + 16) = lse;
    }
}

template <bool BF16, int kStages>
__global__ void __launch_bounds__(32 * kTWarps, kStages == 2 && !BF16 ? 3 : 2)
    frame_compact_tma_kernel(const void* __restrict__ X, int64_t sb, int64_t stt, const int64_t* __restrict__ rowoff,
                             int B, int T, int Vp1, uint8_t* __restrict__ cmp, const char* lo, const char* hi,
                             int sbytes, const double* __restrict__ etab, const WarmRanges warm) {
    extern __shared__ __align__(128) uint8_t smem[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const size_t esz = BF16 ? 2 : 4;
    uint8_t* base = smem + (size_t)wid * warp_smem<kStages>(sbytes);
    uint64_t* keys = (uint64_t*)(base + kStages * sbytes);
    uint64_t* bar = keys + kCmpList;
    int2* meta = (int2*)(bar + kStages);  // (b, t) of the row in each slot
    if (lane == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&bar[s], 1);
        fence_mbar_init();
    }
    __syncwarp();
    const int64_t nrows = __ldg(&rowoff[B]);
    // warp g takes the chunks of kTChunk consecutive rows g, g + W, g + 2W, ... (W = warps in the
    // grid): one utterance search per chunk, the chunk's later rows advance the cursor
    const int64_t W = (int64_t)gridDim.x * kTWarps;
    const int64_t g = (int64_t)blockIdx.x * kTWarps + wid;
    auto row_of = [&](int k) -> int64_t { return (g + (int64_t)(k / kTChunk) * W) * kTChunk + k % kTChunk; };
    int ib = 0;  // issue cursor: utterance of the last issued row, its first and end rows
    int64_t ioff = 0, iend = 0;
    auto issue = [&](int k, int s) {
        const int64_t r = row_of(k);
        if (k % kTChunk == 0) {
            int lo_b = 0, hi_b = B - 1;  // the last b with rowoff[b] <= r (L1-resident)
            while (lo_b < hi_b) {
                const int mid = (lo_b + hi_b + 1) >> 1;
                if (__ldg(&rowoff[mid]) <= r) lo_b = mid; else hi_b = mid - 1;
            }
            ib = lo_b;
            ioff = __ldg(&rowoff[ib]);
            iend = __ldg(&rowoff[ib + 1]);
        }
        while (r >= iend) { ++ib; ioff = iend; iend = __ldg(&rowoff[ib + 1]); }  // skips empty utterances
        const int t = (int)(r - ioff);
        if (lane == 0) meta[s] = make_int2(ib, t);  // published by the arrive (release) / wait (acquire)
        const char* row = (const char*)X + ((int64_t)ib * sb + (int64_t)t * stt) * esz;
        stage_row<BF16>(base + s * sbytes, row, Vp1, &bar[s], lo, hi, lane);
    };
#pragma unroll
    for (int s = 0; s < kStages - 1; ++s)
        if (row_of(s) < nrows) issue(s, s);
    // L2 warm-up of the decode's lookup tables, interleaved with the rows: at row k every thread
    // prefetches line gtid + k * nthreads of the concatenated ranges (evict-last)
    const int64_t wl0 = (warm.n[0] + 127) >> 7, wl1 = (warm.n[1] + 127) >> 7, wl2 = (warm.n[2] + 127) >> 7,
                  wl3 = (warm.n[3] + 127) >> 7;
    const int64_t wlines = wl0 + wl1 + wl2 + wl3;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gthreads = (int64_t)gridDim.x * blockDim.x;
    auto warm_step = [&](int k) {
        const int64_t i = gtid + (int64_t)k * gthreads;
        if (i >= wlines) return;
        const char* q = i < wl0 ? warm.a[0] + (i << 7)
                        : i < wl0 + wl1 ? warm.a[1] + ((i - wl0) << 7)
                        : i < wl0 + wl1 + wl2 ? warm.a[2] + ((i - wl0 - wl1) << 7) : warm.a[3] + ((i - wl0 - wl1 - wl2) << 7);
        asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(q));
    };
    uint32_t ph = 0;
    int s = 0;
    int k = 0;
    for (; row_of(k) < nrows; ++k) {
        warm_step(k);
        const int kn = k + kStages - 1;
        const int sn = s == 0 ? kStages - 1 : s - 1;  // the slot ranked in the previous iteration
        if (row_of(kn) < nrows) issue(kn, sn);
        mbar_wait(&bar[s], (ph >> s) & 1u);
        ph ^= 1u << s;
        const int2 bt = meta[s];
        const char* row = (const char*)X + ((int64_t)bt.x * sb + (int64_t)bt.y * stt) * esz;
        compact_staged<BF16>(base + s * sbytes, (int)((uintptr_t)row & 15), Vp1,
                             cmp + ((int64_t)bt.x * T + bt.y) * kCmpBytes, keys, lane, etab);
        __syncwarp();  // the slot and the key buffer are free again
        s = s + 1 == kStages ? 0 : s + 1;
    }
    for (; gtid + (int64_t)k * gthreads < wlines; ++k) warm_step(k);  // lines left after the rows
}

// rowoff[b] = Σ_{b' < b} len_c[b'], rowoff[B] = Σ L (one CTA; block scan over 1024-wide tiles)
__global__ void __launch_bounds__(1024) rowoff_kernel(const int32_t* __restrict__ len_c, int B, int64_t* rowoff) {
    __shared__ int64_t s_w[32];
    __shared__ int64_t s_carry;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int b0 = 0; b0 < B; b0 += 1024) {
        const int b = b0 + threadIdx.x;
        const int64_t v = b < B ? (int64_t)len_c[b] : 0;
        int64_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_w[wid] = x;
        __syncthreads();
        if (wid == 0) {
            int64_t z = s_w[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t y = __shfl_up_sync(0xffffffffu, z, o);
                if (lane >= o) z += y;
            }
            s_w[lane] = z;  // inclusive warp totals
        }
        __syncthreads();
        const int64_t carry = s_carry;
        const int64_t incl = carry + (wid ? s_w[wid - 1] : 0) + x;
        if (b < B) rowoff[b] = incl - v;
        __syncthreads();
        if (threadIdx.x == 1023) s_carry = incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) rowoff[B] = s_carry;
}

// etab[u] = exp(bf16 value with bits u) in fp64 (inf / NaN patterns and overflowing values give
// inf / NaN; the pass only uses the table when every term of the row is finite)
__global__ void exp_table_kernel(double* etab) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u < 65536) etab[u] = exp((double)bf16f((uint16_t)u));
}

}  // namespace

// one table per device, built on first use and kept for the process lifetime (512 KB)
const double* bf16_exp_table(void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    static std::mutex mu;
    static double* tab[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    double*& t = tab[dev & 63];
    if (!t) {
        // built synchronously (any stream may use it next); never inside a stream capture, where
        // the callers fall back to evaluating exp themselves
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return nullptr;
        double* d = nullptr;
        if (cudaMalloc(&d, 65536 * sizeof(double)) != cudaSuccess) return nullptr;
        exp_table_kernel<<<256, 256, 0, st>>>(d);
        if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess) { cudaFree(d); return nullptr; }
        t = d;
    }
    return t;
}

int launch_rowoff(const int32_t* len_c, int B, int64_t* rowoff, void* stream, std::string& err) {
    rowoff_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(len_c, B, rowoff);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { err = cudaGetErrorString(e); return 1; }
    return 0;
}

// rowoff [B + 1] (launch_rowoff) on the device. Rows that fit the registers: the TMA-staged pass,
// a persistent grid of #SMs x its occupancy; longer rows: the register-loading kernel, one warp per
// 4 rows, grid = #SMs x 16 CTAs at most (grid stride over Σ L_b / 4 row chunks).
bool compact_fuses_warm(int Vp1, bool bf16) {
    const char* e = getenv("FLEXCTC_CMP_TMA");
    if (e && e[0] == '0') return false;
    const int esz = bf16 ? 2 : 4, epb = bf16 ? 8 : 4;
    const int nblk_max = ((16 - esz) / esz + Vp1 + epb - 1) / epb;
    return nblk_max <= 32 * (bf16 ? kBlk<true> : kBlk<false>);
}

int launch_compact(const void* x, bool bf16, int64_t stride_b, int64_t stride_t, const int64_t* rowoff, int B, int T,
                   int Vp1, uint8_t* cmp, void* stream, std::string& err, const WarmRanges* warm) {
    if (B == 0 || T == 0) return 0;
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaStream_t st = (cudaStream_t)stream;
    // the tensor's byte range: no load leaves it (edge blocks of the first / last row are assembled
    // element by element)
    const size_t esz = bf16 ? 2 : 4;
    const char* lo = (const char*)x;
    const char* hi = lo + esz * ((size_t)(B - 1) * stride_b + (size_t)(T - 1) * stride_t + Vp1);
    const int epb = bf16 ? 8 : 4;
    const int nblk_max = ((16 - (int)esz) / (int)esz + Vp1 + epb - 1) / epb;
    const bool staged = getenv("FLEXCTC_CMP_TMA") ? getenv("FLEXCTC_CMP_TMA")[0] != '0' : true;
    if (staged && nblk_max <= 32 * (bf16 ? kBlk<true> : kBlk<false>)) {
        const int sbytes = bf16 ? slot_bytes<true>(Vp1) : slot_bytes<false>(Vp1);
        // 2 row slots per warp (3 slots: 47 us at c4, 4 slots: 61 us, both fewer CTAs per SM than
        // 2 slots' 44.5 us; profiles/r2/ab_compact_tma_stages.txt)
        const int smem = kTWarps * warp_smem<2>(sbytes);
        auto kern = bf16 ? frame_compact_tma_kernel<true, 2> : frame_compact_tma_kernel<false, 2>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        int occ = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 32 * kTWarps, smem);
        const int64_t want = ((int64_t)B * T + kTWarps * kTChunk - 1) / (kTWarps * kTChunk);
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)nsm * std::max(occ, 1)));
        const double* etab = bf16 ? bf16_exp_table(st) : nullptr;  // NULL: the pass evaluates exp itself
        kern<<<grid, 32 * kTWarps, smem, st>>>(x, stride_b, stride_t, rowoff, B, T, Vp1, cmp, lo, hi, sbytes, etab,
                                               warm ? *warm : WarmRanges{});
    } else {
        const int64_t max_chunks = ((int64_t)B * T + kRowsPerWarp - 1) / kRowsPerWarp;
        const int64_t want = (max_chunks + kWarps - 1) / kWarps;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)nsm * 16));
        if (bf16)
            frame_compact_kernel<true><<<grid, 32 * kWarps, 0, st>>>(x, stride_b, stride_t, rowoff, B, T, Vp1, cmp, lo, hi);
        else
            frame_compact_kernel<false><<<grid, 32 * kWarps, 0, st>>>(x, stride_b, stride_t, rowoff, B, T, Vp1, cmp, lo, hi);
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { err = cudaGetErrorString(e); return 1; }
    return 0;
}

}  // namespace flexctc
