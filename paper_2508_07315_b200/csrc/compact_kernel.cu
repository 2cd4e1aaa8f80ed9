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

}  // namespace

int launch_rowoff(const int32_t* len_c, int B, int64_t* rowoff, void* stream, std::string& err) {
    rowoff_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(len_c, B, rowoff);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { err = cudaGetErrorString(e); return 1; }
    return 0;
}

// rowoff [B + 1] (launch_rowoff) on the device; one warp per 8 rows, grid = #SMs x 8 CTAs (grid
// stride over Σ L_b / 8 row chunks).
int launch_compact(const void* x, bool bf16, int64_t stride_b, int64_t stride_t, const int64_t* rowoff, int B, int T,
                   int Vp1, uint8_t* cmp, void* stream, std::string& err) {
    if (B == 0 || T == 0) return 0;
    int dev = 0, nsm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int64_t max_chunks = ((int64_t)B * T + kRowsPerWarp - 1) / kRowsPerWarp;
    const int64_t want = (max_chunks + kWarps - 1) / kWarps;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)nsm * 16));
    cudaStream_t st = (cudaStream_t)stream;
    // the tensor's byte range: no load leaves it (edge blocks of the first / last row are assembled
    // element by element)
    const size_t esz = bf16 ? 2 : 4;
    const char* lo = (const char*)x;
    const char* hi = lo + esz * ((size_t)(B - 1) * stride_b + (size_t)(T - 1) * stride_t + Vp1);
    if (bf16)
        frame_compact_kernel<true><<<grid, 32 * kWarps, 0, st>>>(x, stride_b, stride_t, rowoff, B, T, Vp1, cmp, lo, hi);
    else
        frame_compact_kernel<false><<<grid, 32 * kWarps, 0, st>>>(x, stride_b, stride_t, rowoff, B, T, Vp1, cmp, lo, hi);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { err = cudaGetErrorString(e); return 1; }
    return 0;
}

}  // namespace flexctc
