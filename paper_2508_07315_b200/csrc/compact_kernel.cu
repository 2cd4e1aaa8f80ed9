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
// order_kernel): the grid covers Σ_b L_b rows, not B·T (LibriSpeech-shaped batches are ~80 %
// padding at T_max), 8 consecutive rows per warp.
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
constexpr int kRowsPerWarp = 8;  // consecutive flattened rows per warp
constexpr int kPerLane = 33;     // register-resident elements per lane (V' <= 1056)

template <bool BF16>
__device__ __forceinline__ float ld_x(const void* row, int w) {
    if constexpr (BF16) return bf16f(__ldg((const uint16_t*)row + w));
    else return __ldg((const float*)row + w);
}

// One row -> one record. `v` holds the row when V' <= 32·kPerLane (the usual shape: one HBM
// read); larger rows are re-read from L1/L2 by each pass.
template <bool BF16>
__device__ void compact_row(const void* row, int Vp1, uint8_t* rec, uint64_t* keys, int lane) {
    const int blank = Vp1 - 1;
    const bool in_regs = Vp1 <= 32 * kPerLane;
    float v[kPerLane];
    float mn = kNeg;  // max over non-blank
    float xb = kNeg;  // blank value (logit or D)
    if (in_regs) {
#pragma unroll
        for (int i = 0; i < kPerLane; ++i) {
            const int w = lane + 32 * i;
            v[i] = w < Vp1 ? ld_x<BF16>(row, w) : kNeg;
        }
        xb = ld_x<BF16>(row, blank);  // broadcast (L1 hit)
#pragma unroll
        for (int i = 0; i < kPerLane; ++i)
            if (lane + 32 * i < blank) mn = fmaxf(mn, v[i]);
    } else {
        xb = ld_x<BF16>(row, blank);
        for (int w = lane; w < blank; w += 32) mn = fmaxf(mn, ld_x<BF16>(row, w));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mn = fmaxf(mn, __shfl_xor_sync(0xffffffffu, mn, o));

    double lse = 0.0;
    if constexpr (BF16) {  // R25: m over every logit, S in fp64, lse = m + log S
        const double m = (double)fmaxf(mn, xb);
        double S = 0.0;
        if (in_regs) {
#pragma unroll
            for (int i = 0; i < kPerLane; ++i)
                if (lane + 32 * i < Vp1) S += exp((double)v[i] - m);
        } else {
            for (int w = lane; w < Vp1; w += 32) S += exp((double)ld_x<BF16>(row, w) - m);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) S += __shfl_xor_sync(0xffffffffu, S, o);
        lse = m + log(S);
    }
    auto dval = [&](float x) -> float {
        if constexpr (BF16) return (float)((double)x - lse);
        else return x;
    };

    // band: the widest Δ in {16, 8, 4, 2, 1, 0} with at most kCmpList non-blank values >= mn - Δ
    float thr = INFINITY;
    int n = 0;
    if (mn > kNeg) {
        const float deltas[6] = {16.0f, 8.0f, 4.0f, 2.0f, 1.0f, 0.0f};
        for (int k = 0; k < 6; ++k) {
            const float th = __fsub_rn(mn, deltas[k]);
            int c = 0;
            if (in_regs) {
#pragma unroll
                for (int i = 0; i < kPerLane; ++i) c += (lane + 32 * i < blank && v[i] >= th) ? 1 : 0;
            } else {
                for (int w = lane; w < blank; w += 32) c += ld_x<BF16>(row, w) >= th ? 1 : 0;
            }
            c = __reduce_add_sync(0xffffffffu, c);
            if (c <= kCmpList) { thr = th; n = c; break; }
        }
    }
    // collect the listed tokens (index order), then rank them by (D desc, token asc)
    uint64_t mykey = 0;
    if (n > 0) {
        int base = 0;
        auto take = [&](int w, float x) {
            const bool hit = w < blank && x >= thr;
            const unsigned bal = __ballot_sync(0xffffffffu, hit);
            if (hit) {
                const int q = base + __popc(bal & ((1u << lane) - 1u));
                keys[q] = ((uint64_t)ord_of(x) << 32) | (uint64_t)(0xffffffffu - (uint32_t)w);
            }
            base += __popc(bal);
        };
        if (in_regs) {
#pragma unroll
            for (int i = 0; i < kPerLane; ++i) take(lane + 32 * i, v[i]);
        } else {
            for (int w0 = 0; w0 < blank; w0 += 32) take(w0 + lane, w0 + lane < blank ? ld_x<BF16>(row, w0 + lane) : kNeg);
        }
        __syncwarp();
        if (lane < n) {
            mykey = keys[lane];
            int r = 0;
            for (int j = 0; j < n; ++j) r += keys[j] > mykey ? 1 : 0;
            const int w = (int)(0xffffffffu - (uint32_t)mykey);
            float* val = (float*)(rec + 32);
            uint16_t* tok = (uint16_t*)(rec + 160);
            val[r] = dval(score_of(mykey));
            tok[r] = (uint16_t)w;
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
__global__ void __launch_bounds__(32 * kWarps) frame_compact_kernel(const void* __restrict__ X, int64_t sb, int64_t stt,
                                                                   const int64_t* __restrict__ rowoff, int B, int T,
                                                                   int Vp1, uint8_t* __restrict__ cmp) {
    __shared__ uint64_t s_keys[kWarps][kCmpList];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int64_t nrows = __ldg(&rowoff[B]);
    const int64_t nchunks = (nrows + kRowsPerWarp - 1) / kRowsPerWarp;
    const size_t esz = BF16 ? 2 : 4;
    for (int64_t c = (int64_t)blockIdx.x * kWarps + wid; c < nchunks; c += (int64_t)gridDim.x * kWarps) {
        int64_t r = c * kRowsPerWarp;
        // utterance of row r: the last b with rowoff[b] <= r (binary search, L1-resident)
        int lo = 0, hi = B - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (__ldg(&rowoff[mid]) <= r) lo = mid; else hi = mid - 1;
        }
        int b = lo;
        int64_t off = __ldg(&rowoff[b]), end = __ldg(&rowoff[b + 1]);
        const int64_t rend = min(nrows, r + kRowsPerWarp);
        for (; r < rend; ++r) {
            while (r >= end) { ++b; off = end; end = __ldg(&rowoff[b + 1]); }  // skips empty utterances
            const int t = (int)(r - off);
            const char* row = (const char*)X + ((int64_t)b * sb + (int64_t)t * stt) * esz;
            compact_row<BF16>(row, Vp1, cmp + ((int64_t)b * T + t) * kCmpBytes, s_keys[wid], lane);
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
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)nsm * 8));
    cudaStream_t st = (cudaStream_t)stream;
    if (bf16)
        frame_compact_kernel<true><<<grid, 32 * kWarps, 0, st>>>(x, stride_b, stride_t, rowoff, B, T, Vp1, cmp);
    else
        frame_compact_kernel<false><<<grid, 32 * kWarps, 0, st>>>(x, stride_b, stride_t, rowoff, B, T, Vp1, cmp);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { err = cudaGetErrorString(e); return 1; }
    return 0;
}

}  // namespace flexctc
