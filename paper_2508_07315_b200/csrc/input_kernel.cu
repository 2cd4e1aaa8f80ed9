// Input side: log-softmax of bf16 logits, reading R25.
//
// The frame loop is latency-bound, so the normalisation is NOT fused into it (measured: doing it
// in the helper warps per frame made c4 2.25 -> 2.78 ms, the helpers arrived late at B0). It runs
// as one bandwidth-bound pass before the decode instead: one CTA per 8 consecutive frames of one
// utterance, one warp per row (t < L_b only; padding is never read, R16). Per row: m = max over the
// bf16 values (exact in fp32), S = sum exp(x - m) in fp64, lse = m + log(S) in fp64 (every lane
// the same value), D = (float)(x - lse) written as a dense fp32 row. R25 fixes this arithmetic;
// the fp64 sum runs in a different order than the oracle's (~1e-16 relative), so the fp32 outputs
// agree except at a rounding boundary. When |m| <= 700 the same lse is log(sum exp(x)) with the
// exp of every bf16 value read from a table (bf16_exp_table) instead of evaluated.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>

#include "device_common.cuh"
#include "flexctc_internal.h"

namespace flexctc {
namespace {

using namespace dev;

constexpr int kRows = 8;      // frames (warps) per CTA
constexpr int kPerLane = 33;  // register-resident elements per lane at V' <= 1056

__global__ void __launch_bounds__(32 * kRows) log_softmax_bf16_kernel(const uint16_t* __restrict__ X, int64_t sb,
                                                                     int64_t st, const int32_t* __restrict__ lengths,
                                                                     int B, int T, int Vp1, float* __restrict__ out,
                                                                     int t0, int t1, const double* __restrict__ etab) {
    const int lane = threadIdx.x & 31;
    const int nchunk = (t1 - t0 + kRows - 1) / kRows;
    const int b = blockIdx.x / nchunk;
    const int t = t0 + (blockIdx.x - b * nchunk) * kRows + (threadIdx.x >> 5);
    const int L = min(max(__ldg(&lengths[b]), 0), T);
    if (t >= L || t >= t1) return;
    const uint16_t* x = X + (int64_t)b * sb + (int64_t)t * st;
    float* d = out + ((int64_t)b * T + t) * Vp1;
    if (Vp1 <= 32 * kPerLane) {  // the row in registers: one read of HBM
        float v[kPerLane];
#pragma unroll
        for (int i = 0; i < kPerLane; ++i) {
            const int w = lane + 32 * i;
            v[i] = w < Vp1 ? bf16f(__ldcs(x + w)) : -INFINITY;
        }
        float m = v[0];
#pragma unroll
        for (int i = 1; i < kPerLane; ++i) m = fmaxf(m, v[i]);
#pragma unroll
        for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        double S = 0.0;
        double lse;
        if (etab && m >= -700.0f && m <= 700.0f) {  // log Σ exp(x) from the table (no fp64 exp)
#pragma unroll
            for (int i = 0; i < kPerLane; ++i)
                if (lane + 32 * i < Vp1) S += __ldg(&etab[__float_as_uint(v[i]) >> 16]);
#pragma unroll
            for (int o = 16; o; o >>= 1) S += __shfl_xor_sync(0xffffffffu, S, o);
            lse = log(S);
        } else {
#pragma unroll
            for (int i = 0; i < kPerLane; ++i)
                if (lane + 32 * i < Vp1) S += exp((double)v[i] - (double)m);
#pragma unroll
            for (int o = 16; o; o >>= 1) S += __shfl_xor_sync(0xffffffffu, S, o);
            lse = (double)m + log(S);
        }
#pragma unroll
        for (int i = 0; i < kPerLane; ++i) {
            const int w = lane + 32 * i;
            if (w < Vp1) d[w] = (float)((double)v[i] - lse);
        }
        return;
    }
    // larger vocabularies: three passes over the row (L2-resident after the first)
    float m = -INFINITY;
    for (int w = lane; w < Vp1; w += 32) m = fmaxf(m, bf16f(x[w]));
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    double S = 0.0;
    for (int w = lane; w < Vp1; w += 32) S += exp((double)bf16f(x[w]) - (double)m);
#pragma unroll
    for (int o = 16; o; o >>= 1) S += __shfl_xor_sync(0xffffffffu, S, o);
    const double lse = (double)m + log(S);
    for (int w = lane; w < Vp1; w += 32) d[w] = (float)((double)bf16f(x[w]) - lse);
}

// Streamed host input (flexctc_decode_host): frames [t0, min(L_b, t1)) of n utterances (b =
// order[i], or i) from the
// caller's pinned host buffer (device-mapped: the loads travel over PCIe) to the same offsets of
// the device copy. One CTA per utterance in turn; the byte range of an utterance's chunk is
// contiguous and has the same alignment on both sides (both bases are 16-B aligned and the
// layouts are identical), so it moves as 16-B loads/stores with <= 15 bytes each side done by
// bytes. A few CTAs reach the PCIe rate (~51 GB/s measured with 16 x 1024 threads,
// tools/micro/zc.cu), so the gather runs next to the persistent beam kernel.
__global__ void __launch_bounds__(256) gather_rows_kernel(const char* __restrict__ src, char* __restrict__ dst,
                                                         const int32_t* __restrict__ lengths,
                                                         const int32_t* __restrict__ order, int n, int T,
                                                         int64_t row_bytes, int t0, int t1) {
    for (int i = blockIdx.x; i < n; i += gridDim.x) {
        const int b = order ? __ldg(&order[i]) : i;
        const int L = min(max(__ldg(&lengths[b]), 0), T);
        const int te = min(L, t1);
        if (te <= t0) continue;
        const int64_t lo = ((int64_t)b * T + t0) * row_bytes, hi = ((int64_t)b * T + te) * row_bytes;
        const int64_t a0 = (lo + 15) & ~(int64_t)15, a1 = hi & ~(int64_t)15;
        if (a0 >= a1) {
            for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) dst[i] = src[i];
            continue;
        }
        for (int64_t i = lo + threadIdx.x; i < a0; i += blockDim.x) dst[i] = src[i];
        for (int64_t i = a1 + threadIdx.x; i < hi; i += blockDim.x) dst[i] = src[i];
        const uint4* s4 = (const uint4*)(src + a0);
        uint4* d4 = (uint4*)(dst + a0);
        const int64_t n4 = (a1 - a0) >> 4;
        for (int64_t i = threadIdx.x; i < n4; i += blockDim.x) {
            uint4 v;
            asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(s4 + i));
            d4[i] = v;
        }
    }
}

}  // namespace

int preload_gather_rows() {
    cudaFuncAttributes a{};
    return cudaFuncGetAttributes(&a, gather_rows_kernel) == cudaSuccess ? 0 : 1;
}

int launch_gather_rows(const void* src_dev, void* dst, const int32_t* lengths, const int32_t* order, int n, int T,
                       int64_t row_bytes, int t0, int t1, int ctas, void* stream, std::string& err) {
    if (n <= 0 || t1 <= t0) return 0;
    gather_rows_kernel<<<std::max(1, std::min(n, ctas)), 256, 0, (cudaStream_t)stream>>>(
        (const char*)src_dev, (char*)dst, lengths, order, n, T, row_bytes, t0, t1);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { err = cudaGetErrorString(e); return 1; }
    return 0;
}

// CUDA loads a kernel's module lazily on its first launch, and that load waits for running
// kernels: launched next to a persistent kernel that waits for its output, the first launch
// would deadlock. decode_host_bf16 calls this before the persistent kernel starts.
int preload_log_softmax_bf16() {
    cudaFuncAttributes a{};
    return cudaFuncGetAttributes(&a, log_softmax_bf16_kernel) == cudaSuccess ? 0 : 1;
}

int launch_log_softmax_bf16(const uint16_t* x, int64_t stride_b, int64_t stride_t, const int32_t* lengths, int B,
                            int T, int Vp1, float* out, void* stream, std::string& err, int t0, int t1) {
    if (t1 < 0) t1 = T;
    if (t1 <= t0) return 0;
    const int64_t grid = (int64_t)B * ((t1 - t0 + kRows - 1) / kRows);
    if (grid == 0) return 0;
    if (grid > 0x7fffffff) { err = "B * T too large"; return 2; }
    log_softmax_bf16_kernel<<<(int)grid, 32 * kRows, 0, (cudaStream_t)stream>>>(x, stride_b, stride_t, lengths, B, T,
                                                                                 Vp1, out, t0, t1, bf16_exp_table(stream));
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { err = cudaGetErrorString(e); return 1; }
    return 0;
}

}  // namespace flexctc
