// Microbenchmark: dependent-chain latency (cycles) of warp-level primitives on sm_100a, one warp
// (or one CTA for the barriers). Each op's output feeds the next op's input; clock64 around N ops.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int N = 1024;

__global__ void k_match64(uint64_t seed, long long* out, uint64_t* sink) {
    uint64_t v = seed + (threadIdx.x & 7);
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) { unsigned m = __match_any_sync(0xffffffffu, v); v += m; }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
    sink[threadIdx.x] = v;
}
__global__ void k_match32(uint32_t seed, long long* out, uint64_t* sink) {
    uint32_t v = seed + (threadIdx.x & 7);
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) { unsigned m = __match_any_sync(0xffffffffu, v); v += m; }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
    sink[threadIdx.x] = v;
}
__global__ void k_match64_distinct(uint64_t seed, long long* out, uint64_t* sink) {
    uint64_t v = seed * 977 + threadIdx.x * 0x9E3779B97F4A7C15ull;
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) { unsigned m = __match_any_sync(0xffffffffu, v); v += (m >> 31); }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
    sink[threadIdx.x] = v;
}
__global__ void k_shfl(uint32_t seed, long long* out, uint64_t* sink) {
    uint32_t v = seed + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) v = __shfl_xor_sync(0xffffffffu, v, 1) + 1;
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
    sink[threadIdx.x] = v;
}
__global__ void k_ballot(uint32_t seed, long long* out, uint64_t* sink) {
    uint32_t v = seed + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) v = __ballot_sync(0xffffffffu, v & 1) + threadIdx.x;
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
    sink[threadIdx.x] = v;
}
__global__ void k_lds(uint32_t seed, long long* out, uint64_t* sink) {
    __shared__ uint32_t s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i + 1) & 1023;
    __syncwarp();
    uint32_t v = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) v = s[v];
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
    sink[threadIdx.x] = v;
}
// smem store by one lane, __syncwarp, load by another lane (the phase-to-phase hand-off)
__global__ void k_sts_sync_lds(uint32_t seed, long long* out, uint64_t* sink) {
    __shared__ uint32_t s[64];
    uint32_t v = seed + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) {
        s[threadIdx.x] = v;
        __syncwarp();
        v = s[(threadIdx.x + 1) & 31] + 1;
        __syncwarp();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
    sink[threadIdx.x] = v;
}
__global__ void k_syncthreads(uint32_t seed, long long* out, uint64_t* sink) {
    __shared__ uint32_t s[256];
    uint32_t v = seed + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) {
        s[threadIdx.x] = v;
        __syncthreads();
        v = s[(threadIdx.x + 32) & 255] + 1;
        __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
    sink[threadIdx.x] = v;
}
__global__ void k_atom(uint32_t seed, long long* out, uint64_t* sink) {
    __shared__ int c;
    if (threadIdx.x == 0) c = 0;
    __syncwarp();
    uint32_t v = seed;
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) v += atomicAdd(&c, (int)(v & 1) + 1);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
    sink[threadIdx.x] = v;
}
__global__ void k_exp64(double seed, long long* out, uint64_t* sink) {
    double v = seed * 1e-3 - 0.5 - threadIdx.x * 1e-4;
    long long t0 = clock64();
    for (int i = 0; i < N / 16; ++i) v = -exp(v) * 0.5;
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (t1 - t0) * 16;
    sink[threadIdx.x] = (uint64_t)__double_as_longlong(v);
}
__global__ void k_log1p64(double seed, long long* out, uint64_t* sink) {
    double v = seed * 1e-3 + 0.5 + threadIdx.x * 1e-4;
    long long t0 = clock64();
    for (int i = 0; i < N / 16; ++i) v = log1p(v) + 0.25;
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (t1 - t0) * 16;
    sink[threadIdx.x] = (uint64_t)__double_as_longlong(v);
}

int main() {
    long long* d;
    uint64_t* sink;
    cudaMalloc(&d, 8);
    cudaMalloc(&sink, 8 * 1024);
    long long h;
#define RUN(name, kern, threads)                                                         \
    kern<<<1, threads>>>(1, d, sink);                                                    \
    kern<<<1, threads>>>(1, d, sink);                                                    \
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);                                        \
    printf("{\"op\": \"%s\", \"cycles_per_op\": %.1f}\n", name, (double)h / N);
    RUN("match.any.b64 (8 groups of 4)", k_match64, 32);
    RUN("match.any.b32 (8 groups of 4)", k_match32, 32);
    RUN("match.any.b64 (32 distinct)", k_match64_distinct, 32);
    RUN("shfl.bfly + iadd", k_shfl, 32);
    RUN("vote.ballot + iadd", k_ballot, 32);
    RUN("lds (pointer chase)", k_lds, 32);
    RUN("sts + syncwarp + lds + syncwarp", k_sts_sync_lds, 32);
    RUN("sts + bar.sync(256) + lds + bar.sync(256)", k_syncthreads, 256);
    RUN("atomicAdd smem (32 lanes, same word, dependent)", k_atom, 32);
    RUN("exp(double) (libdevice)", k_exp64, 32);
    RUN("log1p(double) (libdevice)", k_log1p64, 32);
    cudaError_t e = cudaDeviceSynchronize();
    printf("{\"status\": \"%s\"}\n", cudaGetErrorString(e));
    return 0;
}
