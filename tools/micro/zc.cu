// Microbenchmark: H2D bandwidth of (a) cudaMemcpyAsync from pinned memory (copy engine) and
// (b) a kernel reading the pinned buffer directly (zero-copy, 16-B loads) into device memory,
// for a 105 MiB buffer (the c4 log-prob tensor). Build: nvcc -O3 -arch=sm_100a zc.cu -o zc
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void gather(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v;
        asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(src + i));
        dst[i] = v;
    }
}

int main() {
    const size_t n = 105ull << 20;
    char *h, *d;
    cudaHostAlloc(&h, n, cudaHostAllocDefault);
    cudaMalloc(&d, n);
    for (size_t i = 0; i < n; i += 4096) h[i] = (char)i;
    char* hd = nullptr;
    cudaError_t e = cudaHostGetDevicePointer((void**)&hd, h, 0);
    printf("{\"hostGetDevicePointer\": \"%s\", \"same_ptr\": %d", cudaGetErrorString(e), hd == h);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e9, ms;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a); cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice); cudaEventRecord(b);
        cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf(", \"memcpy_GBps\": %.1f", n / best / 1e6);
    int configs[][2] = {{148, 256}, {148, 1024}, {296, 512}, {32, 256}, {64, 512}, {16, 1024}};
    for (auto& c : configs) {
        best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a); gather<<<c[0], c[1]>>>((const uint4*)hd, (uint4*)d, n / 16); cudaEventRecord(b);
            cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
        }
        printf(", \"zerocopy_%dx%d_GBps\": %.1f", c[0], c[1], n / best / 1e6);
    }
    printf(", \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
