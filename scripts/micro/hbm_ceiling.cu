// HBM ceiling microbenchmark on this B200: pure read, 1:1 copy and a
// GMM-shaped 3:1 read:write stream (K1 moves 5.9 GB read + 2.1 GB written
// per launch), 128-bit and 256-bit accesses, grid-stride, CUDA-event timed.
#include <cstdio>
#include <cuda_runtime.h>

struct alignas(32) v8 { unsigned x[8]; };

template <typename V>
__global__ void rd(const V* __restrict__ a, size_t n, unsigned* sink) {
    unsigned acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        V v = a[i];
        const unsigned* u = reinterpret_cast<const unsigned*>(&v);
#pragma unroll
        for (int k = 0; k < (int)(sizeof(V) / 4); ++k) acc ^= u[k];
    }
    if (acc == 0x12345678u) *sink = acc;
}
template <typename V>
__global__ void cp(const V* __restrict__ a, V* __restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        b[i] = a[i];
}
// 3 reads : 1 write
template <typename V>
__global__ void r3w1(const V* __restrict__ a, V* __restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        V x = a[i], y = a[i + n], z = a[i + 2 * n];
        unsigned* ux = reinterpret_cast<unsigned*>(&x);
        const unsigned* uy = reinterpret_cast<const unsigned*>(&y);
        const unsigned* uz = reinterpret_cast<const unsigned*>(&z);
#pragma unroll
        for (int k = 0; k < (int)(sizeof(V) / 4); ++k) ux[k] ^= uy[k] ^ uz[k];
        b[i] = x;
    }
}

template <typename F>
float timeit(F f) {
    cudaEvent_t s, e;
    cudaEventCreate(&s); cudaEventCreate(&e);
    f(); cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
        cudaEventRecord(s); f(); cudaEventRecord(e); cudaEventSynchronize(e);
        float ms; cudaEventElapsedTime(&ms, s, e); if (ms < best) best = ms;
    }
    return best;
}

int main() {
    const size_t bytes = 8ull << 30;
    char *a, *b; unsigned* sink;
    cudaMalloc(&a, bytes); cudaMalloc(&b, bytes); cudaMalloc(&sink, 4);
    cudaMemset(a, 1, bytes); cudaMemset(b, 2, bytes);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int per : {4, 8, 16}) {
        const int grid = sms * per;
        {
            size_t n = bytes / 16;
            float ms = timeit([&] { rd<uint4><<<grid, 256>>>((const uint4*)a, n, sink); });
            printf("blocks/SM %2d read    128b: %7.1f GB/s\n", per, bytes / ms / 1e6);
            size_t n2 = bytes / 32;
            ms = timeit([&] { rd<v8><<<grid, 256>>>((const v8*)a, n2, sink); });
            printf("blocks/SM %2d read    256b: %7.1f GB/s\n", per, bytes / ms / 1e6);
        }
        {
            size_t half = bytes / 2;
            float ms = timeit([&] { cp<uint4><<<grid, 256>>>((const uint4*)a, (uint4*)b, half / 16); });
            printf("blocks/SM %2d copy    128b: %7.1f GB/s (r+w)\n", per, 2.0 * half / ms / 1e6);
            ms = timeit([&] { cp<v8><<<grid, 256>>>((const v8*)a, (v8*)b, half / 32); });
            printf("blocks/SM %2d copy    256b: %7.1f GB/s (r+w)\n", per, 2.0 * half / ms / 1e6);
        }
        {
            size_t q = bytes / 4;  // 3 read streams of q bytes, 1 written
            float ms = timeit([&] { r3w1<uint4><<<grid, 256>>>((const uint4*)a, (uint4*)b, q / 16); });
            printf("blocks/SM %2d r3w1    128b: %7.1f GB/s (r+w)\n", per, 4.0 * q / ms / 1e6);
            ms = timeit([&] { r3w1<v8><<<grid, 256>>>((const v8*)a, (v8*)b, q / 32); });
            printf("blocks/SM %2d r3w1    256b: %7.1f GB/s (r+w)\n", per, 4.0 * q / ms / 1e6);
        }
    }
    return 0;
}
