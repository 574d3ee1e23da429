// Can bulk-async (1D TMA) staging beat K1's 6.55 TB/s for the GMM-7/3 stream?
// Persistent CTAs; per tile of T pixels one thread issues the 20 plane
// segments (7x8 B + 7x32 B + 3x8 B + 3x16 B per pixel) as cp.async.bulk into an
// S-stage shared-memory ring (mbarrier complete_tx); threads consume their
// pixel from shared memory and write 10x8 B + 32 B + 16 B back with STG.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}"
                 ::"r"(smem_u32(b)), "r"(parity) : "memory");
}

struct Planes { char* w; char* r; char* wd; char* rd; size_t P; };
constexpr int PER_PX = 7 * 8 + 7 * 32 + 3 * 8 + 3 * 16;  // 352

template <int T, int S>
__global__ void __launch_bounds__(T) k(Planes pl, int ntiles) {
    extern __shared__ __align__(128) char sm[];
    __shared__ uint64_t bar[S];
    const int tid = threadIdx.x;
    if (tid == 0)
        for (int s = 0; s < S; ++s) mbar_init(&bar[s], 1);
    __syncthreads();
    auto issue = [&](int tile, int st) {
        if (tid != 0 || tile >= ntiles) return;
        char* base = sm + (size_t)st * T * PER_PX;
        mbar_expect(&bar[st], T * PER_PX);
        const size_t p0 = (size_t)tile * T;
        for (int q = 0; q < 7; ++q) bulk_g2s(base + q * T * 8, pl.w + (q * pl.P + p0) * 8, T * 8, &bar[st]);
        for (int q = 0; q < 7; ++q) bulk_g2s(base + 56 * T + q * T * 32, pl.r + (q * pl.P + p0) * 32, T * 32, &bar[st]);
        for (int q = 0; q < 3; ++q) bulk_g2s(base + 280 * T + q * T * 8, pl.wd + (q * pl.P + p0) * 8, T * 8, &bar[st]);
        for (int q = 0; q < 3; ++q) bulk_g2s(base + 304 * T + q * T * 16, pl.rd + (q * pl.P + p0) * 16, T * 16, &bar[st]);
    };
    int k = 0;
    for (int s = 0; s < S; ++s) issue(blockIdx.x + s * gridDim.x, s);
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++k) {
        const int st = k % S;
        mbar_wait(&bar[st], (k / S) & 1);
        const char* base = sm + (size_t)st * T * PER_PX;
        const size_t p = (size_t)tile * T + tid;
        double acc = 0;
        double w[7];
#pragma unroll
        for (int q = 0; q < 7; ++q) {
            w[q] = ((const double*)(base + q * T * 8))[tid];
            const double4 r = ((const double4*)(base + 56 * T + q * T * 32))[tid];
            acc += w[q] * r.x + r.y * r.z - r.w;
        }
        double wd[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            wd[q] = ((const double*)(base + 280 * T + q * T * 8))[tid];
            const double2 r = ((const double2*)(base + 304 * T + q * T * 16))[tid];
            acc += wd[q] * r.x - r.y;
        }
        const double4 r0 = ((const double4*)(base + 56 * T))[tid];
        const double2 d0 = ((const double2*)(base + 304 * T))[tid];
        __syncthreads();  // stage consumed by every thread
        issue(tile + S * gridDim.x, st);
#pragma unroll
        for (int q = 0; q < 7; ++q) ((double*)pl.w)[q * pl.P + p] = w[q] * 0.999 + acc * 1e-9;
#pragma unroll
        for (int q = 0; q < 3; ++q) ((double*)pl.wd)[q * pl.P + p] = wd[q] * 0.999;
        const int m = (int)((p * 2654435761u) % 7), m3 = (int)((p * 40503u) % 3);
        double4 o = r0;
        o.x += acc;
        ((double4*)pl.r)[m * pl.P + p] = o;
        double2 od = d0;
        od.x += acc;
        ((double2*)pl.rd)[m3 * pl.P + p] = od;
    }
}

template <int T, int S>
void run(Planes pl, int ctas_per_sm) {
    const size_t smem = (size_t)T * PER_PX * S;
    cudaFuncSetAttribute(k<T, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int ntiles = (int)(pl.P / T);
    const int grid = sms * ctas_per_sm;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<T, S><<<grid, T, smem>>>(pl, ntiles);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("T=%d S=%d: %s\n", T, S, cudaGetErrorString(e)); return; }
    float best = 1e30f;
    for (int i = 0; i < 6; ++i) {
        cudaEventRecord(a);
        k<T, S><<<grid, T, smem>>>(pl, ntiles);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    const double moved = (double)pl.P * (352 + 80 + 32 + 16);
    printf("T=%4d S=%d ctas/SM=%d smem=%6zu B: %.3f ms  %.0f GB/s\n", T, S, ctas_per_sm, smem, best,
           moved / best / 1e6);
}

int main() {
    Planes pl;
    pl.P = 16588800;  // 8 x 1080p, multiple of 256
    cudaMalloc(&pl.w, pl.P * 7 * 8);
    cudaMalloc(&pl.r, pl.P * 7 * 32);
    cudaMalloc(&pl.wd, pl.P * 3 * 8);
    cudaMalloc(&pl.rd, pl.P * 3 * 16);
    cudaMemset(pl.w, 0, pl.P * 7 * 8);
    cudaMemset(pl.r, 0, pl.P * 7 * 32);
    cudaMemset(pl.wd, 0, pl.P * 3 * 8);
    cudaMemset(pl.rd, 0, pl.P * 3 * 16);
    run<128, 2>(pl, 2);
    run<128, 3>(pl, 1);
    run<64, 3>(pl, 3);
    run<64, 4>(pl, 2);
    run<256, 2>(pl, 1);
    run<32, 4>(pl, 5);
    run<32, 6>(pl, 3);
    return 0;
}
