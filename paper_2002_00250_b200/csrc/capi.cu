// Common C-ABI entry points: errors, version, the device RNG test hook and
// the fused confusion-count epilogue.
#include "common.cuh"

#include <vector>

namespace rgbdseg {

static thread_local char g_last_error[1024] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
    va_end(ap);
}

// Device twin of engine_rng.pixel_rng over a key list (engine_rng.py:36-44):
// exactly the inline functions the PBAS kernel uses.
__global__ void rng_keys_kernel(const uint64_t* __restrict__ keys, int64_t count,
                                double* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t* k = keys + 5 * i;
        out[i] = rng_draw(rng_prefix(k[0], k[1], k[2], k[3]), k[4]);
    }
}

__global__ void rng_stream_kernel(uint64_t seed, uint64_t x, uint64_t y, uint64_t f,
                                  int64_t count, double* __restrict__ out) {
    const uint64_t h = rng_prefix(seed, x, y, f);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = rng_draw(h, (uint64_t)i);
}

// metrics.compare_masks (metrics.py:50-69): fg = mask > 127; labels 1 = fg,
// 0 = bg, 2 = ignore.  Warp-aggregated, one atomic per warp per counter.
__global__ void confusion_kernel(const uint8_t* __restrict__ mask,
                                 const uint8_t* __restrict__ labels, int64_t npix,
                                 unsigned long long* __restrict__ counts) {
    unsigned long long tp = 0, tn = 0, fp = 0, fn = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npix;
         i += (int64_t)gridDim.x * blockDim.x) {
        const bool fg = mask[i] > 127;
        const uint8_t l = labels[i];
        tp += fg && l == 1;
        fn += !fg && l == 1;
        fp += fg && l == 0;
        tn += !fg && l == 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        tp += __shfl_down_sync(0xFFFFFFFFu, tp, o);
        tn += __shfl_down_sync(0xFFFFFFFFu, tn, o);
        fp += __shfl_down_sync(0xFFFFFFFFu, fp, o);
        fn += __shfl_down_sync(0xFFFFFFFFu, fn, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(counts + 0, tp);
        atomicAdd(counts + 1, tn);
        atomicAdd(counts + 2, fp);
        atomicAdd(counts + 3, fn);
    }
}

__global__ void eval_sum_kernel(unsigned long long* __restrict__ slots,
                                long long* __restrict__ counts, int accumulate, int reset) {
    // one warp per counter: lanes stride over the slots, then a warp sum
    const int c = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned long long v = 0;
    for (int i = lane; i < EVAL_SLOTS; i += 32) {
        v += slots[i * 4 + c];
        if (reset) slots[i * 4 + c] = 0ull;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, o);
    if (lane == 0) counts[c] = (accumulate ? counts[c] : 0ll) + (long long)v;
}

int eval_sum_slots(unsigned long long* slots, int64_t* counts_dev, int accumulate, int reset,
                   cudaStream_t st) {
    eval_sum_kernel<<<1, 128, 0, st>>>(slots, reinterpret_cast<long long*>(counts_dev), accumulate,
                                       reset);
    RGBDSEG_LAUNCH_CHECK();
    return RGBDSEG_OK;
}

}  // namespace rgbdseg

using namespace rgbdseg;

extern "C" {

const char* rgbdseg_last_error(void) { return g_last_error; }

int32_t rgbdseg_abi_version(void) { return RGBDSEG_ABI_VERSION; }

int32_t rgbdseg_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int rgbdseg_rng_keys(const uint64_t* keys_host, int64_t count, double* out_host, int32_t device) {
    if (count <= 0) return RGBDSEG_OK;
    if (!keys_host || !out_host) {
        set_error("NULL key/output buffer");
        return RGBDSEG_E_CONFIG;
    }
    DeviceGuard dg(device);
    uint64_t* dk = nullptr;
    double* dout = nullptr;
    RGBDSEG_CUDA_TRY(cudaMalloc(&dk, sizeof(uint64_t) * 5 * count));
    cudaError_t e = cudaMalloc(&dout, sizeof(double) * count);
    if (e == cudaSuccess)
        e = cudaMemcpy(dk, keys_host, sizeof(uint64_t) * 5 * count, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        rng_keys_kernel<<<148, 256>>>(dk, count, dout);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(out_host, dout, sizeof(double) * count, cudaMemcpyDeviceToHost);
    cudaFree(dk);
    if (dout) cudaFree(dout);
    if (e != cudaSuccess) {
        set_error("rgbdseg_rng_keys: %s", cudaGetErrorString(e));
        return RGBDSEG_E_RUNTIME;
    }
    return RGBDSEG_OK;
}

int rgbdseg_rng_stream(uint64_t seed, uint64_t x, uint64_t y, uint64_t frame_idx, int64_t count,
                       double* out_host, int32_t device) {
    if (count <= 0) return RGBDSEG_OK;
    if (!out_host) {
        set_error("NULL output buffer");
        return RGBDSEG_E_CONFIG;
    }
    DeviceGuard dg(device);
    double* dout = nullptr;
    RGBDSEG_CUDA_TRY(cudaMalloc(&dout, sizeof(double) * count));
    rng_stream_kernel<<<296, 256>>>(seed, x, y, frame_idx, count, dout);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpy(out_host, dout, sizeof(double) * count, cudaMemcpyDeviceToHost);
    cudaFree(dout);
    if (e != cudaSuccess) {
        set_error("rgbdseg_rng_stream: %s", cudaGetErrorString(e));
        return RGBDSEG_E_RUNTIME;
    }
    return RGBDSEG_OK;
}

int rgbdseg_confusion_accumulate(const uint8_t* mask_dev, const uint8_t* labels_dev, int64_t npix,
                                 int64_t* counts_dev, void* stream) {
    if (npix <= 0) return RGBDSEG_OK;
    if (!mask_dev || !labels_dev || !counts_dev) {
        set_error("NULL mask/labels/counts");
        return RGBDSEG_E_CONFIG;
    }
    int64_t blocks = (npix + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    confusion_kernel<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        mask_dev, labels_dev, npix, reinterpret_cast<unsigned long long*>(counts_dev));
    RGBDSEG_LAUNCH_CHECK();
    return RGBDSEG_OK;
}

}  // extern "C"
