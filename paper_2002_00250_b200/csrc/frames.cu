// Device-side input staging: the step the reference performs right before the
// hot path (frames.py:46-88, called at engine.py:194-197 and bench.py:91-97):
//   scale_depth_map  d8 = 0 iff d16 == 0, else max(1, (d16 * 255) // 65535)
//   resample_depth   nearest neighbour on pixel centres,
//                    src = min(int((i + 0.5) * src_n / dst_n), src_n - 1) in f64
//   pack_frame       (r, g, b, d8) per pixel
// One thread per output pixel; writes the packed (H, W, 4) frame the GMM/PBAS
// kernels read.  rgb_only callers pass depth16 == NULL (depth byte 0,
// engine.py:199-200).  Exact: integer arithmetic and the same IEEE f64
// expression for the resample index (this TU inherits -fmad=false).
#include "common.cuh"

namespace rgbdseg {

__device__ __forceinline__ uint32_t scale_depth(uint32_t d16) {  // frames.py:46-52
    if (d16 == 0) return 0u;
    const uint32_t d8 = (d16 * 255u) / 65535u;
    return d8 > 1u ? d8 : 1u;
}

__device__ __forceinline__ int nn_index(int i, int src_n, int dst_n) {  // frames.py:86-87
    const double v = ((double)i + 0.5) * (double)src_n / (double)dst_n;
    const int64_t s = (int64_t)v;
    return (int)(s < src_n - 1 ? s : src_n - 1);
}

__global__ void pack_frame_kernel(const uint8_t* __restrict__ rgb, int width, int height,
                                  const uint16_t* __restrict__ depth, int dw, int dh,
                                  uint32_t* __restrict__ frame) {
    const int64_t npix = (int64_t)width * height;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npix;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int y = (int)(p / width), x = (int)(p - (int64_t)y * width);
        uint32_t d8 = 0u;
        if (depth) {
            const int sy = (dh == height) ? y : nn_index(y, dh, height);
            const int sx = (dw == width) ? x : nn_index(x, dw, width);
            d8 = scale_depth(depth[(int64_t)sy * dw + sx]);
        }
        const uint8_t* c = rgb + 3 * p;
        frame[p] = (uint32_t)c[0] | ((uint32_t)c[1] << 8) | ((uint32_t)c[2] << 16) | (d8 << 24);
    }
}

}  // namespace rgbdseg

using namespace rgbdseg;

extern "C" int rgbdseg_pack_frame(const uint8_t* rgb_dev, int32_t width, int32_t height,
                                  const uint16_t* depth16_dev, int32_t depth_w, int32_t depth_h,
                                  uint8_t* frame_dev, void* stream) {
    if (!rgb_dev || !frame_dev) {
        set_error("NULL rgb or frame buffer");
        return RGBDSEG_E_CONFIG;
    }
    if (width <= 0 || height <= 0 || (depth16_dev && (depth_w <= 0 || depth_h <= 0))) {
        set_error("target dimensions must be positive");  // frames.py:80-81
        return RGBDSEG_E_DIMENSION;
    }
    const int64_t npix = (int64_t)width * height;
    int64_t blocks = (npix + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    pack_frame_kernel<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        rgb_dev, width, height, depth16_dev, depth_w, depth_h,
        reinterpret_cast<uint32_t*>(frame_dev));
    RGBDSEG_LAUNCH_CHECK();
    return RGBDSEG_OK;
}

// ------------------------------------------------------------------------
// Opt-in 3x3 median postprocess of a 0/255 mask (north_star "median-filter
// postprocess"; no reference semantics -- SURVEY.md D4 -- so it is off by
// default and pinned to scipy.ndimage.median_filter(size=3, mode="reflect")).
// For a binary mask the median of the 9 values is 255 iff at least 5 are 255.
// Shared-memory tile with a 1-pixel halo; "reflect" mirrors the edge pixel
// (index -1 -> 0, W -> W-1).
namespace rgbdseg {
constexpr int MED_TX = 32, MED_TY = 8;

__device__ __forceinline__ int reflect_idx(int i, int n) {
    return i < 0 ? -i - 1 : (i >= n ? 2 * n - i - 1 : i);
}

__global__ void median3x3_kernel(const uint8_t* __restrict__ in, uint8_t* __restrict__ out,
                                 int width, int height) {
    __shared__ uint8_t tile[MED_TY + 2][MED_TX + 2];
    const int x0 = blockIdx.x * MED_TX, y0 = blockIdx.y * MED_TY;
    for (int i = threadIdx.y * MED_TX + threadIdx.x; i < (MED_TY + 2) * (MED_TX + 2);
         i += MED_TX * MED_TY) {
        const int ty = i / (MED_TX + 2), tx = i - ty * (MED_TX + 2);
        const int gy = reflect_idx(min(max(y0 + ty - 1, -1), height), height);
        const int gx = reflect_idx(min(max(x0 + tx - 1, -1), width), width);
        tile[ty][tx] = in[(int64_t)gy * width + gx] > 127 ? 1 : 0;
    }
    __syncthreads();
    const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
    if (x >= width || y >= height) return;
    int cnt = 0;
#pragma unroll
    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
        for (int dx = 0; dx < 3; ++dx) cnt += tile[threadIdx.y + dy][threadIdx.x + dx];
    out[(int64_t)y * width + x] = cnt >= 5 ? 255 : 0;
}
}  // namespace rgbdseg

extern "C" int rgbdseg_median3x3(const uint8_t* mask_in_dev, uint8_t* mask_out_dev, int32_t width,
                                 int32_t height, void* stream) {
    if (!mask_in_dev || !mask_out_dev || mask_in_dev == mask_out_dev) {
        set_error("median3x3 needs distinct non-NULL input and output masks");
        return RGBDSEG_E_CONFIG;
    }
    if (width <= 0 || height <= 0) {
        set_error("mask dimensions must be positive");
        return RGBDSEG_E_DIMENSION;
    }
    dim3 block(MED_TX, MED_TY), grid((width + MED_TX - 1) / MED_TX, (height + MED_TY - 1) / MED_TY);
    median3x3_kernel<<<grid, block, 0, static_cast<cudaStream_t>(stream)>>>(mask_in_dev, mask_out_dev,
                                                                          width, height);
    RGBDSEG_LAUNCH_CHECK();
    return RGBDSEG_OK;
}
