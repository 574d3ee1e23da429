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
