// Shared device/host helpers for the rgbdseg B200 kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <thread>
#include <string>
#include <utility>

#include <nvtx3/nvToolsExt.h>

#include "../../include/rgbdseg_b200.h"

namespace rgbdseg {

// ------------------------------------------------------------ errors -----
void set_error(const char* fmt, ...);

#define RGBDSEG_CUDA_TRY(expr)                                                          \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess) {                                                        \
            ::rgbdseg::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,             \
                                 cudaGetErrorString(_e));                               \
            return RGBDSEG_E_RUNTIME;                                                   \
        }                                                                               \
    } while (0)

#define RGBDSEG_LAUNCH_CHECK()                                                          \
    do {                                                                                \
        cudaError_t _e = cudaGetLastError();                                            \
        if (_e != cudaSuccess) {                                                        \
            ::rgbdseg::set_error("%s:%d kernel launch: %s", __FILE__, __LINE__,         \
                                 cudaGetErrorString(_e));                               \
            return RGBDSEG_E_RUNTIME;                                                   \
        }                                                                               \
    } while (0)

// Scoped device switch (restores the caller's current device).
struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

// ------------------------------------------- fused evaluation epilogue --
// metrics.compare_masks (src/rgbdseg/metrics.py:50-69) folded into K1/K2:
// fg = this pixel's mask decision, label 0 background / 1 foreground /
// 2 ignore (frames.py:27-29; ignore counts nowhere).  Ballot + popc per
// warp, shared-memory sums per block, one 64-bit atomic per counter per
// block into one of EVAL_SLOTS spread slots (no hot address); the slots
// are summed by rgbdseg_eval_sum_slots.  Every thread of the block must call
// it (it synchronises the block).
constexpr int EVAL_SLOTS = 256;

__device__ __forceinline__ void eval_block_accumulate(bool valid, bool fg, uint8_t label,
                                                      unsigned long long* __restrict__ slots) {
    __shared__ unsigned int sc[4];
    if (threadIdx.x < 4) sc[threadIdx.x] = 0u;
    __syncthreads();
    const bool fgl = valid && label == 1, bgl = valid && label == 0;
    const unsigned tp = __ballot_sync(0xFFFFFFFFu, fg && fgl);
    const unsigned tn = __ballot_sync(0xFFFFFFFFu, !fg && bgl);
    const unsigned fp = __ballot_sync(0xFFFFFFFFu, fg && bgl);
    const unsigned fn = __ballot_sync(0xFFFFFFFFu, !fg && fgl);
    if ((threadIdx.x & 31u) == 0) {
        if (tp) atomicAdd(&sc[0], (unsigned)__popc(tp));
        if (tn) atomicAdd(&sc[1], (unsigned)__popc(tn));
        if (fp) atomicAdd(&sc[2], (unsigned)__popc(fp));
        if (fn) atomicAdd(&sc[3], (unsigned)__popc(fn));
    }
    __syncthreads();
    if (threadIdx.x < 4 && sc[threadIdx.x])
        atomicAdd(slots + (size_t)(blockIdx.x & (EVAL_SLOTS - 1)) * 4 + threadIdx.x,
                  (unsigned long long)sc[threadIdx.x]);
}

// Sum the EVAL_SLOTS x 4 slot counters into counts[4] (device, stream-
// ordered; counts += sum when accumulate, else counts = sum) and optionally
// zero the slots.  Defined in capi.cu.
int eval_sum_slots(unsigned long long* slots, int64_t* counts_dev, int accumulate, int reset,
                   cudaStream_t st);

// ------------------------------------------------- cross-stream order --
// A handle's state may be stepped on different streams (its own for host
// buffers, the caller's for device tensors).  Before work on `st`, wait for
// everything the handle's previous step enqueued on another stream: one
// event record + stream wait, nothing when the stream does not change.
inline int order_after(cudaStream_t last, cudaStream_t st, cudaEvent_t ev) {
    if (!last || last == st || !ev) return RGBDSEG_OK;
    RGBDSEG_CUDA_TRY(cudaEventRecord(ev, last));
    RGBDSEG_CUDA_TRY(cudaStreamWaitEvent(st, ev, 0));
    return RGBDSEG_OK;
}

// ------------------------------------------------ host-buffer staging --
// The drop-in host path (process_frame(numpy): engine.py:99-112 returns the
// mask of THIS frame) and the asynchronous submit() path, per handle:
//   * two device slots (frame + mask), so frame t+1's upload (copy-in stream)
//     overlaps frame t's kernels (handle stream) and frame t-1's download
//     (copy-out stream); all ordering by events;
//   * sync: the caller's pageable buffer is copied into a page-locked staging
//     buffer in chunks on the calling thread, each chunk's DMA enqueued as
//     soon as it is staged (host copy of chunk i+1 overlaps the DMA of chunk
//     i), and the mask comes back the same way (DMA of chunk j+1 overlaps the
//     host copy of chunk j) -- no pageable cudaMemcpy (driver bounce
//     buffers, ~19 GB/s) and no hidden synchronisation;
//   * async: the caller's buffers (pinned, alive until sync) are DMA'd
//     directly.
// Two helper threads that stage a caller's pageable frame into page-locked
// memory chunk by chunk (each copies half of every chunk), so the host copy
// runs at two threads' bandwidth and overlaps the calling thread's CUDA API
// calls (the per-chunk DMA / kernel / download enqueues).  Idle helpers spin
// briefly after a frame (back-to-back frames find them awake), then sleep on
// a condition variable.
struct CopyCrew {
    static constexpr int NT = 2;
    std::thread th[NT];
    std::mutex mu;
    std::condition_variable cv;
    std::atomic<uint64_t> gen{0};
    std::atomic<bool> quit{false};
    const uint8_t* src = nullptr;
    uint8_t* dst = nullptr;
    int64_t chunk = 0, total = 0;
    int nchunks = 0;
    std::atomic<uint64_t> done[NT];  // (job generation << 32) | chunks copied
    bool started = false;

    void start() {
        if (started) return;
        for (int t = 0; t < NT; ++t) done[t].store(0);
        for (int t = 0; t < NT; ++t) th[t] = std::thread([this, t] { worker(t); });
        started = true;
    }
    void stop() {
        if (!started) return;
        {
            std::lock_guard<std::mutex> lk(mu);
            quit.store(true);
        }
        cv.notify_all();
        for (int t = 0; t < NT; ++t) th[t].join();
        started = false;
    }
    void worker(int t) {
        uint64_t seen = 0;
        for (;;) {
            for (int spin = 0; spin < 200000 && gen.load(std::memory_order_acquire) == seen &&
                               !quit.load(std::memory_order_relaxed);
                 ++spin) {
            }
            if (gen.load(std::memory_order_acquire) == seen) {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return gen.load(std::memory_order_acquire) != seen || quit.load(); });
            }
            if (quit.load()) return;
            seen = gen.load(std::memory_order_acquire);
            const uint64_t tag = seen << 32;
            // the job's fields, read once: the next post() may rewrite them as
            // soon as this job's last chunk is reported
            const uint8_t* const js = src;
            uint8_t* const jd = dst;
            const int64_t jc = chunk, jt = total;
            const int jn = nchunks;
            for (int c = 0; c < jn; ++c) {
                const int64_t off = c * jc, n = jt - off < jc ? jt - off : jc;
                const int64_t half = (n / NT + 63) / 64 * 64;
                const int64_t o = off + t * half;
                const int64_t m = o >= off + n ? 0 : (off + n - o < half || t == NT - 1 ? off + n - o : half);
                if (m > 0) memcpy(jd + o, js + o, (size_t)m);
                done[t].store(tag | (uint64_t)(c + 1), std::memory_order_release);
            }
        }
    }
    // Stage src[0, total) into dst in `chunk`-byte chunks; returns at once.
    void post(const uint8_t* s, uint8_t* d, int64_t ch, int64_t n) {
        src = s;
        dst = d;
        chunk = ch;
        total = n;
        nchunks = (int)((n + ch - 1) / ch);
        {
            std::lock_guard<std::mutex> lk(mu);
            gen.fetch_add(1, std::memory_order_release);
        }
        cv.notify_all();
    }
    // Chunk c of the latest post() is staged (each helper finished its part).
    void wait_chunk(int c) {
        const uint64_t want = (gen.load(std::memory_order_relaxed) << 32) | (uint64_t)(c + 1);
        for (int t = 0; t < NT; ++t)
            while (done[t].load(std::memory_order_acquire) < want) {
            }
    }
    void wait_all() {
        if (nchunks > 0) wait_chunk(nchunks - 1);
    }
};

struct HostStaging {
    static constexpr int IN_CHUNKS = 8, OUT_CHUNKS = 4, ROW_CHUNKS = 8;
    int64_t in_bytes = 0, out_bytes = 0;
    uint8_t* pin_in = nullptr;
    uint8_t* pin_out = nullptr;
    uint8_t* dev_in[2] = {nullptr, nullptr};
    uint8_t* dev_out[2] = {nullptr, nullptr};
    cudaStream_t s_in = nullptr, s_out = nullptr;
    cudaEvent_t in_ready[2] = {}, step_done[2] = {}, out_done[2] = {}, out_chunk[OUT_CHUNKS] = {};
    cudaEvent_t chunk_in[ROW_CHUNKS + 1] = {}, chunk_step[ROW_CHUNKS + 1] = {},
                chunk_out[ROW_CHUNKS + 1] = {};
    bool used[2] = {false, false};
    int slot = 0;
    // The process-wide helper crew (one pair of threads for every handle, so
    // alternating GMM / PBAS calls keep it awake), held for one call at a
    // time; a concurrent caller copies on its own thread instead.
    CopyCrew* crew = nullptr;
    std::unique_lock<std::mutex> crew_hold;
    static constexpr int64_t CREW_MIN_BYTES = 1 << 20;   // smaller frames copy on the caller
    static constexpr int64_t ROWS_MIN_BYTES = 4 << 20;   // row-chunked device work from here up

    static std::mutex& crew_mutex() {
        static std::mutex m;
        return m;
    }
    static CopyCrew* shared_crew() {
        static CopyCrew* c = [] {
            CopyCrew* k = new (std::nothrow) CopyCrew();
            if (k) k->start();  // never stopped: lives for the process
            return k;
        }();
        return c;
    }
    bool ensure_crew() {
        crew_hold = std::unique_lock<std::mutex>(crew_mutex(), std::try_to_lock);
        crew = crew_hold.owns_lock() ? shared_crew() : nullptr;
        if (!crew && crew_hold.owns_lock()) crew_hold.unlock();
        return crew != nullptr;
    }
    void drop_crew() {
        if (crew) crew->wait_all();  // (error paths) nothing may still write pin_in
        crew = nullptr;
        if (crew_hold.owns_lock()) crew_hold.unlock();
    }
    struct CrewRelease {  // drops the crew when a staging call returns, however it returns
        HostStaging* h;
        ~CrewRelease() { h->drop_crew(); }
    };

    bool ready = false;  // every buffer, event and stream below exists

    int ensure(int64_t ib, int64_t ob) {
        if (ready) return RGBDSEG_OK;
        if (int rc = allocate(ib, ob)) {
            release();  // a partial allocation is not kept
            return rc;
        }
        ready = true;
        return RGBDSEG_OK;
    }
    int allocate(int64_t ib, int64_t ob) {
        in_bytes = ib;
        out_bytes = ob;
        RGBDSEG_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&pin_in), ib, cudaHostAllocDefault));
        RGBDSEG_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&pin_out), ob, cudaHostAllocDefault));
        for (int i = 0; i < 2; ++i) {
            RGBDSEG_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&dev_in[i]), ib));
            RGBDSEG_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&dev_out[i]), ob));
            RGBDSEG_CUDA_TRY(cudaEventCreateWithFlags(&in_ready[i], cudaEventDisableTiming));
            RGBDSEG_CUDA_TRY(cudaEventCreateWithFlags(&step_done[i], cudaEventDisableTiming));
            RGBDSEG_CUDA_TRY(cudaEventCreateWithFlags(&out_done[i], cudaEventDisableTiming));
        }
        for (int j = 0; j < OUT_CHUNKS; ++j)
            RGBDSEG_CUDA_TRY(cudaEventCreateWithFlags(&out_chunk[j], cudaEventDisableTiming));
        for (int j = 0; j <= ROW_CHUNKS; ++j) {
            RGBDSEG_CUDA_TRY(cudaEventCreateWithFlags(&chunk_in[j], cudaEventDisableTiming));
            RGBDSEG_CUDA_TRY(cudaEventCreateWithFlags(&chunk_step[j], cudaEventDisableTiming));
            RGBDSEG_CUDA_TRY(cudaEventCreateWithFlags(&chunk_out[j], cudaEventDisableTiming));
        }
        RGBDSEG_CUDA_TRY(cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking));
        RGBDSEG_CUDA_TRY(cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking));
        return RGBDSEG_OK;
    }

    void release() {
        drop_crew();
        if (s_in) cudaStreamSynchronize(s_in);
        if (s_out) cudaStreamSynchronize(s_out);
        for (int i = 0; i < 2; ++i) {
            if (dev_in[i]) cudaFree(dev_in[i]);
            if (dev_out[i]) cudaFree(dev_out[i]);
            if (in_ready[i]) cudaEventDestroy(in_ready[i]);
            if (step_done[i]) cudaEventDestroy(step_done[i]);
            if (out_done[i]) cudaEventDestroy(out_done[i]);
        }
        for (int j = 0; j < OUT_CHUNKS; ++j)
            if (out_chunk[j]) cudaEventDestroy(out_chunk[j]);
        for (int j = 0; j <= ROW_CHUNKS; ++j) {
            if (chunk_in[j]) cudaEventDestroy(chunk_in[j]);
            if (chunk_step[j]) cudaEventDestroy(chunk_step[j]);
            if (chunk_out[j]) cudaEventDestroy(chunk_out[j]);
        }
        if (pin_in) cudaFreeHost(pin_in);
        if (pin_out) cudaFreeHost(pin_out);
        if (s_in) cudaStreamDestroy(s_in);
        if (s_out) cudaStreamDestroy(s_out);
        *this = HostStaging();
    }

    // One frame: in (in_bytes) -> step(dev frame, dev mask) on `st` -> out
    // (out_bytes).  sync = 1: pageable caller buffers, returns with the mask
    // in `out`; sync = 0: pinned caller buffers, returns after enqueueing.
    template <typename Step>
    int run(const uint8_t* in, uint8_t* out, int sync, cudaStream_t st, Step step) {
        const int k = slot;
        slot ^= 1;
        // the slot's previous frame: its step read dev_in[k] and its
        // download read dev_out[k]
        if (used[k]) {
            RGBDSEG_CUDA_TRY(cudaStreamWaitEvent(s_in, step_done[k], 0));
            RGBDSEG_CUDA_TRY(cudaStreamWaitEvent(st, out_done[k], 0));
        }
        used[k] = true;
        if (sync) {
            // pin_in / pin_out are free: the previous sync call drained them,
            // and async calls never touch them
            const int64_t ch = ((in_bytes + IN_CHUNKS - 1) / IN_CHUNKS + 4095) / 4096 * 4096;  // >= 4096
            const bool helpers = in_bytes >= CREW_MIN_BYTES && ensure_crew();
            CrewRelease release_on_exit{this};  // error returns included
            if (helpers) crew->post(in, pin_in, ch, in_bytes);
            int c = 0;
            for (int64_t off = 0; off < in_bytes; off += ch, ++c) {
                const int64_t n = in_bytes - off < ch ? in_bytes - off : ch;
                if (helpers)
                    crew->wait_chunk(c);
                else
                    memcpy(pin_in + off, in + off, (size_t)n);
                RGBDSEG_CUDA_TRY(cudaMemcpyAsync(dev_in[k] + off, pin_in + off, n,
                                                 cudaMemcpyHostToDevice, s_in));
            }
            if (helpers) drop_crew();
        } else {
            RGBDSEG_CUDA_TRY(cudaMemcpyAsync(dev_in[k], in, in_bytes, cudaMemcpyHostToDevice, s_in));
        }
        RGBDSEG_CUDA_TRY(cudaEventRecord(in_ready[k], s_in));
        RGBDSEG_CUDA_TRY(cudaStreamWaitEvent(st, in_ready[k], 0));
        if (int rc = step(dev_in[k], dev_out[k], st)) return rc;
        RGBDSEG_CUDA_TRY(cudaEventRecord(step_done[k], st));
        RGBDSEG_CUDA_TRY(cudaStreamWaitEvent(s_out, step_done[k], 0));
        if (sync) {
            const int64_t ch = ((out_bytes + OUT_CHUNKS - 1) / OUT_CHUNKS + 4095) / 4096 * 4096;  // >= 4096
            int nch = 0;
            for (int64_t off = 0; off < out_bytes; off += ch, ++nch) {
                const int64_t n = out_bytes - off < ch ? out_bytes - off : ch;
                RGBDSEG_CUDA_TRY(cudaMemcpyAsync(pin_out + off, dev_out[k] + off, n,
                                                 cudaMemcpyDeviceToHost, s_out));
                RGBDSEG_CUDA_TRY(cudaEventRecord(out_chunk[nch], s_out));
            }
            RGBDSEG_CUDA_TRY(cudaEventRecord(out_done[k], s_out));
            nch = 0;
            for (int64_t off = 0; off < out_bytes; off += ch, ++nch) {
                const int64_t n = out_bytes - off < ch ? out_bytes - off : ch;
                RGBDSEG_CUDA_TRY(cudaEventSynchronize(out_chunk[nch]));
                memcpy(out + off, pin_out + off, (size_t)n);
            }
        } else {
            RGBDSEG_CUDA_TRY(cudaMemcpyAsync(out, dev_out[k], out_bytes, cudaMemcpyDeviceToHost, s_out));
            RGBDSEG_CUDA_TRY(cudaEventRecord(out_done[k], s_out));
        }
        return RGBDSEG_OK;
    }

    // The synchronous path with the device work split in row chunks too:
    // chunk i is staged, uploaded, segmented (rows_step on rows [r0, r1))
    // and its mask rows downloaded while the calling thread stages chunk
    // i+1, so the kernels and both DMAs hide under the host copy; finish()
    // runs once after the last chunk (PBAS: the neighbour-update phase).
    // Chunks hold a multiple of `align` rows (PBAS row launches start on
    // 32-pixel boundaries).
    template <typename RowsStep, typename Finish>
    int run_rows(const uint8_t* in, uint8_t* out, cudaStream_t st, int64_t rows, int64_t in_row,
                 int64_t out_row, int64_t align, RowsStep rows_step, Finish finish) {
        const int k = slot;
        slot ^= 1;
        if (used[k]) {
            RGBDSEG_CUDA_TRY(cudaStreamWaitEvent(s_in, step_done[k], 0));
            RGBDSEG_CUDA_TRY(cudaStreamWaitEvent(st, out_done[k], 0));
        }
        used[k] = true;
        int64_t ch = (rows + ROW_CHUNKS - 1) / ROW_CHUNKS;
        ch = (ch + align - 1) / align * align;
        int n = 0, taken = 0;  // chunks enqueued / masks copied out
        auto take = [&](int j) {
            const int64_t r0 = j * ch, r1 = r0 + ch < rows ? r0 + ch : rows;
            memcpy(out + r0 * out_row, pin_out + r0 * out_row, (size_t)((r1 - r0) * out_row));
        };
        const bool helpers = ensure_crew();
        CrewRelease release_on_exit{this};  // error returns included
        if (helpers) crew->post(in, pin_in, ch * in_row, rows * in_row);
        for (int64_t r0 = 0; r0 < rows; r0 += ch, ++n) {
            // masks of finished chunks leave while later chunks still upload
            while (taken < n && cudaEventQuery(chunk_out[taken]) == cudaSuccess) take(taken++);
            const int64_t r1 = r0 + ch < rows ? r0 + ch : rows;
            const int64_t ib = r0 * in_row, in_n = (r1 - r0) * in_row;
            if (helpers)
                crew->wait_chunk(n);
            else
                memcpy(pin_in + ib, in + ib, (size_t)in_n);
            RGBDSEG_CUDA_TRY(cudaMemcpyAsync(dev_in[k] + ib, pin_in + ib, in_n, cudaMemcpyHostToDevice,
                                             s_in));
            RGBDSEG_CUDA_TRY(cudaEventRecord(chunk_in[n], s_in));
            RGBDSEG_CUDA_TRY(cudaStreamWaitEvent(st, chunk_in[n], 0));
            if (int rc = rows_step(dev_in[k], dev_out[k], r0, r1, st)) return rc;
            RGBDSEG_CUDA_TRY(cudaEventRecord(chunk_step[n], st));
            RGBDSEG_CUDA_TRY(cudaStreamWaitEvent(s_out, chunk_step[n], 0));
            const int64_t ob = r0 * out_row, out_n = (r1 - r0) * out_row;
            RGBDSEG_CUDA_TRY(cudaMemcpyAsync(pin_out + ob, dev_out[k] + ob, out_n,
                                             cudaMemcpyDeviceToHost, s_out));
            RGBDSEG_CUDA_TRY(cudaEventRecord(chunk_out[n], s_out));
        }
        if (helpers) drop_crew();
        if (int rc = finish(dev_in[k], dev_out[k], st)) return rc;
        RGBDSEG_CUDA_TRY(cudaEventRecord(step_done[k], st));
        RGBDSEG_CUDA_TRY(cudaEventRecord(out_done[k], s_out));
        for (; taken < n; ++taken) {
            RGBDSEG_CUDA_TRY(cudaEventSynchronize(chunk_out[taken]));
            take(taken);
        }
        return RGBDSEG_OK;  // finish() may still run: later steps are stream-ordered
    }

    // Everything enqueued by run() has finished.
    int drain() {
        if (s_in) RGBDSEG_CUDA_TRY(cudaStreamSynchronize(s_in));
        if (s_out) RGBDSEG_CUDA_TRY(cudaStreamSynchronize(s_out));
        return RGBDSEG_OK;
    }
};

// ------------------------------------------------------------- tracing --
// NVTX range around every C-ABI step (SURVEY.md §5 "tracing"): what an
// nsys / ncu --nvtx capture of a host application groups the K1/K2/K3
// launches under.  Header-only NVTX3: a pointer test when no tool attaches.
#ifndef RGBDSEG_NVTX
#define RGBDSEG_NVTX 1
#endif
struct NvtxRange {
#if RGBDSEG_NVTX
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
#else
    explicit NvtxRange(const char*) {}
#endif
};

// ------------------------------------------ programmatic dependent launch --
// K1, K2 and K3 are launched with programmatic stream serialisation: the
// next kernel of the stream (the next frame's K1, K3 after K2, the next
// frame's K2 after K3) is scheduled into the SMs the previous one's tail
// frees, and waits on the device (griddepcontrol.wait = the previous grid
// completed and its memory is visible) instead of paying a full launch gap.
// Every kernel launched this way calls pdl_enter() before touching memory.
#ifndef RGBDSEG_PDL
#define RGBDSEG_PDL 1
#endif
__device__ __forceinline__ void pdl_enter() {
#if RGBDSEG_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, cudaStream_t st,
                       Args&&... args) {
#if RGBDSEG_PDL
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
#else
    kern<<<grid, block, 0, st>>>(std::forward<Args>(args)...);
#endif
}

// Round a plane length up so every plane of 8/16/32-byte records starts on a
// 256-byte boundary (full-sector, 256-bit-load friendly).
inline int64_t plane_pitch(int64_t npix) { return (npix + 31) / 32 * 32; }

// Granlund-Montgomery unsigned division by a runtime-constant d < 2^31
// (host computes m, l once; exhaustively checked in tests/test_capi.py's
// Python twin).  d == 1 is encoded as l == 0.
struct UDivMagic {
    uint32_t m;
    int32_t l;
};
inline UDivMagic udiv_magic(uint32_t d) {
    if (d <= 1) return {0u, 0};
    int l = 0;
    while ((1ull << l) < d) ++l;
    const uint64_t m = ((1ull << 32) * ((1ull << l) - d)) / d + 1;
    return {(uint32_t)m, l};
}
__device__ __forceinline__ uint32_t udiv(uint32_t n, UDivMagic g) {
    if (g.l == 0) return n;
    const uint32_t t = __umulhi(n, g.m);
    return (t + ((n - t) >> 1)) >> (g.l - 1);
}

// ------------------------------------------------- counter-based RNG -----
// Device twin of engine_rng.py:15-44 (SplitMix64 finalizer chain).  The
// (seed, x, y, frame) prefix is shared by the three draws of a pixel
// (pbas.py:470, :479, :492): 3 + 3 mixes instead of 12.
constexpr uint64_t RNG_SALT = 0x5851F42D4C957F2DULL;
constexpr uint64_t RNG_KX = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t RNG_KY = 0xC2B2AE3D27D4EB4FULL;
constexpr uint64_t RNG_KF = 0x165667B19E3779F9ULL;
constexpr uint64_t RNG_KD = 0xD6E8FEB86659FD93ULL;
constexpr uint64_t RNG_M1 = 0xBF58476D1CE4E5B9ULL;
constexpr uint64_t RNG_M2 = 0x94D049BB133111EBULL;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * RNG_M1;
    z = (z ^ (z >> 27)) * RNG_M2;
    return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t rng_prefix(uint64_t seed, uint64_t x, uint64_t y,
                                                        uint64_t f) {
    uint64_t h = seed ^ RNG_SALT;
    h = mix64(h ^ (x * RNG_KX));
    h = mix64(h ^ (y * RNG_KY));
    return mix64(h ^ (f * RNG_KF));
}

// The first absorption depends on (seed, x) only: a per-column table of it
// (computed once per handle) saves one mix per pixel; identical values.
__host__ __device__ __forceinline__ uint64_t rng_column(uint64_t seed, uint64_t x) {
    return mix64((seed ^ RNG_SALT) ^ (x * RNG_KX));
}
__host__ __device__ __forceinline__ uint64_t rng_prefix_col(uint64_t hcol, uint64_t y, uint64_t f) {
    return mix64(mix64(hcol ^ (y * RNG_KY)) ^ (f * RNG_KF));
}

__host__ __device__ __forceinline__ double rng_draw(uint64_t prefix, uint64_t d) {
    uint64_t h = mix64(prefix ^ (d * RNG_KD));
    return (double)(h >> 11) * (1.0 / 9007199254740992.0);  // exact: (h>>11) < 2^53
}

}  // namespace rgbdseg
