// Peer-memory intent-halo exchange for row bands (BASELINE config 5,
// SURVEY.md §8(e)): one oversized frame split into row bands, one band per
// GPU.  The only cross-band data of PBAS is one row of intent codes per
// boundary per direction (a band's edge rows may ask a pixel of the adjacent
// band to absorb its own value, pbas.py:479-507; the reference applies them
// after every band has classified, engine.py:140-143).
//
// Each band owns a MAILBOX in its own HBM (cudaMalloc, exportable with CUDA
// IPC so a neighbour process maps it over NVLink / NVSwitch):
//
//   [0, 256)     flags: u64 ready[2]    step number of the mail in data[.][side]
//                       u64 consumed[2] step the neighbour has drained from us
//                       u32 error       a wait timed out (set by this band)
//   [256, ...)   data[parity 2][side 2][rowcap]   side 0 = from the band above
//                                                 side 1 = from the band below
//
// push(k)  (after this band's two edge rows are classified): one CTA waits
//          until the target slot (k & 1) of each neighbour was drained
//          (consumed >= k - 2), stores the edge row straight into the
//          neighbour's mailbox with peer stores, fences at system scope and
//          publishes ready = k in the NEIGHBOUR's flags.
// pull(k)  (before apply): one CTA waits for ready >= k in its OWN flags,
//          copies the mail into the intent map's halo rows and tells the
//          senders consumed = k.
//
// No host round trip and no NCCL on the data path; the exchange overlaps
// the interior classify.  Every wait is bounded (timeout -> error flag,
// reported by rgbdseg_halo_link_status) so a lost neighbour cannot hang
// the GPU.
#include "common.cuh"

#include <new>

namespace rgbdseg {

constexpr int64_t LINK_FLAGS = 256;

struct LinkFlags {
    unsigned long long ready[2];
    unsigned long long consumed[2];
    unsigned int error;
};

struct HaloArgs {
    const uint8_t* first_row;  // this band's intent rows
    const uint8_t* last_row;
    uint8_t* halo_above;  // this band's halo rows in its intent map
    uint8_t* halo_below;
    char* mine;  // this band's mailbox
    char* above;  // the neighbours' mailboxes (peer / IPC mapped), NULL at the frame edge
    char* below;
    unsigned long long step;
    int64_t row_bytes, rowcap;
    unsigned long long timeout_ns;
    unsigned int* err_host;  // device alias of the link's host-mapped error word
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Spin until *flag >= want (or the timeout passes: error flag, no hang).
// The error is raised in the mailbox (read by rgbdseg_halo_link_status) and
// in host-mapped memory, which the host polls after every step without a
// device sync (rgbdseg_halo_link_error).
__device__ bool wait_flag(const unsigned long long* flag, unsigned long long want,
                          unsigned long long timeout_ns, unsigned int* err,
                          unsigned int* err_host) {
    if (ld_acquire_sys(flag) >= want) return true;
    const unsigned long long t0 = globaltimer();
    while (ld_acquire_sys(flag) < want) {
        if (globaltimer() - t0 > timeout_ns) {
            atomicExch(err, 1u);
            if (err_host) *reinterpret_cast<volatile unsigned int*>(err_host) = 1u;
            __threadfence_system();
            return false;
        }
        __nanosleep(256);
    }
    return true;
}

__device__ __forceinline__ LinkFlags* flags_of(char* box) { return reinterpret_cast<LinkFlags*>(box); }
__device__ __forceinline__ uint8_t* slot_of(char* box, int parity, int side, int64_t rowcap) {
    return reinterpret_cast<uint8_t*>(box + LINK_FLAGS + ((int64_t)parity * 2 + side) * rowcap);
}

// 16-byte vector copy of one code row (rows are 16-B aligned, rowcap too).
__device__ __forceinline__ void copy_row(uint8_t* dst, const uint8_t* src, int64_t bytes) {
    const int64_t nv = bytes / 16;
    for (int64_t i = threadIdx.x; i < nv; i += blockDim.x)
        reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
    for (int64_t i = nv * 16 + threadIdx.x; i < bytes; i += blockDim.x) dst[i] = src[i];
}

__global__ void __launch_bounds__(512) halo_push_kernel(HaloArgs a) {
    __shared__ int ok;
    LinkFlags* mine = flags_of(a.mine);
    const int parity = (int)(a.step & 1ull);
    if (threadIdx.x == 0) {
        // slot `parity` was last used at step k - 2: wait until it was drained
        const unsigned long long want = a.step >= 2 ? a.step - 2 : 0ull;
        bool good = true;
        if (a.above) good &= wait_flag(&mine->consumed[0], want, a.timeout_ns, &mine->error, a.err_host);
        if (a.below) good &= wait_flag(&mine->consumed[1], want, a.timeout_ns, &mine->error, a.err_host);
        ok = good;
    }
    __syncthreads();
    if (!ok) return;
    // my first row is the band above's "from below" mail, my last row the
    // band below's "from above" mail (peer stores over NVLink)
    if (a.above) copy_row(slot_of(a.above, parity, 1, a.rowcap), a.first_row, a.row_bytes);
    if (a.below) copy_row(slot_of(a.below, parity, 0, a.rowcap), a.last_row, a.row_bytes);
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        if (a.above) st_release_sys(&flags_of(a.above)->ready[1], a.step);
        if (a.below) st_release_sys(&flags_of(a.below)->ready[0], a.step);
    }
}

__global__ void __launch_bounds__(512) halo_pull_kernel(HaloArgs a) {
    __shared__ int ok;
    LinkFlags* mine = flags_of(a.mine);
    const int parity = (int)(a.step & 1ull);
    if (threadIdx.x == 0) {
        bool good = true;
        if (a.above) good &= wait_flag(&mine->ready[0], a.step, a.timeout_ns, &mine->error, a.err_host);
        if (a.below) good &= wait_flag(&mine->ready[1], a.step, a.timeout_ns, &mine->error, a.err_host);
        ok = good;
    }
    __syncthreads();
    if (!ok) {
        // No mail this step: the halo rows must not keep the previous
        // frame's codes (K3 would replay them).  "No intent" everywhere; the
        // error is raised to the host on its next step / status call.
        for (int64_t i = threadIdx.x; i < a.row_bytes; i += blockDim.x) {
            if (a.above) a.halo_above[i] = 0xFFu;
            if (a.below) a.halo_below[i] = 0xFFu;
        }
        return;
    }
    if (a.above) copy_row(a.halo_above, slot_of(a.mine, parity, 0, a.rowcap), a.row_bytes);
    if (a.below) copy_row(a.halo_below, slot_of(a.mine, parity, 1, a.rowcap), a.row_bytes);
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        // drained: the senders may reuse slot `parity` (at step k + 2)
        if (a.above) st_release_sys(&flags_of(a.above)->consumed[1], a.step);
        if (a.below) st_release_sys(&flags_of(a.below)->consumed[0], a.step);
    }
}

}  // namespace rgbdseg

using namespace rgbdseg;

struct rgbdseg_halo_link {
    rgbdseg_pbas* band = nullptr;
    int device = 0;
    char* mine = nullptr;  // own mailbox (cudaMalloc)
    char* above = nullptr;
    char* below = nullptr;
    bool above_ipc = false, below_ipc = false;  // opened with cudaIpcOpenMemHandle
    int64_t row_bytes = 0, rowcap = 0, box_bytes = 0;
    uint8_t *first = nullptr, *last = nullptr, *halo_above = nullptr, *halo_below = nullptr;
    unsigned long long timeout_ns = 20ull * 1000 * 1000 * 1000;
    volatile unsigned int* err_host = nullptr;  // mapped pinned error word
    unsigned int* err_host_dev = nullptr;       // its device alias
};

static_assert(sizeof(cudaIpcMemHandle_t) == RGBDSEG_IPC_HANDLE_BYTES, "IPC handle size");

extern "C" {

int rgbdseg_halo_link_create(rgbdseg_pbas* band, int32_t device, rgbdseg_halo_link** out) {
    if (!band || !out) {
        set_error("NULL band or out pointer");
        return RGBDSEG_E_CONFIG;
    }
    *out = nullptr;
    rgbdseg_halo_link* l = new (std::nothrow) rgbdseg_halo_link();
    if (!l) {
        set_error("out of host memory");
        return RGBDSEG_E_RUNTIME;
    }
    l->band = band;
    l->device = device;
    void *f, *la, *ha, *hb;
    int rc = rgbdseg_pbas_halo_ptrs(band, &f, &la, &ha, &hb, &l->row_bytes);
    if (rc != RGBDSEG_OK) {
        delete l;
        return rc;
    }
    l->first = static_cast<uint8_t*>(f);
    l->last = static_cast<uint8_t*>(la);
    l->halo_above = static_cast<uint8_t*>(ha);
    l->halo_below = static_cast<uint8_t*>(hb);
    l->rowcap = (l->row_bytes + 255) / 256 * 256;
    l->box_bytes = LINK_FLAGS + 4 * l->rowcap;
    DeviceGuard dg(device);
    cudaError_t e = cudaMalloc(&l->mine, (size_t)l->box_bytes);
    if (e == cudaSuccess) e = cudaMemset(l->mine, 0, (size_t)l->box_bytes);
    void* hp = nullptr;
    if (e == cudaSuccess) e = cudaHostAlloc(&hp, sizeof(unsigned int), cudaHostAllocMapped);
    if (e == cudaSuccess) {
        l->err_host = static_cast<volatile unsigned int*>(hp);
        *l->err_host = 0u;
        void* dp = nullptr;
        e = cudaHostGetDevicePointer(&dp, hp, 0);
        l->err_host_dev = static_cast<unsigned int*>(dp);
    }
    if (e != cudaSuccess) {
        set_error("mailbox allocation: %s", cudaGetErrorString(e));
        if (l->mine) cudaFree(l->mine);
        if (l->err_host) cudaFreeHost(const_cast<unsigned int*>(l->err_host));
        delete l;
        return RGBDSEG_E_RUNTIME;
    }
    *out = l;
    return RGBDSEG_OK;
}

int rgbdseg_halo_link_export(rgbdseg_halo_link* l, void* handle_out) {
    if (!l || !handle_out) {
        set_error("NULL link or handle buffer");
        return RGBDSEG_E_CONFIG;
    }
    DeviceGuard dg(l->device);
    RGBDSEG_CUDA_TRY(cudaIpcGetMemHandle(static_cast<cudaIpcMemHandle_t*>(handle_out), l->mine));
    return RGBDSEG_OK;
}

static int open_peer(rgbdseg_halo_link* l, const void* handle, char** dst, bool* ipc) {
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    void* p = nullptr;
    RGBDSEG_CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    *dst = static_cast<char*>(p);
    *ipc = true;
    (void)l;
    return RGBDSEG_OK;
}

static int reset_halos(rgbdseg_halo_link* l) {
    // no neighbour on a side: its halo row stays "no intent" for good
    RGBDSEG_CUDA_TRY(cudaMemset(l->halo_above, 0xFF, (size_t)l->row_bytes));
    RGBDSEG_CUDA_TRY(cudaMemset(l->halo_below, 0xFF, (size_t)l->row_bytes));
    return RGBDSEG_OK;
}

int rgbdseg_halo_link_connect(rgbdseg_halo_link* l, const void* above_handle,
                              const void* below_handle) {
    if (!l) {
        set_error("NULL link");
        return RGBDSEG_E_CONFIG;
    }
    if (l->above || l->below) {
        set_error("halo link already connected");
        return RGBDSEG_E_CONFIG;
    }
    DeviceGuard dg(l->device);
    int rc = reset_halos(l);
    if (rc == RGBDSEG_OK && above_handle) rc = open_peer(l, above_handle, &l->above, &l->above_ipc);
    if (rc == RGBDSEG_OK && below_handle) rc = open_peer(l, below_handle, &l->below, &l->below_ipc);
    return rc;
}

int rgbdseg_halo_link_connect_local(rgbdseg_halo_link* l, rgbdseg_halo_link* above,
                                    rgbdseg_halo_link* below) {
    if (!l) {
        set_error("NULL link");
        return RGBDSEG_E_CONFIG;
    }
    if (l->above || l->below) {
        set_error("halo link already connected");
        return RGBDSEG_E_CONFIG;
    }
    for (rgbdseg_halo_link* p : {above, below}) {
        if (!p) continue;
        if (p->row_bytes != l->row_bytes) {
            set_error("neighbouring bands must have the same width / code size");
            return RGBDSEG_E_DIMENSION;
        }
        if (p->device != l->device) {
            int can = 0;
            cudaDeviceCanAccessPeer(&can, l->device, p->device);
            if (!can) {
                set_error("device %d cannot access device %d's memory", l->device, p->device);
                return RGBDSEG_E_RUNTIME;
            }
            DeviceGuard dg(l->device);
            cudaError_t e = cudaDeviceEnablePeerAccess(p->device, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
                set_error("peer access %d -> %d: %s", l->device, p->device, cudaGetErrorString(e));
                return RGBDSEG_E_RUNTIME;
            }
            cudaGetLastError();
        }
    }
    DeviceGuard dg(l->device);
    int rc = reset_halos(l);
    if (rc != RGBDSEG_OK) return rc;
    l->above = above ? above->mine : nullptr;
    l->below = below ? below->mine : nullptr;
    return RGBDSEG_OK;
}

static HaloArgs args_of(const rgbdseg_halo_link* l, uint64_t step) {
    HaloArgs a;
    a.first_row = l->first;
    a.last_row = l->last;
    a.halo_above = l->halo_above;
    a.halo_below = l->halo_below;
    a.mine = l->mine;
    a.above = l->above;
    a.below = l->below;
    a.step = step;
    a.row_bytes = l->row_bytes;
    a.rowcap = l->rowcap;
    a.timeout_ns = l->timeout_ns;
    a.err_host = l->err_host_dev;
    return a;
}

int rgbdseg_halo_link_push(rgbdseg_halo_link* l, uint64_t step, void* stream) {
    if (!l || step == 0) {
        set_error("NULL link or step 0 (steps count from 1)");
        return RGBDSEG_E_CONFIG;
    }
    if (!l->above && !l->below) return RGBDSEG_OK;
    DeviceGuard dg(l->device);
    NvtxRange nvtx("rgbdseg.halo_push");
    halo_push_kernel<<<1, 512, 0, static_cast<cudaStream_t>(stream)>>>(args_of(l, step));
    RGBDSEG_LAUNCH_CHECK();
    return RGBDSEG_OK;
}

int rgbdseg_halo_link_pull(rgbdseg_halo_link* l, uint64_t step, void* stream) {
    if (!l || step == 0) {
        set_error("NULL link or step 0 (steps count from 1)");
        return RGBDSEG_E_CONFIG;
    }
    if (!l->above && !l->below) return RGBDSEG_OK;
    DeviceGuard dg(l->device);
    NvtxRange nvtx("rgbdseg.halo_pull");
    halo_pull_kernel<<<1, 512, 0, static_cast<cudaStream_t>(stream)>>>(args_of(l, step));
    RGBDSEG_LAUNCH_CHECK();
    return RGBDSEG_OK;
}

int rgbdseg_halo_link_set_timeout(rgbdseg_halo_link* l, uint64_t timeout_ns) {
    if (!l || timeout_ns == 0) {
        set_error("NULL link or zero timeout");
        return RGBDSEG_E_CONFIG;
    }
    l->timeout_ns = timeout_ns;
    return RGBDSEG_OK;
}

int rgbdseg_halo_link_status(rgbdseg_halo_link* l) {
    if (!l) {
        set_error("NULL link");
        return RGBDSEG_E_CONFIG;
    }
    DeviceGuard dg(l->device);
    RGBDSEG_CUDA_TRY(cudaDeviceSynchronize());
    LinkFlags f;
    RGBDSEG_CUDA_TRY(cudaMemcpy(&f, l->mine, sizeof(f), cudaMemcpyDeviceToHost));
    if (f.error) {
        set_error("halo exchange wait timed out (ready %llu/%llu, consumed %llu/%llu)", f.ready[0],
                  f.ready[1], f.consumed[0], f.consumed[1]);
        return RGBDSEG_E_RUNTIME;
    }
    return RGBDSEG_OK;
}

int32_t rgbdseg_halo_link_error(const rgbdseg_halo_link* l) {
    if (!l || !l->err_host) return -1;
    return *l->err_host ? 1 : 0;
}

void rgbdseg_halo_link_destroy(rgbdseg_halo_link* l) {
    if (!l) return;
    DeviceGuard dg(l->device);
    cudaDeviceSynchronize();  // no kernel may still post to the mapped error word
    if (l->err_host) cudaFreeHost(const_cast<unsigned int*>(l->err_host));
    if (l->above_ipc && l->above) cudaIpcCloseMemHandle(l->above);
    if (l->below_ipc && l->below) cudaIpcCloseMemHandle(l->below);
    if (l->mine) cudaFree(l->mine);
    delete l;
}

}  // extern "C"
