/*
 * rgbdseg_b200.h -- C-ABI of the B200-native RGB-D segmentation path.
 *
 * Drop-in for the reference's per-pixel segmentation layer
 * (/root/reference/pkg, citations relative to it).  The reference has no
 * native FFI of its own (it is Python + numba); the boundary it exposes is
 *   - the engine: SegmentationEngine.__init__ / process_frame / state_arrays
 *     (src/rgbdseg/engine.py:60-83, :99-112, :96-97), and
 *   - the per-algorithm "plugin" calls the engine makes:
 *     GmmState.segment_rows   (src/rgbdseg/gmm.py:272-280),
 *     PbasState.segment_rows  (src/rgbdseg/pbas.py:320-333),
 *     PbasState.apply_intents (src/rgbdseg/pbas.py:335-337),
 *     GmmState/PbasState.arrays (gmm.py:251-255, pbas.py:296-303).
 * Each entry point below names the reference interface it replaces.
 *
 * Conventions
 *   - Plain C types only: pointers, sizes, fixed-width integers, doubles.
 *   - Device memory for the model state is owned by the handle (allocated
 *     once at create, like GmmState/PbasState).
 *   - `frame` is packed (H, W, 4) uint8 (r, g, b, d), d == 0 = invalid depth
 *     (frames.py:46-70); `mask` is (H, W) uint8, 0 = background, 255 =
 *     foreground.  *_dev pointers are CUDA device pointers; *_host pointers
 *     are host pointers (pinned memory gives full-speed DMA).
 *   - `stream` is a cudaStream_t passed as void*; NULL means the handle's own
 *     stream.  One frame in flight per handle; handles are not thread-safe
 *     (the service serialises per session: service.py:416-418).
 *   - Return codes map onto the reference's exception classes
 *     (src/rgbdseg/errors.py:4-21):
 *       RGBDSEG_OK 0, RGBDSEG_E_DIMENSION 1 -> DimensionError,
 *       RGBDSEG_E_CONFIG 2 -> ConfigError, RGBDSEG_E_RUNTIME 3 -> RgbdSegError
 *     with a message from rgbdseg_last_error() (thread-local).
 */
#ifndef RGBDSEG_B200_H
#define RGBDSEG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RGBDSEG_OK 0
#define RGBDSEG_E_DIMENSION 1
#define RGBDSEG_E_CONFIG 2
#define RGBDSEG_E_RUNTIME 3

#define RGBDSEG_ABI_VERSION 1

/* GmmParams (src/rgbdseg/gmm.py:37-62).  Validation = GmmParams.validate. */
typedef struct rgbdseg_gmm_params {
    int32_t k_rgb;
    int32_t k_d;
    double alpha;
    double s;
    double tau;
    double match_lambda;
    double var_init;
    double w_init;
} rgbdseg_gmm_params;

/* PbasParams (src/rgbdseg/pbas.py:37-63).  Validation = PbasParams.validate,
 * plus n <= 255 (u8 pos/len state, pbas.py:288-291). */
typedef struct rgbdseg_pbas_params {
    int32_t n;
    int32_t min_matches;
    double r_init;
    double r_lower;
    double r_scale;
    double r_inc_dec;
    double t_init;
    double t_lower;
    double t_upper;
    double t_inc;
    double t_dec;
} rgbdseg_pbas_params;

typedef struct rgbdseg_gmm rgbdseg_gmm;   /* opaque */
typedef struct rgbdseg_pbas rgbdseg_pbas; /* opaque */
typedef struct rgbdseg_halo_link rgbdseg_halo_link; /* opaque */
#define RGBDSEG_IPC_HANDLE_BYTES 64 /* sizeof(cudaIpcMemHandle_t) */

/* State field ids; read/write use the reference layout and dtypes. */
enum {
    RGBDSEG_GMM_RGB_W = 0,   /* (H,W,k_rgb)   f64   gmm.py:244 */
    RGBDSEG_GMM_RGB_MU = 1,  /* (H,W,k_rgb,3) f64   gmm.py:245 */
    RGBDSEG_GMM_RGB_VAR = 2, /* (H,W,k_rgb)   f64   gmm.py:246 */
    RGBDSEG_GMM_D_W = 3,     /* (H,W,k_d)     f64   gmm.py:247 */
    RGBDSEG_GMM_D_MU = 4,    /* (H,W,k_d,1)   f64   gmm.py:248 */
    RGBDSEG_GMM_D_VAR = 5    /* (H,W,k_d)     f64   gmm.py:249 */
};
enum {
    RGBDSEG_PBAS_SAMPLES = 0,  /* (H,W,n,4) u8  pbas.py:285 */
    RGBDSEG_PBAS_DMIN_RGB = 1, /* (H,W,n)   u8  pbas.py:286 */
    RGBDSEG_PBAS_DMIN_D = 2,   /* (H,W,n)   u8  pbas.py:287 */
    RGBDSEG_PBAS_LEN_RGB = 3,  /* (H,W)     u8  pbas.py:288 */
    RGBDSEG_PBAS_POS_RGB = 4,  /* (H,W)     u8  pbas.py:289 */
    RGBDSEG_PBAS_LEN_D = 5,    /* (H,W)     u8  pbas.py:290 */
    RGBDSEG_PBAS_POS_D = 6,    /* (H,W)     u8  pbas.py:291 */
    RGBDSEG_PBAS_R_RGB = 7,    /* (H,W)     f64 pbas.py:292 */
    RGBDSEG_PBAS_R_D = 8,      /* (H,W)     f64 pbas.py:293 */
    RGBDSEG_PBAS_T = 9,        /* (H,W)     f64 pbas.py:294 */
    /* opt-in gradient feature only (rgbdseg_pbas_set_gradient; no reference
     * counterpart): */
    RGBDSEG_PBAS_GSAMPLES = 10,  /* (H,W,n) u8  gradient magnitude of every sample */
    RGBDSEG_PBAS_GRAD_PREV = 11  /* ()      u64 previous frame's magnitude sum (~0: none) */
};

/* ------------------------------------------------------------ common ---- */
const char* rgbdseg_last_error(void);
int32_t rgbdseg_abi_version(void);
/* Number of visible CUDA devices (0 when there is no GPU); never fails. */
int32_t rgbdseg_device_count(void);

/* Device twin of the counter-based RNG, for tests
 * (engine_rng.pixel_rng / rng_stream, src/rgbdseg/engine_rng.py:55-64):
 * out_host[i] = pixel_rng(seed, x, y, frame_idx, i) for i < count, computed
 * by the same __device__ code the PBAS kernel inlines. */
int rgbdseg_rng_stream(uint64_t seed, uint64_t x, uint64_t y, uint64_t frame_idx, int64_t count,
                       double* out_host, int32_t device);
/* Batched draws: out_host[i] = pixel_rng(keys[5i..5i+4]) on the device. */
int rgbdseg_rng_keys(const uint64_t* keys_host, int64_t count, double* out_host, int32_t device);

/* --------------------------------------------------------------- GMM ---- */
/* GmmState(width, height, params) (gmm.py:238-249) + engine setup
 * (engine.py:60-72).  use_depth = (config.mode == "rgbd"). */
int rgbdseg_gmm_create(int32_t width, int32_t height, const rgbdseg_gmm_params* params,
                       int32_t use_depth, int32_t device, rgbdseg_gmm** out);
/* Same, with creation flags (no reference counterpart; 0 == rgbdseg_gmm_create):
 *   RGBDSEG_GMM_STATE_F32  opt-in f32 state storage (SURVEY.md §8(d) "GMM 7/3
 *       f32-storage", 245 instead of 485 B/px at 7/3): loads widen to f64,
 *       the update runs the reference's f64 expressions, stores round to
 *       nearest f32.  Masks / state stay within the north_star tolerance of
 *       the f64 reference (>= 99.99 % of mask pixels, state 1e-5 relative,
 *       tests/test_gmm_f32.py); read/write_state still exchange f64 in the
 *       reference layout (writes round to f32). */
#define RGBDSEG_GMM_STATE_F32 1u
int rgbdseg_gmm_create_ex(int32_t width, int32_t height, const rgbdseg_gmm_params* params,
                          int32_t use_depth, int32_t device, uint32_t flags, rgbdseg_gmm** out);
void rgbdseg_gmm_destroy(rgbdseg_gmm* h);

/* One frame, device buffers: GmmState.segment_rows over all rows
 * (gmm.py:272-280 -> _gmm_band gmm.py:350-368).  Enqueued on `stream`. */
int rgbdseg_gmm_step(rgbdseg_gmm* h, const uint8_t* frame_dev, uint8_t* mask_dev, void* stream);

/* Multi-camera batching: one launch advances `count` independent handles
 * (same k_rgb/k_d/use_depth/device).  The reference has no multi-stream
 * scheduler; this is the B200 grid over (stream, pixel). */
int rgbdseg_gmm_step_batch(rgbdseg_gmm* const* hs, int32_t count, const uint8_t* const* frames_dev,
                           uint8_t* const* masks_dev, void* stream);

/* SegmentationEngine.process_frame with host buffers (engine.py:99-112):
 * H2D of the frame, the step, D2H of the mask, on the handle's stream.
 * sync != 0 waits for completion; sync == 0 returns after enqueueing (the
 * caller must keep both host buffers alive until rgbdseg_gmm_sync). */
int rgbdseg_gmm_process_host(rgbdseg_gmm* h, const uint8_t* frame_host, uint8_t* mask_host,
                             int32_t sync);
int rgbdseg_gmm_sync(rgbdseg_gmm* h);

/* state_arrays()[field] (gmm.py:251-255), reference layout, synchronous. */
int64_t rgbdseg_gmm_state_bytes(const rgbdseg_gmm* h, int32_t field);
int rgbdseg_gmm_read_state(rgbdseg_gmm* h, int32_t field, void* host_dst, int64_t bytes);
int rgbdseg_gmm_write_state(rgbdseg_gmm* h, int32_t field, const void* host_src, int64_t bytes);
/* The handle's own CUDA stream (cudaStream_t as void*). */
void* rgbdseg_gmm_stream(rgbdseg_gmm* h);

/* -------------------------------------------------------------- PBAS ---- */
/* PbasState(width, height, params) (pbas.py:279-294) + engine setup
 * (engine.py:60-78).  seed = config.seed as u64 (engine.py:127). */
int rgbdseg_pbas_create(int32_t width, int32_t height, const rgbdseg_pbas_params* params,
                        int32_t use_depth, uint64_t seed, int32_t device, rgbdseg_pbas** out);
/* Row band [y0, y1) of a (width x height) frame: the multi-GPU split of one
 * oversized frame (engine.py:48-50 bands, one per GPU).  RNG keys and
 * neighbour bounds use GLOBAL coordinates (pbas.py:470-500). */
int rgbdseg_pbas_create_band(int32_t width, int32_t height, int32_t y0, int32_t y1,
                             const rgbdseg_pbas_params* params, int32_t use_depth, uint64_t seed,
                             int32_t device, rgbdseg_pbas** out);
void rgbdseg_pbas_destroy(rgbdseg_pbas* h);

/* One full frame = classify (PbasState.segment_rows, pbas.py:320-333) +
 * intent application (PbasState.apply_intents, pbas.py:335-337), then
 * frame_idx += 1 (engine.py:111).  frame_dev covers the handle's rows. */
int rgbdseg_pbas_step(rgbdseg_pbas* h, const uint8_t* frame_dev, uint8_t* mask_dev, void* stream);
/* The two phases separately, for row bands: classify emits this band's
 * intent codes (own rows + which neighbour + slot); the caller then moves
 * the edge rows into the neighbours' halos (rgbdseg_pbas_halo_ptrs) and
 * calls apply, which pulls every intent targeting this band's pixels and
 * advances frame_idx. */
int rgbdseg_pbas_classify(rgbdseg_pbas* h, const uint8_t* frame_dev, uint8_t* mask_dev,
                          void* stream);
int rgbdseg_pbas_apply(rgbdseg_pbas* h, const uint8_t* frame_dev, void* stream);
/* Classify only band rows [row0, row1) (same frame, same frame_idx): lets a
 * row band classify its two edge rows first and overlap the halo exchange
 * with the interior.  Every row must be classified before apply. */
int rgbdseg_pbas_classify_rows(rgbdseg_pbas* h, const uint8_t* frame_dev, uint8_t* mask_dev,
                               int32_t row0, int32_t row1, void* stream);
/* Copy the band's first/last intent-code rows out (device to device, W codes
 * each; NULL skips), and set the halo rows from the neighbours' copies (NULL
 * = no neighbour: "no intent").  Stream-ordered. */
int rgbdseg_pbas_copy_edges(rgbdseg_pbas* h, void* first_dst, void* last_dst, void* stream);
int rgbdseg_pbas_set_halos(rgbdseg_pbas* h, const void* above_src, const void* below_src,
                           void* stream);
/* Device pointers of the intent rows: the band's first/last own rows and
 * the halo rows above/below it; each row is row_bytes long.  Halo rows hold
 * "no intent" unless the caller fills them between classify and apply. */
int rgbdseg_pbas_halo_ptrs(rgbdseg_pbas* h, void** first_row, void** last_row, void** halo_above,
                           void** halo_below, int64_t* row_bytes);
/* Peer-memory halo exchange between row bands on different GPUs (SURVEY.md
 * §8(e); replaces the reference's in-process band loop, engine.py:126-143,
 * whose sequential intent phase _apply_intents, pbas.py:511-522, sees every
 * band's intents).  Each band owns a mailbox in its HBM; neighbours map it
 * with CUDA IPC (one process per GPU) or directly (same process) and push
 * their edge intent rows into it with peer stores, synchronised by device
 * flags -- no host round trip, no NCCL.  Per frame, steps counted from 1:
 *   classify_rows(edge rows) -> push(step) -> classify_rows(interior)
 *   -> pull(step) -> apply.
 * Waits are bounded (default 20 s): a timeout sets an error flag that
 * status() reports (RGBDSEG_E_RUNTIME) instead of hanging the GPU; the pull
 * then leaves "no intent" in the halo rows (never the previous frame's
 * codes).  error() reads the same flag from host-mapped memory without a
 * device sync (1 = a wait timed out, 0 = none so far, -1 = NULL link): the
 * Python band step polls it every frame. */
int rgbdseg_halo_link_create(rgbdseg_pbas* band, int32_t device, rgbdseg_halo_link** out);
int rgbdseg_halo_link_export(rgbdseg_halo_link* l, void* ipc_handle_out /* IPC_HANDLE_BYTES */);
/* Map the neighbours' exported mailboxes (NULL: no band above / below). */
int rgbdseg_halo_link_connect(rgbdseg_halo_link* l, const void* above_handle,
                              const void* below_handle);
/* Same, for neighbour bands owned by this process (same or peer device). */
int rgbdseg_halo_link_connect_local(rgbdseg_halo_link* l, rgbdseg_halo_link* above,
                                    rgbdseg_halo_link* below);
int rgbdseg_halo_link_push(rgbdseg_halo_link* l, uint64_t step, void* stream);
int rgbdseg_halo_link_pull(rgbdseg_halo_link* l, uint64_t step, void* stream);
int rgbdseg_halo_link_set_timeout(rgbdseg_halo_link* l, uint64_t timeout_ns);
int rgbdseg_halo_link_status(rgbdseg_halo_link* l);
int32_t rgbdseg_halo_link_error(const rgbdseg_halo_link* l);
void rgbdseg_halo_link_destroy(rgbdseg_halo_link* l);
/* Opt-in PBAS gradient-magnitude feature (no reference counterpart: the
 * reference drops the original PBAS gradient term; semantics in
 * DESIGN.md §3 "K2G", CPU checker oracle_pbas_frame_g).  Switched before the
 * first frame of a single-band handle: enable = 1 with alpha >= 0 (sample
 * distance 256 dist + w |g - g_i| against 256 R, w = min(65535, floor(alpha *
 * 256 / max(mean g of the previous frame, 1) + 0.5))) and mean_init > 0 (the
 * mean before the first frame); enable = 0 returns to
 * the reference algorithm.  Adds state fields RGBDSEG_PBAS_GSAMPLES and
 * RGBDSEG_PBAS_GRAD_PREV. */
int rgbdseg_pbas_set_gradient(rgbdseg_pbas* h, int32_t enable, double alpha, double mean_init);
/* K2 variant (performance only; every variant gives the same result):
 * 0 auto (default) -- small frames (a whole single-band batch whose grid
 * fits on the GPU at once) run K2 + K3 as ONE cooperative launch; larger ones
 * run the row kernel while few pixels emit neighbour updates and the warp-strip
 * kernel (in-strip updates applied inside K2) once many do, chosen from the
 * update count K3 posts each frame; 1 always rows; 2 always strips (a
 * single-band handle with width % 32 == 0); 3 fused whenever the step is
 * eligible, else auto; 4 auto without the fused launch (rows / strips by
 * the update rate).  get returns the variant of the
 * latest step in auto mode when it ran fused (3), else the one the next step
 * will use (1 rows, 2 strips).  Results are identical in every variant. */
int rgbdseg_pbas_set_k2_mode(rgbdseg_pbas* h, int32_t mode);
int32_t rgbdseg_pbas_get_k2_mode(const rgbdseg_pbas* h);
int rgbdseg_pbas_step_batch(rgbdseg_pbas* const* hs, int32_t count,
                            const uint8_t* const* frames_dev, uint8_t* const* masks_dev,
                            void* stream);
int rgbdseg_pbas_process_host(rgbdseg_pbas* h, const uint8_t* frame_host, uint8_t* mask_host,
                              int32_t sync);
int rgbdseg_pbas_sync(rgbdseg_pbas* h);
uint64_t rgbdseg_pbas_get_frame_idx(const rgbdseg_pbas* h);
int rgbdseg_pbas_set_frame_idx(rgbdseg_pbas* h, uint64_t frame_idx);
int64_t rgbdseg_pbas_state_bytes(const rgbdseg_pbas* h, int32_t field);
int rgbdseg_pbas_read_state(rgbdseg_pbas* h, int32_t field, void* host_dst, int64_t bytes);
int rgbdseg_pbas_write_state(rgbdseg_pbas* h, int32_t field, const void* host_src, int64_t bytes);
void* rgbdseg_pbas_stream(rgbdseg_pbas* h);

/* Device self-test of K2's divide without the IEEE slow-path branch
 * (csrc/pbas.cu fdiv_rn) against `/`: *mismatches = number of i with
 * bitwise-different quotients a_dev[i] / b_dev[i] (synchronous). */
int rgbdseg_selftest_fdiv(const double* a_dev, const double* b_dev, int64_t n,
                          int64_t* mismatches);

/* Fused evaluation epilogue: metrics.compare_masks (src/rgbdseg/metrics.py:50-69)
 * inside K1/K2.  set_eval(h, labels_dev) makes the following steps compare
 * each pixel's decision with labels_dev (H*W u8 of the handle's rows:
 * 0 background, 1 foreground, 2 ignore; frames.py:27-29) and accumulate
 * TP/TN/FP/FN on the device; NULL turns it off.  eval_counts writes (or with
 * accumulate=1 adds) the pooled counts {tp, tn, fp, fn} (aggregate_sequence's
 * pooling, metrics.py:89-101) into counts_dev[4] (int64, device) on `stream`
 * and, with reset=1, restarts the pool.  Stream-ordered, no host sync. */
int rgbdseg_gmm_set_eval(rgbdseg_gmm* h, const uint8_t* labels_dev);
int rgbdseg_gmm_eval_counts(rgbdseg_gmm* h, int64_t* counts_dev, int32_t accumulate, int32_t reset,
                            void* stream);
int rgbdseg_pbas_set_eval(rgbdseg_pbas* h, const uint8_t* labels_dev);
int rgbdseg_pbas_eval_counts(rgbdseg_pbas* h, int64_t* counts_dev, int32_t accumulate,
                             int32_t reset, void* stream);

/* ------------------------------------------------- input staging ------ */
/* frames.scale_depth_map + resample_depth + pack_frame (src/rgbdseg/frames.py:46-88)
 * on the device: rgb (H,W,3) u8 and depth16 (depth_h, depth_w) u16 (nearest-
 * neighbour resampled to (H,W) when the sizes differ; NULL = rgb_only, depth
 * byte 0, engine.py:199-200) -> packed frame (H,W,4) u8.  Bit-exact. */
int rgbdseg_pack_frame(const uint8_t* rgb_dev, int32_t width, int32_t height,
                       const uint16_t* depth16_dev, int32_t depth_w, int32_t depth_h,
                       uint8_t* frame_dev, void* stream);

/* Opt-in 3x3 median postprocess of a 0/255 mask (north_star; no reference
 * semantics, default off): scipy.ndimage.median_filter(size=3,
 * mode="reflect") on the device.  Input and output must differ. */
int rgbdseg_median3x3(const uint8_t* mask_in_dev, uint8_t* mask_out_dev, int32_t width,
                      int32_t height, void* stream);

/* ---------------------------------------------------- evaluation ------- */
/* Confusion counts of a device mask against a device ground-truth label
 * plane (0 bg / 1 fg / 2 ignore; frames.py:27-29), accumulated into
 * counts_dev[4] = {tp, tn, fp, fn} (int64): metrics.compare_masks
 * (src/rgbdseg/metrics.py:50-69) fused on the device. */
int rgbdseg_confusion_accumulate(const uint8_t* mask_dev, const uint8_t* labels_dev, int64_t npix,
                                 int64_t* counts_dev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RGBDSEG_B200_H */
