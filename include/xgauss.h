/*
 * xgauss.h - C ABI of the B200-native DRR engine (libxgauss.so, sm_100a).
 *
 * Plain C: device pointers, sizes, POD structs and cudaStream_t (passed as
 * void*).  No torch / C++ types cross this boundary.  Every entry point is
 * stream-ordered, allocates nothing (caller-provided buffers and workspace)
 * and returns an xg_status.  Data-dependent failures that the reference
 * raises as exceptions (degenerate covariance, zero quaternion, non-finite
 * features / gradients, entry-buffer overflow) are recorded as bits of a
 * device status word (counters[XG_CTR_STATUS]) so that no entry point has
 * to synchronise; the host maps them to the reference's exception classes.
 *
 * Reference interfaces replaced (paths relative to /root/reference):
 *   xg_preprocess_fwd   pkg/src/xsplat/rasterizer/frontend.py:104-158
 *                       (project_splats: projection, cull, cov2D, conic,
 *                       radius, tile rect) + gaussians.py:110-124,222-232
 *   xg_bin_sort         frontend.py:160-173 (duplicate, np.lexsort by
 *                       (tile, depth, index), np.searchsorted tile ranges)
 *   xg_composite_fwd    rasterizer/_kernels.pyx:23-74 forward_tiles
 *   xg_forward_tiles    rasterizer/_kernels.pyx:23-32 - the reference's own
 *                       kernel-backend signature (backend.py:20-46)
 *   xg_composite_bwd    rasterizer/_kernels.pyx:77-178 backward_tiles, with
 *                       the L1 pixel gradient of trainer.py:117-121 fused
 *   xg_backward_tiles   rasterizer/_kernels.pyx:77-87 - kernel-backend signature
 *   xg_preprocess_bwd   rasterizer/backward.py:61-158 (+ trainer.py:185-188
 *                       DensifyStats.accumulate fused)
 *   xg_adam             trainer.py:147-170 adam_step (+ gaussians.py:234-235)
 *   xg_densify_mark     trainer.py:206-225 densify masks and counts
 *   xg_densify_apply    trainer.py:227-261 compaction, clone shift, split
 *   xg_intensities      gaussians.py:230-232 GaussianCloud.intensities
 *   xg_view_invariants  gaussians.py:47-69, 222-228 (covariance, opacity)
 *   xg_project_volume   phantom.py:181-250 project_phantom (cone-beam ray march
 *                       of a voxel phantom: the training-target generator)
 *   xg_ssim             metrics.py:57-124 ssim / ssim_and_gradient, fused into
 *                       the trainer.py:109-123 loss gradient for gamma > 0
 */
#ifndef XGAUSS_H
#define XGAUSS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define XG_ABI_VERSION 5

typedef enum xg_status {
  XG_OK = 0,
  XG_ERR_INVALID = 1,    /* bad argument (null pointer, size)          */
  XG_ERR_CUDA = 2,       /* CUDA launch / runtime failure              */
  XG_ERR_WORKSPACE = 3   /* caller workspace smaller than required     */
} xg_status;

/* Device status word bits (counters[XG_CTR_STATUS]). */
#define XG_ST_ZERO_QUAT        0x1u  /* InvalidParameterError  gaussians.py:56-57  */
#define XG_ST_DEGENERATE       0x2u  /* NumericalDegeneracyError frontend.py:134-136 */
#define XG_ST_NONFINITE_FEAT   0x4u  /* InvalidParameterError  gaussians.py:122-123 */
#define XG_ST_ENTRY_OVERFLOW   0x8u  /* entry_capacity too small: re-run larger */
#define XG_ST_GRAD_NONFINITE_SHIFT 8 /* bits 8..12: non-finite gradient per field
                                        positions, rotations, log_scales,
                                        raw_opacities, features (trainer.py:160-162) */
#define XG_ST_PEER_TIMEOUT     0x10u /* a peer-exchange wait timed out (xg_peer_*) */

/* counters[] layout (uint32, device). */
#define XG_CTR_ACTIVE   0   /* splats surviving near-plane + on-screen cull  */
#define XG_CTR_ENTRIES  1   /* (tile, splat) entries (may exceed capacity)    */
#define XG_CTR_STATUS   2   /* status bits above                              */
#define XG_CTR_TOUCH    3   /* scratch                                        */
#define XG_CTR_STICKY   4   /* caller-owned; the library only ORs gradient
                               flags into it (xg_preprocess_bwd), never clears */
#define XG_CTR_QUEUE    5   /* tile work-queue head of the compositing kernels */
#define XG_CTR_ITEMS    6   /* chunk count of the checkpointed reverse replay  */
#define XG_CTR_L1       8   /* words 8-9: a double, zeroed by xg_preprocess_fwd:
                               pass (double*)(counters + XG_CTR_L1) as the
                               forward's l1_sum (no separate clearing)      */
#define XG_NCOUNTERS    10  /* (the buffer must be 8-byte aligned)           */

/* Blend constants (rasterizer/kernels_py.py:13-19, frontend.py:36,
 * gaussians.py:26, geometry.py:41). */
#define XG_TILE_SIZE 16
#define XG_POWER_CUTOFF (-30.0)
#define XG_TRANSMITTANCE_FLOOR 1e-4
#define XG_SIGMA_CLAMP 0.99
#define XG_CUTOFF_SIGMA 7.5
#define XG_COV2_LOWPASS 0.3

/* One view (geometry.py:166-192): world->camera rotation (row-major) and
 * translation of the 4x4 extrinsic, pixel focal length, principal point,
 * near plane (0.01 * L_SO) and detector size.  All float64, as the
 * reference's matrices. */
typedef struct xg_camera {
  double rot[9];
  double trans[3];
  double focal;
  double cx, cy;
  double near_plane;
  int32_t width, height;
} xg_camera;

/* A Gaussian cloud: one flat float32 buffer
 *   [positions N*3 | rotations N*4 (w,x,y,z) | log_scales N*3 |
 *    raw_opacities N | features N*F]
 * plus basis_weights[F] (gaussians.py:154-193). */
typedef struct xg_cloud {
  const float* params;
  const float* basis;
  int64_t n;
  int32_t n_features;
  int32_t _pad;
  const float* intensities;  /* optional [N] sigmoid(F . lambda) from xg_intensities: the
                                projection copies (or, when xg_splats.inten points at this
                                very buffer, just uses) it instead of recomputing the
                                view-independent intensity per view - the non-finite
                                feature check is then xg_intensities' */
  const double* invariants;  /* optional [N][8] from xg_view_invariants: Sigma3 (xx xy xz yy
                                yz zz), opacity, zero-quaternion flag - the view-independent
                                part of the projection, computed once per cloud by the same
                                code, so every per-view output stays bit-identical */
} xg_cloud;

/* Per-view screen-space buffers.  Per-Gaussian arrays are indexed by cloud
 * row (culled rows have n_tiles == 0 and are never referenced). */
typedef struct xg_splats {
  double*   mean2d;       /* [N][2] projected mean, pixels                  */
  float*    coef;         /* [N][4] A2,B2,C2,alpha: log2-density coefficients
                             p2 = A2 dx^2 + B2 dx dy + C2 dy^2 (= power*log2 e)
                             and opacity                                     */
  float*    inten;        /* [N]    intensity sigmoid(F . lambda)           */
  uint16_t* rect;         /* [N][4] tile rect tx0,ty0,tx1,ty1 (inclusive)   */
  uint32_t* n_tiles;      /* [N]    tiles covered (0 = culled)              */
  uint64_t* depth_key;    /* [N]    float64 bits of t_z (all ones if culled) */
  uint32_t* order;        /* [N]    Gaussians sorted by (depth, index)      */
  uint32_t* entry_splat;  /* [entry_capacity] Gaussian per (tile, splat) entry,
                             sorted by (tile, depth, index)                  */
  int64_t*  tile_ranges;  /* [n_tiles_x*n_tiles_y][2] [start, end)          */
  uint32_t* counters;     /* [XG_NCOUNTERS]                                 */
  int64_t   n;
  int64_t   entry_capacity;
  int32_t*  tile_order;   /* [n_tiles_x*n_tiles_y] tiles by descending entry
                             count (compositing schedule; written by
                             xg_bin_sort)                                   */
  int32_t*  unit_cost;    /* [4*n_tiles] entries each 8x8 quarter-tile's
                             reverse replay walks (written by
                             xg_composite_fwd; optional)                    */
  int32_t*  unit_order;   /* [4*n_tiles] quarter-tiles by descending
                             unit_cost (reverse-replay schedule; scratch)   */
  /* Optional replay checkpoints (training frames).  When replay_ckpt is set,
   * a tracking xg_composite_fwd stores every pixel's (T, acc) before each
   * XG_REPLAY_CHUNK-th entry of its tile, and xg_composite_bwd (given
   * unit_cost and the forward's image) splits every tile's reverse replay
   * into independent XG_REPLAY_CHUNK-entry chunks.  Both calls must see the
   * same buffers. */
  float*    replay_ckpt;  /* [replay_slots][256][2]                          */
  uint32_t* replay_items; /* [4*replay_slots][2] chunk list (scratch)        */
  int64_t   replay_slots; /* >= xg_replay_slots(entry_capacity, n_tiles)     */
} xg_splats;

/* Optional float64 API outputs of the projection (frontend.py:58-74); any
 * pointer may be NULL.  All [N]-row, written for active rows only. */
typedef struct xg_splat_extras {
  double* cov2d;   /* [N][3] xx, xy, yy of the low-pass-filtered covariance */
  double* conic;   /* [N][3] its inverse                                    */
  double* depth;   /* [N]                                                   */
  double* t_cam;   /* [N][3]                                                */
  double* radius;  /* [N]                                                   */
  double* opacity; /* [N]                                                   */
} xg_splat_extras;

int32_t xg_abi_version(void);
const char* xg_last_error(void);
/* Running count of kernels this library has launched (process-wide). */
uint64_t xg_kernel_launches(void);

/* Tile grid of a camera. */
int32_t xg_tiles_x(const xg_camera* cam);
int32_t xg_tiles_y(const xg_camera* cam);

/* Checkpoint slots a view with entry_capacity entries over n_tiles tiles
 * needs (xg_splats.replay_slots): entry_capacity / XG_REPLAY_CHUNK + n_tiles + 1. */
#ifndef XG_REPLAY_CHUNK
#define XG_REPLAY_CHUNK 256 /* (a power of two >= 32; tuning builds may override) */
#endif
int64_t xg_replay_slots(int64_t entry_capacity, int32_t n_tiles_total);

/* Scratch bytes needed by xg_bin_sort. */
size_t xg_bin_workspace_bytes(int64_t n, int64_t entry_capacity, int32_t n_tiles_total);

/* K1: per-Gaussian projection (float64 arithmetic), writes mean2d, coef,
 * inten, rect, n_tiles, depth_key, counters[ACTIVE], status bits.
 * Resets counters[0..3] first (counters[4] is left to the caller).
 * extras may be NULL. */
xg_status xg_preprocess_fwd(const xg_cloud* cloud, const xg_camera* cam, xg_splats* sp,
                            const xg_splat_extras* extras, void* stream);

/* K2: depth sort (stable radix over the float64 bits of t_z, index
 * tie-break: the reference's exact order, frontend.py:169), tile
 * duplication (exclusive scan), stable radix sort by tile, tile ranges.
 * Fills order, entry_splat, tile_ranges, tile_order, counters[ENTRIES]. */
xg_status xg_bin_sort(const xg_camera* cam, xg_splats* sp, void* workspace, size_t workspace_bytes,
                      void* stream);

/* K3: front-to-back compositing.  Writes image[H][W], t_final[H][W] (final
 * transmittance) and n_contrib[H][W] (1 + index of the last blended entry
 * relative to the tile start, 0 if none).  If target != NULL also
 * accumulates sum |image - target| into *l1_sum (double, device). */
xg_status xg_composite_fwd(const xg_camera* cam, const xg_splats* sp, float* image, float* t_final,
                           int32_t* n_contrib, const float* target, double* l1_sum, void* stream);

/* Training forward: as the tracking xg_composite_fwd (t_final, checkpoints,
 * fused L1) for a following xg_composite_bwd, but n_contrib is the reverse
 * replay's start rather than the reference's contributor count: exact for a
 * pixel whose transmittance fell below the floor, the tile list's length for
 * a pixel still above it (the entries in between have power < -30).  Its
 * speculative batches take the image-only step (opacity in the exponent), so
 * image, t_final and the following xg_composite_bwd's gradients agree with
 * the xg_composite_fwd path to float32 rounding.  Replaces, for the trainer,
 * the same _kernels.pyx:23-74 forward as xg_composite_fwd. */
xg_status xg_composite_fwd_train(const xg_camera* cam, const xg_splats* sp, float* image, float* t_final,
                                 int32_t* n_contrib, const float* target, double* l1_sum, void* stream);

/* K3 over a batch of binned views that share the detector size (image only,
 * e.g. a novel-view sweep): ONE persistent launch with one heaviest-first
 * queue over every (view, tile, quarter) unit, so per-view tails overlap.
 * images[i] is a device pointer to view i's [H][W] output (the array itself
 * is host memory); 1 <= n_views <= XG_MAX_BATCH.  An overflowed view
 * (counters[ENTRIES] > entry_capacity) is skipped.  workspace >=
 * xg_composite_batch_workspace_bytes(cams, n_views). */
#define XG_MAX_BATCH 16
size_t xg_composite_batch_workspace_bytes(const xg_camera* cam, int32_t n_views);
xg_status xg_composite_fwd_batch(const xg_camera* cams, const xg_splats* sps, float* const* images,
                                 int32_t n_views, void* workspace, size_t workspace_bytes, void* stream);

/* K4a: reverse replay.  Per-pixel upstream gradient is dl_dimage[H][W], or,
 * when dl_dimage == NULL, the fused L1 gradient l1_scale*sign(image-target).
 * image (the forward's output) is also what the checkpointed replay
 * (xg_splats.replay_ckpt) restarts each chunk from; without it, or without
 * checkpoints, every quarter-tile is replayed whole from t_final.
 * Accumulates (atomically) into grad_acc[N][8]:
 *   {sum G dx, sum G dy, sum G dx^2, sum G dx dy, sum G dy^2, sum g w, sum G, 0}
 * over (pixel, entry) pairs, dx = px - mx, w = sigma T, g = dL/dI,
 * G = dL/dsigma * sigma on unclamped pairs (= the reference's g_power).
 * grad_acc ([N][8], caller-allocated) is zeroed here first (a memset on the
 * stream: no caller-side clearing launch). */
xg_status xg_composite_bwd(const xg_camera* cam, const xg_splats* sp, const float* t_final,
                           const int32_t* n_contrib, const float* dl_dimage, const float* image,
                           const float* target, float l1_scale, float* grad_acc, void* stream);

/* The trainer's K3 + K4a pair (_kernels.pyx:23-74 forward, :77-178 backward
 * with the fused L1 gradient l1_scale*sign(image-target)): the results of
 * xg_composite_fwd_train followed by xg_composite_bwd(dl_dimage = NULL), as
 * one stream segment in which the reverse replay starts on each tile as soon
 * as that tile's forward is done (the forward publishes every finished
 * tile's replay chunks to a device ring, the replay kernel - launched with
 * programmatic dependent launch - consumes them).  Needs a training frame
 * (replay_ckpt, replay_items, unit_cost); target and grad_acc are required,
 * grad_acc is zeroed here.  Uses counters 5-7.  Falls back to the two calls
 * when the build's tiling does not allow it (or XG_TRAIN_STREAM=0). */
xg_status xg_composite_train_pair(const xg_camera* cam, const xg_splats* sp, float* image, float* t_final,
                                  int32_t* n_contrib, const float* target, double* l1_sum, float l1_scale,
                                  float* grad_acc, void* stream);

/* Reproducible K4a (the reference's single-threaded backward is bitwise
 * reproducible, pkg/tests/test_trainer.py:336-353): the same reverse replay,
 * but each (splat, tile) sum - written by exactly one warp - is STORED into
 * the splat's own slot for that tile (slots of splat g: an exclusive scan of
 * n_tiles, one per tile of its rectangle, row-major), and
 * xg_reduce_entry_grads writes grad_acc[N][8] by adding each splat's slots
 * in order.  entry_ws: xg_entry_grad_bytes(n, entry_capacity) bytes of
 * caller scratch (zeroed / scanned here).  Needs the checkpointed replay (a
 * tracking forward with replay_ckpt / replay_items / unit_cost, and image).
 * Same numbers as xg_composite_bwd up to the summation order, identical run
 * to run. */
size_t xg_entry_grad_bytes(int64_t n_splats, int64_t entry_capacity);
xg_status xg_composite_bwd_entries(const xg_camera* cam, const xg_splats* sp, const float* t_final,
                                   const int32_t* n_contrib, const float* dl_dimage, const float* image,
                                   const float* target, float l1_scale, void* entry_ws, size_t entry_ws_bytes,
                                   void* stream);
xg_status xg_reduce_entry_grads(const xg_camera* cam, const xg_splats* sp, const void* entry_ws,
                                size_t entry_ws_bytes, float* grad_acc, void* stream);

/* K4b: chain rule to every cloud field (float64 arithmetic).  Writes
 * grads (flat, same layout as params; zero rows for culled Gaussians),
 * screen_norms[N], visible[N]; flags non-finite fields in the status word
 * and ORs the same flags into counters[XG_CTR_STICKY].
 * If norm_sum/obs_count/world_grad_sum are non-NULL they are accumulated
 * (DensifyStats.accumulate, trainer.py:185-188).  g_mean_out / g_conic_out /
 * g_int_out / g_alpha_out (optional, [N][2],[N][3],[N],[N] float64) receive
 * the reference's kernel-level gradients (backward_tiles outputs). */
xg_status xg_preprocess_bwd(const xg_cloud* cloud, const xg_camera* cam, const xg_splats* sp,
                            const float* grad_acc, float* grads, float* screen_norms,
                            uint8_t* visible, float* norm_sum, int32_t* obs_count,
                            float* world_grad_sum, double* g_mean_out, double* g_conic_out,
                            double* g_int_out, double* g_alpha_out, void* stream);

/* Finite check of a flat gradient buffer: sets status bit 8+f for every
 * field f holding a NaN/Inf. */
xg_status xg_check_finite(const float* grads, int64_t n, int32_t n_features, uint32_t* counters,
                          void* stream);
/* Same over flat elements [elem_begin, elem_end) (one gradient bucket). */
xg_status xg_check_finite_range(const float* grads, int64_t n, int32_t n_features, int64_t elem_begin,
                                int64_t elem_end, uint32_t* counters, void* stream);

/* K4c: fused Adam over all fields + quaternion renormalisation, in place.
 * lr[5] per field (positions, rotations, log_scales, raw_opacities,
 * features).  bc1 = 1-beta1^t, bc2 = 1-beta2^t.  Honours the non-finite bits
 * in the device word *status (if non-NULL) with the reference's
 * partial-update semantics: fields before the first non-finite one are
 * updated, the rest (and the renorm) are not.  lr is HOST memory. */
xg_status xg_adam(float* params, const float* grads, float* exp_avg, float* exp_avg_sq,
                  int64_t n, int32_t n_features, const double* lr, double beta1, double beta2,
                  double eps, double bc1, double bc2, const uint32_t* status, void* stream);

/* The two halves of xg_adam: the element-wise update restricted to flat
 * elements [elem_begin, elem_end) (one gradient bucket, so data-parallel
 * training can update bucket i while bucket i+1 is being all-reduced), and
 * the quaternion renormalisation (after every bucket is done). */
xg_status xg_adam_range(float* params, const float* grads, float* exp_avg, float* exp_avg_sq,
                        int64_t n, int32_t n_features, const double* lr, double beta1, double beta2,
                        double eps, double bc1, double bc2, const uint32_t* status,
                        int64_t elem_begin, int64_t elem_end, void* stream);
xg_status xg_adam_renorm(float* params, int64_t n, int32_t n_features, const uint32_t* status,
                         void* stream);

/* K5: the data-parallel step's gradient exchange fused with Adam, over peer
 * memory (one process per GPU, each rank's buffers mapped into every process
 * by CUDA IPC; parallel.PeerExchange).  Replaces the bucketed NCCL
 * all-reduce + xg_adam_range of parallel.DataParallelTrainer
 * (trainer.py:158-170 semantics on the SUMMED gradient):
 *   xg_peer_reduce_scatter  signal ready, wait for every rank, sum slice
 *     `rank` of the flat gradient over the ranks in rank order (peer loads)
 *     into xbuf[rank] (epoch parity half), publish its per-field non-finite
 *     bits to every rank, signal arrived;
 *   xg_peer_allgather_adam  wait for every rank's arrival, read each slice
 *     from its owner (peer loads) and apply Adam to the whole buffer (the
 *     arithmetic of xg_adam_range), honouring the global non-finite bits;
 *     the quaternion renorm follows with xg_adam_renorm(sticky).
 * Slice length: xg_peer_slice (multiple of 4); xbuf[k] holds 2 slices,
 * sync[k] 8 zero-initialised words.  epoch = 1, 2, ... (one per exchange).
 * Waits are bounded (~10 s): a timeout ORs XG_ST_PEER_TIMEOUT into *sticky.
 * Every rank adds the same values in the same order: bit-identical replicas. */
#define XG_PEER_MAX 8
typedef struct xg_peer_group {
  int32_t rank, world;
  uint32_t epoch;
  const float* grads[XG_PEER_MAX];  /* each rank's flat gradient (peer-mapped) */
  float* xbuf[XG_PEER_MAX];         /* each rank's exchange buffer, 2 x slice  */
  uint32_t* sync[XG_PEER_MAX];      /* each rank's 8 sync words                */
} xg_peer_group;
int64_t xg_peer_slice(int64_t n, int32_t n_features, int32_t world);
xg_status xg_peer_reduce_scatter(const xg_peer_group* pg, int64_t n, int32_t n_features, uint32_t* sticky,
                                 void* stream);
xg_status xg_peer_allgather_adam(const xg_peer_group* pg, float* params, float* exp_avg, float* exp_avg_sq,
                                 int64_t n, int32_t n_features, const double* lr, double beta1, double beta2,
                                 double eps, double bc1, double bc2, uint32_t* sticky, void* stream);

/* K4d (1): density-control masks.  flags[N] bit0 high-gradient, bit1 large,
 * bit2 prune, bit3 clone, bit4 split; counts[4] = {prune, clone, split, keep}
 * (counts zeroed by the callee). */
xg_status xg_densify_mark(const float* params, int64_t n, int32_t n_features,
                          const float* norm_sum, const int32_t* obs_count, double grad_threshold,
                          double size_threshold, double prune_opacity, uint8_t* flags,
                          uint32_t* counts, void* stream);

/* K4d (2): compaction into new buffers laid out [keep | clone | split x2]
 * (trainer.py:227-261).  allow_growth = 0 drops clone/split (cap reached).
 * split_normals: [n_split][2][3] float64 standard normals (host PCG64 draw,
 * uploaded).  new_params / new_exp_avg / new_exp_avg_sq sized n_new rows;
 * moments of new rows are zeroed.  scratch: xg_densify_scratch_bytes(n). */
size_t xg_densify_scratch_bytes(int64_t n);
xg_status xg_densify_apply(const float* params, const float* exp_avg, const float* exp_avg_sq,
                           int64_t n, int32_t n_features, const uint8_t* flags,
                           const float* world_grad_sum, const double* split_normals,
                           double log_split_factor, int32_t allow_growth, float* new_params,
                           float* new_exp_avg, float* new_exp_avg_sq, int64_t n_new,
                           uint32_t* scratch, void* stream);

/* sigmoid(F . lambda) for all N (float32 out); flags non-finite features. */
xg_status xg_intensities(const xg_cloud* cloud, float* out, uint32_t* counters, void* stream);

/* View-independent projection terms for all N (float64 out[N][8], see
 * xg_cloud.invariants): R(q/|q|) diag(e^s) squared (gaussians.py:47-69,
 * frontend.py:126-128) and sigmoid(raw opacity) (gaussians.py:222-228).
 * A sweep over a static cloud computes them once instead of per view. */
xg_status xg_view_invariants(const xg_cloud* cloud, double* out, void* stream);

/* The reference kernel-backend contract (_kernels.pyx:23-32, 77-87) on
 * device buffers: n_splats active rows with float64 means2d[A][2],
 * conics[A][3], intensities[A], opacities[A]; entry_splat[E] (row indices),
 * tile_ranges[T][2].  image out float64 [h][w].  workspace >=
 * xg_tiles_workspace_bytes(n_splats, h, w). */
size_t xg_tiles_workspace_bytes(int64_t n_splats, int32_t h, int32_t w);
xg_status xg_forward_tiles(int32_t h, int32_t w, const double* means2d, const double* conics,
                           const double* intensities, const double* opacities,
                           const int32_t* entry_splat, int64_t n_entries,
                           const int64_t* tile_ranges, int64_t n_splats, double* image,
                           void* workspace, size_t workspace_bytes, void* stream);
xg_status xg_backward_tiles(int32_t h, int32_t w, const double* means2d, const double* conics,
                            const double* intensities, const double* opacities,
                            const int32_t* entry_splat, int64_t n_entries,
                            const int64_t* tile_ranges, int64_t n_splats, const double* dl_dimage,
                            double* g_mean, double* g_conic, double* g_int, double* g_alpha,
                            void* workspace, size_t workspace_bytes, void* stream);

/* The same contract at the reference's precision: float64 arithmetic in
 * _kernels.pyx's operation order (compiled without FMA contraction), for the
 * "cuda" kernel backend registered in xsplat itself
 * (paper_2403_04116_b200/rasterizer/xsplat_backend.py).  Replaces
 * rasterizer/_kernels.pyx:23-74 (forward_tiles) and :77-178
 * (backward_tiles) one for one; all arrays device-resident, outputs zeroed
 * here, no workspace. */
xg_status xg_forward_tiles_f64(int32_t h, int32_t w, const double* means2d, const double* conics,
                               const double* intensities, const double* opacities, const int32_t* entry_splat,
                               int64_t n_entries, const int64_t* tile_ranges, int64_t n_splats, double* image,
                               void* stream);
xg_status xg_backward_tiles_f64(int32_t h, int32_t w, const double* means2d, const double* conics,
                                const double* intensities, const double* opacities, const int32_t* entry_splat,
                                int64_t n_entries, const int64_t* tile_ranges, int64_t n_splats,
                                const double* dl_dimage, double* g_mean, double* g_conic, double* g_int,
                                double* g_alpha, void* stream);

/* A voxel phantom (phantom.py:117-140): float64 densities [m0][m1][m2]
 * (C order; axes = world x, y, z), centred on the world origin. */
typedef struct xg_volume {
  const double* densities;
  int32_t m[3];
  int32_t _pad;
  double voxel_size[3];  /* mm per voxel, per axis */
} xg_volume;

/* One cone-beam view for the projector (phantom.py:193-213): source
 * position, world->camera rotation R (row-major; ray directions are
 * d_cam @ R, d_cam = ((x - W/2) / f, (y - H/2) / f, 1)), focal length in
 * pixels, detector size.  Host-computed (math.sin / math.cos). */
typedef struct xg_cone_view {
  double source[3];
  double rot[9];
  double focal;
  int32_t width, height;
} xg_cone_view;

/* Raw line integrals of one view (project_phantom, phantom.py:181-236):
 * out float64 [H][W].  step_factor in (0, 0.5].  workspace >=
 * xg_project_workspace_bytes(H, W). */
size_t xg_project_workspace_bytes(int32_t h, int32_t w);
xg_status xg_project_volume(const xg_volume* vol, const xg_cone_view* view, double step_factor, double* out,
                            void* workspace, size_t workspace_bytes, void* stream);

/* SSIM of pred vs ref (metrics.py:57-124): mean over every fully-interior
 * 11x11 Gaussian window (sigma 1.5, K1 0.01, K2 0.03), float64 arithmetic;
 * pred / ref float32 (is_f64 = 0) or float64 [h][w], h, w >= 11.
 * ssim_out (device double, optional) receives the mean; grad_out (optional,
 * float64 [h][w]) d(mean SSIM)/d pred (metrics.py:98-124); dl_out
 * (optional, float32 [h][w]) the trainer's fused upstream gradient
 *   dl = dl_ssim_scale * dSSIM/dpred + dl_l1_scale * sign(pred - ref)
 * (trainer.py:117-123 with dl_ssim_scale = -gamma, dl_l1_scale =
 * (1 - gamma) / (h w)).  workspace >= xg_ssim_workspace_bytes(h, w). */
size_t xg_ssim_workspace_bytes(int32_t h, int32_t w);
xg_status xg_ssim(const void* pred, const void* ref, int32_t is_f64, int32_t h, int32_t w, double data_range,
                  double* ssim_out, double* grad_out, float* dl_out, double dl_ssim_scale, double dl_l1_scale,
                  void* workspace, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* XGAUSS_H */
