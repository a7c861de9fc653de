/*
 * softsphere_b200.h -- C ABI of the B200-native sphere-render hot path.
 *
 * The reference (`softsphere`, pure NumPy) has no FFI; this header declares the entry
 * points a reference-side binding for the render path would bind.  Each one names the
 * reference interface it replaces (paths relative to pkg/src/softsphere/):
 *
 *   ss_forward   <- render_forward     raster.py:437-512  (compute_bounds :181-236,
 *                                      sort_draw_records :239-244, _bin_tiles :267-293,
 *                                      _draw_tile :328-417)
 *   ss_backward  <- render_backward    grad.py:323-357    (_hit_gradients :89-179,
 *                                      _accumulate_tiles :210-259,
 *                                      accumulate_and_normalize :262-302,
 *                                      gate_small_spheres :305-320)
 *   ss_workspace_bytes / SsDims        the arrays render_forward allocates per call
 *                                      (raster.py:462-474) become one caller-owned buffer
 *   ss_read_status                     RenderStats raster.py:113-123 + the ValidationError
 *                                      conditions of SphereScene.validate scene.py:91-114
 *   ss_debug_tile_lists                (record_seq, tile_starts) of _bin_tiles, parity only
 *
 * Conventions (camera.py:3-13): p_cam = R (p_world - t), camera looks down +z, pixel
 * (i, j) centre ray through u = i + 0.5, v = j + 0.5, NDC z = (far - depth)/(far - near).
 *
 * Everything is plain pointers and sizes; no torch types.  All data pointers are DEVICE
 * pointers unless marked host.  The library never allocates, frees or synchronises
 * (except ss_read_status); all work is enqueued on the caller's stream.
 */
#ifndef SOFTSPHERE_B200_H
#define SOFTSPHERE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SS_ABI_VERSION 2

/* ---- return codes (host-side argument checking; errors.py classes in parentheses) ---- */
#define SS_OK 0
#define SS_ERR_NULL 1         /* a required pointer is NULL */
#define SS_ERR_DIMS 2         /* bad dims: M < 0, d outside 1..32, W/H outside 1..16384 (ConfigurationError) */
#define SS_ERR_PARAMS 3       /* eps <= 0, tau outside [0,1), top_k outside 1..64 (ValidationError, blend.py:40-45) */
#define SS_ERR_CAMERA 4       /* focal/sensor <= 0, near >= far, bad mode (ConfigurationError, camera.py:153-177) */
#define SS_ERR_WORKSPACE 5    /* workspace_bytes < ss_workspace_bytes(dims) */
#define SS_ERR_UNSUPPORTED 6  /* tile != 16 or chunk outside 1..256 */
#define SS_ERR_CUDA 7         /* a CUDA runtime call failed (see ss_last_cuda_error) */

/* ---- device-side status flags (status[0], read with ss_read_status) ---- */
#define SS_FLAG_INVALID_INPUT 1u  /* NaN/Inf field or radius <= 0 (ValidationError, scene.py:91-114) */
#define SS_FLAG_PAIR_OVERFLOW 2u  /* tile-sphere pairs > dims.max_pairs; nothing was drawn */
#define SS_FLAG_LIST_FALLBACK 4u  /* informational: a tile held more than 4096 spheres, the tile lists were built by
                                     the two-pass path (count, scan, emit) instead of the direct per-tile buckets */

/* ---- option flags ---- */
#define SS_OPT_STORE_BUFFER 1u   /* forward: write ids/z/closeness/log_denom (store_buffer, raster.py:445) */
#define SS_OPT_COLLECT_STATS 2u  /* forward: fill candidates_tested/hits_blended/pixels_early_stopped */
#define SS_OPT_NORMALIZE 4u      /* backward: normalize=True (grad.py:331) */
#define SS_OPT_GATE 8u           /* backward: gate=True (grad.py:332) */
#define SS_OPT_CAMERA_GRADS 16u  /* backward: also reduce camera gradients */
#define SS_OPT_ACCUMULATE 32u    /* backward: add into d_* / pixel_count instead of overwriting (multi-view) */
#define SS_OPT_REUSE_RECORDS 64u /* backward: camera-frame records in the workspace are still those of the
                                    matching forward call; skip recomputing them (grad.py:213, :351) */
#define SS_OPT_SKIP_VALIDATE 128u /* forward: do not scan inputs for NaN/Inf/radius <= 0 */
#define SS_OPT_DETERMINISTIC 256u /* backward: bit-reproducible gradients (needs det_workspace).  The reference
                                    * merges its per-tile sums in a fixed order and is bit-identical run to run
                                    * (grad.py:231-250); the default device path sums with float32
                                    * L2 atomics, whose order varies.  In this mode every per-sphere sum is
                                    * accumulated in 64-bit fixed point (integer addition is associative) on a
                                    * per-sphere power-of-two grid found by a first pass (order-independent max),
                                    * and the camera sums are reduced in block order: two passes of k_backward. */

#define SS_MODE_PINHOLE 0
#define SS_MODE_ORTHOGRAPHIC 1

#define SS_MAX_FEATURE_DIM 32
#define SS_MAX_TOP_K 64
#define SS_TILE 16
#define SS_MAX_CHUNK 256

/* Camera (camera.py:130-177), passed by value from the host. */
typedef struct SsCamera {
    double t[3];      /* camera position in world units */
    double R[9];      /* row-major rotation, p_cam = R (p - t) */
    double focal;     /* focal_length */
    double sensor_w;  /* sensor_width; pixel size = sensor_w / width */
    double near_;     /* min depth */
    double far_;      /* max depth */
    int32_t width;
    int32_t height;
    int32_t mode;     /* SS_MODE_* */
    int32_t pad_;
} SsCamera;

/* Problem size; fixes the workspace layout. */
typedef struct SsDims {
    int64_t num_spheres;  /* M */
    int64_t max_pairs;    /* capacity for (tile, sphere) pairs, < 2^31 */
    int32_t feature_dim;  /* d, 1..32 */
    int32_t width;        /* W */
    int32_t height;       /* H */
    int32_t top_k;        /* K = n_track, 1..64 */
} SsDims;

/* BlendParams (blend.py:25-45) + pipeline knobs of render_forward (raster.py:437-447). */
typedef struct SsBlend {
    double gamma;   /* clamped to [1e-5, 1] by the library, like BlendParams.__post_init__ */
    double eps;     /* epsilon > 0 */
    double tau;     /* in [0, 1); 0 disables early stopping */
    int32_t tile;   /* must be 16 */
    int32_t chunk;  /* candidates per vote/batch, 1..256 (reference default 256) */
    uint32_t flags; /* SS_OPT_* */
    uint32_t pad_;
} SsBlend;

/*
 * Forward.  Inputs are float32 SoA tensors (the reference holds float64 columns of the
 * same values): pos (M,3), rad (M), opa (M, raw/unclamped), feat (M,d), bg (d).
 * Outputs: image (H,W,d), bg_weight (H,W) and -- with SS_OPT_STORE_BUFFER -- the backward
 * buffer in SLOT-MAJOR layout: ids/z/closeness are (K,H,W) (the reference's (H,W,K)
 * transposed so that pixel-parallel access is coalesced), log_denom (H,W).
 * Empty slots: id -1, z 0, closeness 0 (raster.py:410-413).
 * Optional parity outputs (NULL to skip): rect (M,4) int32 = x_min,x_max,y_min,y_max;
 * on_sensor (M) uint8; earliest (M) float64; proj_radius_px (M) float64.
 */
typedef struct SsForwardArgs {
    SsDims dims;
    SsCamera cam;
    SsBlend blend;
    const float *pos, *rad, *opa, *feat, *bg;
    void *workspace;
    size_t workspace_bytes;
    float *image;
    float *bg_weight;
    int32_t *ids;
    float *z;
    float *closeness;
    float *log_denom;
    int32_t *rect;
    uint8_t *on_sensor;
    double *earliest;
    double *proj_radius_px;
} SsForwardArgs;

/*
 * Backward.  Consumes the buffer written by ss_forward and upstream (H,W,d).
 * Outputs: d_pos (M,3), d_rad (M), d_opa (M), d_feat (M,d) float32; pixel_count (M) int32;
 * cam_grad: 16 float64 on the device = d_translation[3], G[9] (= d loss / d R, row-major,
 * to be pulled back through the rotation parameterisation by the host, camera.py:57-117),
 * d_focal, d_sensor_width, 2 reserved.  cam_grad may be NULL without SS_OPT_CAMERA_GRADS.
 */
typedef struct SsBackwardArgs {
    SsDims dims;
    SsCamera cam;
    SsBlend blend;
    const float *pos, *rad, *opa, *feat, *bg;
    void *workspace;
    size_t workspace_bytes;
    const int32_t *ids;
    const float *z;
    const float *closeness;
    const float *log_denom;
    const float *upstream;
    float *d_pos;
    float *d_rad;
    float *d_opa;
    float *d_feat;
    int32_t *pixel_count;
    double *cam_grad;
    void *det_workspace;        /* SS_OPT_DETERMINISTIC: caller-owned scratch of ss_deterministic_workspace_bytes, else NULL */
    size_t det_workspace_bytes;
} SsBackwardArgs;

/* status block, host copy (ss_read_status) */
typedef struct SsStatus {
    int64_t flags;                 /* SS_FLAG_* */
    int64_t spheres_on_sensor;     /* RenderStats.spheres_on_sensor */
    int64_t num_pairs;             /* tile-sphere pairs the scene needs (T) */
    int64_t candidates_tested;     /* RenderStats.candidates_tested (SS_OPT_COLLECT_STATS) */
    int64_t hits_blended;          /* RenderStats.hits_blended */
    int64_t pixels_early_stopped;  /* RenderStats.pixels_early_stopped */
    int64_t first_invalid;         /* lowest sphere index that failed validation, or -1 */
    int64_t reserved[9];
} SsStatus;

int ss_abi_version(void);
const char *ss_status_string(int code);
const char *ss_last_cuda_error(void);

/* Bytes of caller-owned device workspace for `dims` (256-byte aligned base required). */
int ss_workspace_bytes(const SsDims *dims, size_t *out_bytes);

/* Must be called once on a freshly allocated (or re-laid-out) workspace before its first use: clears
 * the status block and the "gradient accumulators are clean" tag.  ss_backward re-zeroes only the
 * accumulator rows it touched and trusts that tag on the next call (instead of a 48 MB memset per
 * call at 1M spheres); a stale tag in recycled memory would be trusted wrongly. */
int ss_workspace_init(const SsDims *dims, void *workspace, size_t workspace_bytes, void *stream);

/* `stream` is a cudaStream_t passed as void* (NULL = default stream). */
int ss_forward(const SsForwardArgs *args, void *stream);
int ss_backward(const SsBackwardArgs *args, void *stream);

/* ss_forward with the image drawn in `n_bands` (1..SS_MAX_BANDS) bands of whole tile rows, top to bottom, one
 * raster launch per band.  band_events: HOST array of n_bands cudaEvent_t (as void*), created by the caller;
 * event b is recorded on `stream` right after band b and completes when rows [row_begin, row_end) of
 * ss_band_rows(height, n_bands, b) are final in image / bg_weight / ids / z / closeness / log_denom.  A host
 * caller lets a copy stream wait on event b and downloads those image rows while the later bands are still being
 * drawn (the reference returns the whole image at once, raster.py:504-512; results are identical to ss_forward:
 * tiles are independent).  The status counters are complete after the last band.  Bands 1.. are launched on a
 * library-owned side stream beside band 0 (fork after the binning pass, join on `stream` before the last event, which
 * therefore marks the end of the whole pass on `stream`; graph edges under stream capture), so that their CTAs fill
 * the partial last wave of the band before; the events of the bands in between are recorded on that side stream.
 * SS_BAND_FORK=0 in the environment keeps every launch on `stream`. */
#define SS_MAX_BANDS 16
int ss_forward_banded(const SsForwardArgs *args, int n_bands, void *const *band_events, void *stream);
int ss_band_rows(int height, int n_bands, int band, int *row_begin, int *row_end);

/* Scratch size of the SS_OPT_DETERMINISTIC backward for these dimensions (per-sphere grid exponents +
 * 64-bit fixed-point accumulator rows). */
int ss_deterministic_workspace_bytes(const SsDims *dims, size_t *out_bytes);

/* Copies the status block of the last forward on `workspace` to the host; synchronises `stream`. */
int ss_read_status(const void *workspace, SsStatus *out_host, void *stream);

/* Parity/debug: copy the per-tile candidate lists of the last forward (sphere ids grouped by
 * tile in scan order) into tile_starts_out (n_tiles + 1, int32) and ids_out (max_pairs, int32). */
int ss_debug_tile_lists(const SsDims *dims, const void *workspace, int32_t *tile_starts_out,
                        int32_t *ids_out, void *stream);

/* ------------------------------------------------------------------------------------------------
 * the step either side of the render path in the reference's fit loop.
 *
 *   ss_photometric_loss <- photometric_loss           optim.py:87-97
 *   ss_fit_step         <- opacity_depth_regularizer  optim.py:100-121  (gradients added in place)
 *                          visibility += pixel_count  optim.py:307
 *                          adam_step x 4 groups + radius floor  optim.py:142-154, :309-329
 *   ss_adam_flat        <- adam_step on one array     optim.py:142-154  (camera vectors)
 * ---------------------------------------------------------------------------------------------- */

/* loss_out (device, float64) = mean |image - target|; upstream = sign(image - target) / n (0 at ties). */
int ss_photometric_loss(const float *image, const float *target, float *upstream, int64_t n,
                        double *loss_out, void *stream);

/* Parameter groups: 0 position, 1 radius, 2 opacity, 3 feature.  lr[g] == 0 freezes group g
 * (its state pointers may be NULL); step[g] is the group's Adam step count AFTER this update (>= 1). */
typedef struct SsFitStepArgs {
    int64_t num_spheres;
    int32_t feature_dim;
    int32_t pad_;
    float *pos, *rad, *opa, *feat;                       /* parameters, updated in place */
    const float *d_pos, *d_rad, *d_opa, *d_feat;         /* gradients from ss_backward */
    const int32_t *pixel_count;                          /* from ss_backward (may be NULL without visibility) */
    int32_t *visibility;                                 /* += pixel_count, or NULL */
    float *m_pos, *v_pos, *m_rad, *v_rad, *m_opa, *v_opa, *m_feat, *v_feat; /* Adam moments, in place */
    double lr[4];
    int64_t step[4];
    double beta1, beta2, adam_eps;
    double radius_min;                                   /* radius floor (FitConfig.radius_min) */
    double lambda_od;                                    /* opacity-depth regulariser weight; 0 disables */
    SsCamera cam;                                        /* for the regulariser */
    double *energy;                                      /* device float64: regulariser energy, or NULL */
} SsFitStepArgs;

int ss_fit_step(const SsFitStepArgs *args, void *stream);

int ss_adam_flat(float *params, const float *grads, float *m, float *v, int64_t n, double lr, double beta1,
                 double beta2, double adam_eps, int64_t step, int use_floor, double floor_value, void *stream);

/* ------------------------------------------------------------------------------------------------
 * scene surgery on the device (the sphere set changes between steps).
 *
 *   ss_prune_mask    <- prune's keep mask            optim.py:161-175
 *   ss_compact_rows  <- scene.positions[keep] ... and states[name].take(keep)   optim.py:176-183, :351-352
 *   ss_subdivide     <- subdivide (FCC x12)          optim.py:186-213
 * ---------------------------------------------------------------------------------------------- */

/* keep[i] = clip(opa[i],0,1) >= opacity_min  &&  (background_dist <= 0 || |feat[i] - bg| >= background_dist)
 *           && (visibility == NULL || visibility[i] > 0);  comparisons in float64 like the reference. */
int ss_prune_mask(const float *opa, const float *feat, const float *bg, const int32_t *visibility, int64_t M,
                  int32_t d, double opacity_min, double background_dist, uint8_t *keep, void *stream);
/* Same rule on float64 device columns (the reference-signature prune() wrapper: an opacity exactly at the
 * threshold must compare as the reference's float64 value does). */
int ss_prune_mask_f64(const double *opa, const double *feat, const double *bg, const int32_t *visibility, int64_t M,
                      int32_t d, double opacity_min, double background_dist, uint8_t *keep, void *stream);

/* keep[i] = values[i] != 0.  With values = pixel_count this marks the spheres that received gradient
 * (SceneGradients.pixel_count > 0, grad.py:45-61): a host caller then compacts and downloads only those rows. */
int ss_mask_nonzero_i32(const int32_t *values, int64_t M, uint8_t *keep, void *stream);

/* One per-sphere column to compact: `row_bytes` (a multiple of 4) bytes per sphere, device pointers.
 * `dst_stride_bytes` = 0 packs the kept rows back to back (scene.positions[keep], optim.py:176-181); a larger
 * multiple of 4 leaves that distance between consecutive kept rows, so that several columns can be interleaved
 * into ONE array of records (dst pointers offset inside the first record): one copy moves them all. */
typedef struct SsColumn {
    const void *src;
    void *dst;
    int64_t row_bytes;
    int64_t dst_stride_bytes;
} SsColumn;

int ss_compact_workspace_bytes(int64_t M, size_t *out_bytes);

/* Stable compaction of up to 16 columns by `keep` (M bytes, device) into their dst buffers (capacity M
 * rows each, must not alias src); count_out (device int64) receives the number of kept rows.  `cols` is
 * a HOST array.  Columns that interleave into one array of records (equal dst strides, the columns tiling a
 * record of <= 48 words without gaps) are assembled per block in shared memory and written as whole 128-byte lines;
 * for that form dst and count_out may also be MAPPED PINNED HOST memory (the pass then is the download: the records
 * are written over PCIe as the kernel runs and are valid on the host once the stream has been synchronised). */
int ss_compact_rows(const uint8_t *keep, int64_t M, const SsColumn *cols, int32_t n_cols, void *workspace,
                    size_t workspace_bytes, int64_t *count_out, void *stream);

/* Outputs hold 12 M rows; child c of parent p is row 12 p + c (reshape(m * 12, 3), optim.py:204). */
int ss_subdivide(const float *pos, const float *rad, const float *opa, const float *feat, int64_t M, int32_t d,
                 double scale, float *pos_out, float *rad_out, float *opa_out, float *feat_out, void *stream);
/* float64 columns in and out (the reference-signature subdivide() wrapper: children exact in float64). */
int ss_subdivide_f64(const double *pos, const double *rad, const double *opa, const double *feat, int64_t M,
                     int32_t d, double scale, double *pos_out, double *rad_out, double *opa_out, double *feat_out,
                     void *stream);

/* ------------------------------------------------------------------------------------------------
 * the on-disk record formats straight into / out of the device SoA columns.
 *
 *   ss_psc1_unpack / ss_psc1_pack  <- the record block of scene_from_bytes / scene_to_bytes
 *                                     scene.py:179-227: (5 + d) little-endian float32 per sphere
 *                                     (position*3, radius, opacity, feature*d); `records` is a DEVICE
 *                                     copy of that block (the 16-byte header and the background are
 *                                     parsed on the host).
 *   ss_convert_f64_f32 / _f32_f64  <- the <f8 Adam-moment blobs of the PSK1 checkpoint, optim.py:397-405
 * ---------------------------------------------------------------------------------------------- */
int ss_psc1_unpack(const void *records, int64_t M, int32_t d, float *pos, float *rad, float *opa, float *feat,
                   void *stream);
int ss_psc1_pack(const float *pos, const float *rad, const float *opa, const float *feat, int64_t M, int32_t d,
                 void *records_out, void *stream);
int ss_convert_f64_f32(const double *in, float *out, int64_t n, void *stream);
int ss_convert_f32_f64(const float *in, double *out, int64_t n, void *stream);

/* ------------------------------------------------------------------------------------------------
 * per-pixel shading of the feature map, forward and backward (shade.py).
 * Images are (n_pixels, channels) float32, row-major, device.
 *
 *   ss_shade_identity[_backward]  <- shade_identity[_backward]   shade.py:66-77   (any channel count)
 *   ss_shade_diffuse[_backward]   <- shade_diffuse[_backward]    shade.py:84-131  ([albedo:3, normal:3])
 *   ss_shade_linear[_backward]    <- shade_linear[_backward]     shade.py:148-171 (weight (d_in,3), bias (3),
 *                                    d_in = d + 3 when view_dirs is given)
 *   ss_view_directions            <- view_direction_plane        shade.py:138-142
 * ---------------------------------------------------------------------------------------------- */
typedef struct SsLight {
    double direction[3]; /* pointing from the light into the scene; normalised by the library */
    double intensity;    /* >= 0 */
    double ambient;      /* in [0, 1] */
} SsLight;

int ss_shade_identity(const float *image, int64_t n_values, float *out, void *stream);
int ss_shade_identity_backward(const float *image, const float *upstream, int64_t n_values, float *d_image,
                               void *stream);
/* `lights` is a HOST array of at most 8 lights; SS_ERR_PARAMS mirrors DirectionalLight's ValidationError. */
int ss_shade_diffuse(const float *image, int64_t n_pixels, const SsLight *lights, int32_t n_lights, float *out,
                     void *stream);
int ss_shade_diffuse_backward(const float *image, const float *upstream, int64_t n_pixels, const SsLight *lights,
                              int32_t n_lights, float *d_image, void *stream);
/* weight, bias: device float32.  view_dirs (n_pixels, 3) or NULL. */
int ss_shade_linear(const float *image, const float *view_dirs, int64_t n_pixels, int32_t d, const float *weight,
                    const float *bias, float *out, void *stream);
/* d_weight (d_in * 3) and d_bias (3): device float64, or both NULL for a frozen shader. */
int ss_shade_linear_backward(const float *image, const float *view_dirs, int64_t n_pixels, int32_t d,
                             const float *weight, const float *bias, const float *upstream, float *d_image,
                             double *d_weight, double *d_bias, void *stream);
/* out: (H, W, 3) unit view directions in the camera frame (pinhole) or (0, 0, 1) (orthographic). */
int ss_view_directions(const SsCamera *cam, float *out, void *stream);

/* Number of kernels this library has launched in this process (bench.py's gpu_launches). */
int64_t ss_launch_count(void);

/* Measurement only (no reference counterpart): when enabled, every kernel the library launches
 * is bracketed by a CUDA event pair on the launching stream.  ss_profile_collect synchronises
 * the device and returns, per kernel id, the summed duration in ms and the launch count since
 * the last enable/collect. */
void ss_profile_enable(int on);
void ss_profile_enable_mask(unsigned mask); /* bit k = time kernel id k only */
int ss_profile_collect(double *ms_sum, int64_t *launches, int n);
/* The same for launches captured into a CUDA graph while profiling was enabled: they carry external event-record
 * nodes, re-recorded by every replay.  ss_profile_collect_captured synchronises the device and returns, per kernel
 * id, the summed duration and launch count of the MOST RECENT replay (call it after each replay to accumulate);
 * ss_profile_captured_reset forgets the captured pairs (before capturing another graph). */
void ss_profile_captured_reset(void);
int ss_profile_collect_captured(double *ms_sum, int64_t *launches, int n);
int ss_profile_kernel_count(void);
const char *ss_profile_kernel_name(int kid);

#ifdef __cplusplus
}
#endif
#endif /* SOFTSPHERE_B200_H */
