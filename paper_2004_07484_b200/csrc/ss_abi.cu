// C ABI of the sphere-render hot path (see include/softsphere_b200.h).  Host-side argument
// checks mirror the reference's exceptions; kernels are enqueued on the caller's stream and
// nothing here allocates, frees or synchronises (except ss_read_status).
#include <stdlib.h>
#include <atomic>
#include <cmath>
#include <cstring>

#include "ss_common.cuh"

namespace ss {
static std::atomic<long long> g_launches{0};
static thread_local cudaError_t g_last_cuda = cudaSuccess;
void count_launch(int n) { g_launches += n; }

// ---- per-kernel event timing -------------------------------------------------------------
static unsigned g_prof_mask = 0;  // bit k: time kernel id k
static const int kProfCap = 8192;
static cudaEvent_t g_ev0[kProfCap], g_ev1[kProfCap];
static int g_ev_kid[kProfCap];
static int g_ev_made = 0, g_ev_used = 0;
// Launches made while the stream is being captured into a CUDA graph get EXTERNAL event-record nodes (their events
// are re-recorded by every replay and can be read from outside the graph): one pair per captured launch, kept until
// ss_profile_captured_reset; ss_profile_collect_captured reads the pairs of the most recent replay.
static const int kCapCap = 1024;
static cudaEvent_t g_cev0[kCapCap], g_cev1[kCapCap];
static int g_cev_kid[kCapCap];
static int g_cev_made = 0, g_cev_used = 0;
static bool capturing(cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    return cudaStreamIsCapturing(s, &st) == cudaSuccess && st == cudaStreamCaptureStatusActive;
}
void prof_begin(int kid, cudaStream_t s) {
    if (!((g_prof_mask >> kid) & 1u)) return;
    if (capturing(s)) {
        if (g_cev_used >= kCapCap) return;
        if (g_cev_used >= g_cev_made) {
            cudaEventCreate(&g_cev0[g_cev_made]);
            cudaEventCreate(&g_cev1[g_cev_made]);
            ++g_cev_made;
        }
        g_cev_kid[g_cev_used] = kid;
        cudaEventRecordWithFlags(g_cev0[g_cev_used], s, cudaEventRecordExternal);
        return;
    }
    if (g_ev_used >= kProfCap) return;
    if (g_ev_used >= g_ev_made) {
        cudaEventCreate(&g_ev0[g_ev_made]);
        cudaEventCreate(&g_ev1[g_ev_made]);
        ++g_ev_made;
    }
    g_ev_kid[g_ev_used] = kid;
    cudaEventRecord(g_ev0[g_ev_used], s);
}
void prof_end(int kid, cudaStream_t s) {
    if (!((g_prof_mask >> kid) & 1u)) return;
    if (capturing(s)) {
        if (g_cev_used >= kCapCap) return;
        cudaEventRecordWithFlags(g_cev1[g_cev_used], s, cudaEventRecordExternal);
        ++g_cev_used;
        return;
    }
    if (g_ev_used >= kProfCap) return;
    cudaEventRecord(g_ev1[g_ev_used], s);
    ++g_ev_used;
}
}  // namespace ss

using namespace ss;

namespace {

int check_dims(const SsDims &d) {
    if (d.num_spheres < 0 || d.num_spheres > 0x7fffffffLL) return SS_ERR_DIMS;
    if (d.max_pairs < 0 || d.max_pairs > 0x7fffffffLL) return SS_ERR_DIMS;
    if (d.feature_dim < 1 || d.feature_dim > SS_MAX_FEATURE_DIM) return SS_ERR_DIMS;
    if (d.width < 1 || d.height < 1 || d.width > 16384 || d.height > 16384) return SS_ERR_DIMS;
    if ((long long)d.width * d.height > (1LL << 24)) return SS_ERR_DIMS;  // float32 pixel counter is exact up to 2^24
    if (d.top_k < 1 || d.top_k > SS_MAX_TOP_K) return SS_ERR_PARAMS;
    return SS_OK;
}

int check_camera(const SsCamera &c, const SsDims &d) {
    if (c.width != d.width || c.height != d.height) return SS_ERR_DIMS;
    if (c.mode != SS_MODE_PINHOLE && c.mode != SS_MODE_ORTHOGRAPHIC) return SS_ERR_CAMERA;
    if (!(c.focal > 0.0) || !(c.sensor_w > 0.0)) return SS_ERR_CAMERA;
    if (!(c.near_ < c.far_) || c.near_ < 0.0 || c.far_ - c.near_ < 1e-12) return SS_ERR_CAMERA;
    for (int i = 0; i < 3; ++i)
        if (!std::isfinite(c.t[i])) return SS_ERR_CAMERA;
    for (int i = 0; i < 9; ++i)
        if (!std::isfinite(c.R[i])) return SS_ERR_CAMERA;
    return SS_OK;
}

int check_blend(const SsBlend &b) {
    if (!(b.eps > 0.0)) return SS_ERR_PARAMS;
    if (!(b.tau >= 0.0 && b.tau < 1.0)) return SS_ERR_PARAMS;
    if (!std::isfinite(b.gamma)) return SS_ERR_PARAMS;
    if (b.tile != SS_TILE) return SS_ERR_UNSUPPORTED;
    if (b.chunk < 1 || b.chunk > SS_MAX_CHUNK) return SS_ERR_UNSUPPORTED;
    return SS_OK;
}

double clamp_gamma(double g) { return g < 1e-5 ? 1e-5 : (g > 1.0 ? 1.0 : g); }  // blend.py:39

int cuda_fail(cudaError_t e) {
    ss::g_last_cuda = e;
    return SS_ERR_CUDA;
}

}  // namespace

extern "C" {

int ss_abi_version(void) { return SS_ABI_VERSION; }

const char *ss_status_string(int code) {
    switch (code) {
        case SS_OK: return "ok";
        case SS_ERR_NULL: return "required pointer is NULL";
        case SS_ERR_DIMS: return "invalid dimensions";
        case SS_ERR_PARAMS: return "invalid blend parameters";
        case SS_ERR_CAMERA: return "invalid camera";
        case SS_ERR_WORKSPACE: return "workspace too small";
        case SS_ERR_UNSUPPORTED: return "unsupported tile or chunk size";
        case SS_ERR_CUDA: return "CUDA runtime error";
        default: return "unknown status";
    }
}

const char *ss_last_cuda_error(void) { return cudaGetErrorString(ss::g_last_cuda); }

int64_t ss_launch_count(void) { return (int64_t)ss::g_launches.load(); }

void ss_profile_enable(int on) { ss::g_prof_mask = on ? 0xffffffffu : 0u; ss::g_ev_used = 0; }

void ss_profile_enable_mask(unsigned mask) { ss::g_prof_mask = mask; ss::g_ev_used = 0; }

int ss_profile_collect(double *ms_sum, int64_t *launches, int n) {
    if (!ms_sum || !launches) return SS_ERR_NULL;
    for (int i = 0; i < n; ++i) { ms_sum[i] = 0.0; launches[i] = 0; }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(e);
    for (int i = 0; i < ss::g_ev_used; ++i) {
        float ms = 0.f;
        e = cudaEventElapsedTime(&ms, ss::g_ev0[i], ss::g_ev1[i]);
        if (e != cudaSuccess) return cuda_fail(e);
        int k = ss::g_ev_kid[i];
        if (k >= 0 && k < n) { ms_sum[k] += ms; launches[k] += 1; }
    }
    ss::g_ev_used = 0;
    return SS_OK;
}

void ss_profile_captured_reset(void) { ss::g_cev_used = 0; }

int ss_profile_collect_captured(double *ms_sum, int64_t *launches, int n) {
    if (!ms_sum || !launches) return SS_ERR_NULL;
    for (int i = 0; i < n; ++i) { ms_sum[i] = 0.0; launches[i] = 0; }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(e);
    for (int i = 0; i < ss::g_cev_used; ++i) {
        float ms = 0.f;
        e = cudaEventElapsedTime(&ms, ss::g_cev0[i], ss::g_cev1[i]);
        if (e != cudaSuccess) return cuda_fail(e);
        int k = ss::g_cev_kid[i];
        if (k >= 0 && k < n) { ms_sum[k] += ms; launches[k] += 1; }
    }
    return SS_OK;
}

int ss_profile_kernel_count(void) { return ss::KID_COUNT; }

const char *ss_profile_kernel_name(int kid) {
    static const char *names[] = {"k_project", "k_scan", "k_emit", "k_tile_sort_small", "k_tile_sort_big",
                                  "k_raster", "k_backward", "k_finalize", "memset_fwd", "memset_bwd"};
    return (kid >= 0 && kid < ss::KID_COUNT) ? names[kid] : "?";
}

int ss_workspace_bytes(const SsDims *dims, size_t *out_bytes) {
    if (!dims || !out_bytes) return SS_ERR_NULL;
    int rc = check_dims(*dims);
    if (rc != SS_OK) return rc;
    *out_bytes = make_layout(*dims).total;
    return SS_OK;
}

int ss_workspace_init(const SsDims *dims, void *workspace, size_t workspace_bytes, void *stream) {
    if (!dims || !workspace) return SS_ERR_NULL;
    int rc = check_dims(*dims);
    if (rc != SS_OK) return rc;
    const Layout L = make_layout(*dims);
    if (workspace_bytes < L.total) return SS_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync((char *)workspace + L.status, 0, 16 * sizeof(int64_t), s);
    if (e != cudaSuccess) return cuda_fail(e);
    e = cudaMemsetAsync((char *)workspace + L.cam_part, 0, (CAM_VALS + 2) * sizeof(double), s);
    if (e != cudaSuccess) return cuda_fail(e);
    return SS_OK;
}

static int forward_impl(const SsForwardArgs *a, int n_bands, void *const *band_events, void *stream);

int ss_forward(const SsForwardArgs *a, void *stream) { return forward_impl(a, 1, nullptr, stream); }

int ss_forward_banded(const SsForwardArgs *a, int n_bands, void *const *band_events, void *stream) {
    if (n_bands < 1 || n_bands > SS_MAX_BANDS) return SS_ERR_PARAMS;
    if (!band_events) return SS_ERR_NULL;
    for (int b = 0; b < n_bands; ++b)
        if (!band_events[b]) return SS_ERR_NULL;
    return forward_impl(a, n_bands, band_events, stream);
}

int ss_band_rows(int height, int n_bands, int band, int *row_begin, int *row_end) {
    if (!row_begin || !row_end) return SS_ERR_NULL;
    if (height < 1 || n_bands < 1 || n_bands > SS_MAX_BANDS || band < 0 || band >= n_bands) return SS_ERR_PARAMS;
    const int nty = (height + SS_TILE - 1) / SS_TILE;
    const int r0 = (int)((long long)nty * band / n_bands) * SS_TILE;
    const int r1 = (int)((long long)nty * (band + 1) / n_bands) * SS_TILE;
    *row_begin = r0 < height ? r0 : height;
    *row_end = r1 < height ? r1 : height;
    return SS_OK;
}

static int forward_impl(const SsForwardArgs *a, int n_bands, void *const *band_events, void *stream) {
    if (!a) return SS_ERR_NULL;
    int rc = check_dims(a->dims);
    if (rc == SS_OK) rc = check_camera(a->cam, a->dims);
    if (rc == SS_OK) rc = check_blend(a->blend);
    if (rc != SS_OK) return rc;
    const bool store = (a->blend.flags & SS_OPT_STORE_BUFFER) != 0;
    if (!a->workspace || !a->image || !a->bg_weight || !a->bg) return SS_ERR_NULL;
    if (a->dims.num_spheres > 0 && (!a->pos || !a->rad || !a->opa || !a->feat)) return SS_ERR_NULL;
    if (store && (!a->ids || !a->z || !a->closeness || !a->log_denom)) return SS_ERR_NULL;
    FwdLaunch f;
    f.dims = a->dims; f.cam = make_cam(a->cam); f.blend = a->blend; f.gamma = clamp_gamma(a->blend.gamma);
    f.pos = a->pos; f.rad = a->rad; f.opa = a->opa; f.feat = a->feat; f.bg = a->bg;
    f.ws = (char *)a->workspace; f.L = make_layout(a->dims);
    if (a->workspace_bytes < f.L.total) return SS_ERR_WORKSPACE;
    f.image = a->image; f.bg_weight = a->bg_weight; f.ids = a->ids; f.z = a->z; f.clos = a->closeness;
    f.log_denom = a->log_denom;
    f.rect = a->rect; f.on_sensor = a->on_sensor; f.earliest = a->earliest; f.proj_r_out = a->proj_radius_px;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = launch_project(f, false, s);
    if (e != cudaSuccess) return cuda_fail(e);
    e = launch_binning(f, s);
    if (e != cudaSuccess) return cuda_fail(e);
    if (n_bands <= 1 && !band_events) {
        e = launch_raster(f, s);
        if (e != cudaSuccess) return cuda_fail(e);
        return SS_OK;
    }
    // bands of whole tile rows, one raster launch each; the event after band b completes when rows
    // [ss_band_rows(b)) of every forward output are final (a copy stream can start downloading them)
    // Every band is a launch of its own and would pay its own partial last wave (1 024 tiles on 592 resident CTAs are
    // 1.7 waves).  The bands are independent, so bands 1.. are launched on a library-owned side stream (fork after the
    // binning pass, join before the last band's event): their CTAs fill the SMs that band 0's last wave leaves idle,
    // band b's event still completes with band b alone, and the whole pass costs about one unbanded launch.  Under
    // stream capture the fork / join become graph edges.  SS_BAND_FORK=0: all bands in order on the caller's stream.
    static const bool fork_bands = [] { const char *v = getenv("SS_BAND_FORK"); return !(v && v[0] == '0'); }();
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    const bool forked = fork_bands && n_bands > 1 && side_stream(&side, &ev_fork, &ev_join);
    if (forked) {
        if (cudaEventRecord(ev_fork, s) != cudaSuccess || cudaStreamWaitEvent(side, ev_fork, 0) != cudaSuccess)
            return cuda_fail(cudaGetLastError());
    }
    for (int b = 0; b < n_bands; ++b) {
        const int ty0 = (int)((long long)f.L.nty * b / n_bands), ty1 = (int)((long long)f.L.nty * (b + 1) / n_bands);
        cudaStream_t sb = (forked && b > 0) ? side : s;
        e = launch_raster(f, sb, ty0 * f.L.ntx, (ty1 - ty0) * f.L.ntx);
        if (e != cudaSuccess) return cuda_fail(e);
        if (forked && b == n_bands - 1) {  // the caller's stream rejoins: its last event = the whole pass
            if (cudaEventRecord(ev_join, side) != cudaSuccess || cudaStreamWaitEvent(s, ev_join, 0) != cudaSuccess)
                return cuda_fail(cudaGetLastError());
            sb = s;
        }
        e = cudaEventRecord((cudaEvent_t)band_events[b], sb);
        if (e != cudaSuccess) return cuda_fail(e);
    }
    return SS_OK;
}

int ss_backward(const SsBackwardArgs *a, void *stream) {
    if (!a) return SS_ERR_NULL;
    int rc = check_dims(a->dims);
    if (rc == SS_OK) rc = check_camera(a->cam, a->dims);
    if (rc == SS_OK) rc = check_blend(a->blend);
    if (rc != SS_OK) return rc;
    const bool cam_grads = (a->blend.flags & SS_OPT_CAMERA_GRADS) != 0;
    if (!a->workspace || !a->bg || !a->ids || !a->z || !a->closeness || !a->log_denom || !a->upstream)
        return SS_ERR_NULL;
    if (cam_grads && !a->cam_grad) return SS_ERR_NULL;
    if (a->dims.num_spheres > 0 && (!a->pos || !a->rad || !a->opa || !a->feat || !a->d_pos || !a->d_rad ||
                                    !a->d_opa || !a->d_feat || !a->pixel_count))
        return SS_ERR_NULL;
    BwdLaunch b;
    b.dims = a->dims; b.cam = make_cam(a->cam); b.blend = a->blend; b.gamma = clamp_gamma(a->blend.gamma);
    b.pos = a->pos; b.rad = a->rad; b.opa = a->opa; b.feat = a->feat; b.bg = a->bg;
    b.ws = (char *)a->workspace; b.L = make_layout(a->dims);
    if (a->workspace_bytes < b.L.total) return SS_ERR_WORKSPACE;
    b.ids = a->ids; b.z = a->z; b.clos = a->closeness; b.log_denom = a->log_denom; b.upstream = a->upstream;
    b.d_pos = a->d_pos; b.d_rad = a->d_rad; b.d_opa = a->d_opa; b.d_feat = a->d_feat;
    b.pixel_count = a->pixel_count; b.cam_grad = a->cam_grad;
    b.det_ws = nullptr;
    if (a->blend.flags & SS_OPT_DETERMINISTIC) {
        if (!a->det_workspace) return SS_ERR_NULL;
        if (a->det_workspace_bytes < make_det_layout(a->dims).total) return SS_ERR_WORKSPACE;
        b.det_ws = (char *)a->det_workspace;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (!(a->blend.flags & SS_OPT_REUSE_RECORDS)) {
        // the reference recomputes camera-frame centres and projected radii (grad.py:213, :351)
        FwdLaunch f;
        std::memset(&f, 0, sizeof(f));
        f.dims = b.dims; f.cam = b.cam; f.blend = b.blend; f.gamma = b.gamma;
        f.pos = b.pos; f.rad = b.rad; f.opa = b.opa; f.feat = b.feat; f.bg = b.bg;
        f.ws = b.ws; f.L = b.L;
        cudaError_t e = launch_project(f, true, s);
        if (e != cudaSuccess) return cuda_fail(e);
    }
    cudaError_t e = launch_backward(b, s);
    if (e != cudaSuccess) return cuda_fail(e);
    return SS_OK;
}

int ss_deterministic_workspace_bytes(const SsDims *dims, size_t *out_bytes) {
    if (!dims || !out_bytes) return SS_ERR_NULL;
    int rc = check_dims(*dims);
    if (rc != SS_OK) return rc;
    *out_bytes = make_det_layout(*dims).total;
    return SS_OK;
}

int ss_read_status(const void *workspace, SsStatus *out_host, void *stream) {
    if (!workspace || !out_host) return SS_ERR_NULL;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemcpyAsync(out_host, workspace, sizeof(SsStatus), cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return cuda_fail(e);
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e);
    return SS_OK;
}

int ss_debug_tile_lists(const SsDims *dims, const void *workspace, int32_t *tile_starts_out, int32_t *ids_out,
                        void *stream) {
    if (!dims || !workspace || !tile_starts_out || !ids_out) return SS_ERR_NULL;
    int rc = check_dims(*dims);
    if (rc != SS_OK) return rc;
    Layout L = make_layout(*dims);
    const char *ws = (const char *)workspace;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemcpyAsync(tile_starts_out, ws + L.tile_start, (size_t)(L.n_tiles + 1) * 4,
                                    cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e);
    if (dims->max_pairs > 0) {
        e = cudaMemcpyAsync(ids_out, ws + L.pair_id, (size_t)dims->max_pairs * 4, cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return cuda_fail(e);
    }
    return SS_OK;
}

}  // extern "C"
