// Forward raster kernel for sm_100a (reference _draw_tile, raster.py:328-417).
//
// One 256-thread CTA per 16x16 tile, one thread per pixel.  The tile's depth-ordered
// candidate list is streamed in batches of `chunk` (<= 256) records staged in shared memory;
// all lanes of a warp look at the same candidate at the same time, so every shared-memory
// read in the test loop is a broadcast.
//
// Precision plan: the float64 reference decides hits with
// dist^2 = |c|^2 - t^2 and orders the per-pixel top-K by float64 NDC depth.  Here a float32
// test in the cancellation-free form d = c - t u, widened by a rigorous error band, filters
// candidates; every candidate that passes is re-evaluated with the reference's own float64
// formula, which alone decides hit / miss and produces the depth used for ordering.  The
// blend (online softmax of Eq. 1) runs in float32.
#include <math.h>

#include "ss_common.cuh"

namespace ss {

namespace {

struct RasterArgs {
    Cam cam;
    const int *tile_start;
    const int *pair_id;
    const Rec *rec;
    const float *feat;
    const float *bg;
    int d, K, chunk;
    double gamma, eps_over_g, log_tau;
    int tau_on, store_buffer, collect_stats;
    float *image, *bg_weight;
    int *ids; float *z, *clos, *log_denom;
    long long *status;
};

template <int KT>
struct TopK {
    double z[KT];
    int id[KT];
    float c[KT];
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int k = 0; k < KT; ++k) { z[k] = -INFINITY; id[k] = -1; c[k] = 0.0f; }
    }
    // keep the KT largest by (z desc, id asc) -- raster.py:389-399
    __device__ __forceinline__ void insert(double zz, int sid, float cl) {
        if (!(zz > z[KT - 1] || (zz == z[KT - 1] && sid < id[KT - 1]))) return;
        z[KT - 1] = zz; id[KT - 1] = sid; c[KT - 1] = cl;
        if (KT <= 8) {
#pragma unroll
            for (int k = KT - 1; k > 0; --k) {
                bool up = z[k] > z[k - 1] || (z[k] == z[k - 1] && id[k] < id[k - 1]);
                if (up) {
                    double tz = z[k]; z[k] = z[k - 1]; z[k - 1] = tz;
                    int ti = id[k]; id[k] = id[k - 1]; id[k - 1] = ti;
                    float tc = c[k]; c[k] = c[k - 1]; c[k - 1] = tc;
                }
            }
        } else {
            for (int k = KT - 1; k > 0; --k) {
                bool up = z[k] > z[k - 1] || (z[k] == z[k - 1] && id[k] < id[k - 1]);
                if (!up) break;
                double tz = z[k]; z[k] = z[k - 1]; z[k - 1] = tz;
                int ti = id[k]; id[k] = id[k - 1]; id[k - 1] = ti;
                float tc = c[k]; c[k] = c[k - 1]; c[k - 1] = tc;
            }
        }
    }
};

template <int DP, int KT, int MODE>
__global__ void __launch_bounds__(TILE_PX) k_raster(RasterArgs a) {
    __shared__ float4 s_cf[SS_MAX_CHUNK];  // float centre (or ortho cx, cy), band-widened r^2
    __shared__ double s_cx[SS_MAX_CHUNK], s_cy[SS_MAX_CHUNK], s_cz[SS_MAX_CHUNK], s_n2[SS_MAX_CHUNK];
    __shared__ float s_r[SS_MAX_CHUNK], s_o[SS_MAX_CHUNK];
    __shared__ int s_id[SS_MAX_CHUNK];
    __shared__ float s_f[SS_MAX_CHUNK * DP];
    __shared__ double s_red[8];
    __shared__ unsigned long long s_stat[3];

    const Cam &cam = a.cam;
    const int tile = blockIdx.x;
    const int tid = threadIdx.x;
    const int px = (tile % cam.ntx) * TILE + (tid & (TILE - 1));
    const int py = (tile / cam.ntx) * TILE + (tid >> 4);
    const bool valid = px < cam.W && py < cam.H;

    // pixel-centre ray, camera frame (camera.py:332-357)
    const double xs = ((px + 0.5) - cam.W / 2.0) * cam.pix;
    const double ys = ((py + 0.5) - cam.H / 2.0) * cam.pix;
    double ux = 0.0, uy = 0.0, uz = 1.0;
    if (MODE == SS_MODE_PINHOLE) {
        double vn = sqrt(xs * xs + ys * ys + cam.focal * cam.focal);
        ux = xs / vn; uy = ys / vn; uz = cam.focal / vn;
    }
    const float uxf = (float)ux, uyf = (float)uy, uzf = (float)uz;
    const float xsf = (float)xs, ysf = (float)ys;

    const bool overflow = (a.status[ST_FLAGS] & SS_FLAG_PAIR_OVERFLOW) != 0;  // lists not built
    const int s0 = a.tile_start[tile];
    const int n_cand = overflow ? 0 : a.tile_start[tile + 1] - s0;

    // tile-wide minimum ray cosine for the early-stop bound (raster.py:358)
    double tile_cos = 1.0;
    if (a.tau_on && MODE == SS_MODE_PINHOLE && n_cand > 0) {
        double v = valid ? uz : INFINITY;
        for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
        if ((tid & 31) == 0) s_red[tid >> 5] = v;
        __syncthreads();
        v = s_red[0];
#pragma unroll
        for (int w = 1; w < 8; ++w) v = fmin(v, s_red[w]);
        tile_cos = v;
    }
    if (tid < 3) s_stat[tid] = 0;

    float m = (float)a.eps_over_g, denom = 1.0f;
    float num[DP];
#pragma unroll
    for (int i = 0; i < DP; ++i) num[i] = 0.0f;
    TopK<KT> top;
    top.init();
    bool done = !valid;
    unsigned n_hits = 0;
    long long scanned = 0;
    const double near_ = cam.near_, far_ = cam.far_, inv_range = cam.inv_range;

    for (int start = 0; start < n_cand; start += a.chunk) {
        const int cn = min(a.chunk, n_cand - start);
        __syncthreads();  // previous batch fully consumed
        if (tid < cn) {
            const int sid = a.pair_id[s0 + start + tid];
            const Rec rc = a.rec[sid];
            const double n2 = rc.cx * rc.cx + rc.cy * rc.cy + rc.cz * rc.cz;
            s_cx[tid] = rc.cx; s_cy[tid] = rc.cy; s_cz[tid] = rc.cz; s_n2[tid] = n2;
            s_r[tid] = rc.r; s_o[tid] = rc.o; s_id[tid] = sid;
            // float32 filter radius: r + delta with delta >= the worst-case error of the
            // float32 distance, rounded up.
            float cn32 = (MODE == SS_MODE_PINHOLE)
                             ? (float)sqrt(n2)
                             : fabsf((float)rc.cx) + fabsf((float)rc.cy) + (float)(cam.sensor_w);
            float rb = rc.r + 1e-6f * (cn32 + rc.r);
            s_cf[tid] = make_float4((float)rc.cx, (float)rc.cy, (float)rc.cz, rb * rb * 1.000001f);
            const float *f = a.feat + (size_t)sid * a.d;
#pragma unroll
            for (int i = 0; i < DP; ++i) s_f[tid * DP + i] = i < a.d ? f[i] : 0.0f;
        }
        __syncthreads();
        if (a.tau_on) {  // vote, raster.py:364-368
            const double e0 = (MODE == SS_MODE_PINHOLE) ? sqrt(s_n2[0]) - (double)s_r[0]
                                                       : s_cz[0] - (double)s_r[0];
            const double zb = (far_ - fmin(fmax(e0 * tile_cos, near_), far_)) * inv_range;
            const double z_stop = a.gamma * (a.log_tau + (double)m + (double)logf(denom));
            done = done || (zb < z_stop);
            if (__syncthreads_and(done)) break;
        }
        scanned += cn;
        if (done) continue;
        for (int j = 0; j < cn; ++j) {
            const float4 c = s_cf[j];
            float d2;
            if (MODE == SS_MODE_PINHOLE) {
                const float t = fmaf(uxf, c.x, fmaf(uyf, c.y, uzf * c.z));
                const float dx = fmaf(-t, uxf, c.x), dy = fmaf(-t, uyf, c.y), dz = fmaf(-t, uzf, c.z);
                d2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
            } else {
                const float dx = c.x - xsf, dy = c.y - ysf;
                d2 = fmaf(dx, dx, dy * dy);
            }
            if (d2 < c.w) {
                // exact decision with the reference's float64 formula (raster.py:307-324)
                double t, dist2, zeta;
                if (MODE == SS_MODE_PINHOLE) {
                    t = ux * s_cx[j] + uy * s_cy[j] + uz * s_cz[j];
                    dist2 = fmax(s_n2[j] - t * t, 0.0);
                    zeta = t * uz;
                } else {
                    t = s_cz[j];
                    const double dx = s_cx[j] - xs, dy = s_cy[j] - ys;
                    dist2 = dx * dx + dy * dy;
                    zeta = t;
                }
                const float rf = s_r[j];
                const double rr = (double)rf * (double)rf;
                if (dist2 < rr && (t > 0.0 || t + sqrt(rr - dist2) > 0.0)) {
                    ++n_hits;
                    const double zz = (far_ - fmin(fmax(zeta, near_), far_)) * inv_range;
                    // closeness 1 - dist/r in the cancellation-free form (r^2 - dist^2) / (r (r + dist)):
                    // near the rim the float32 subtraction would lose all relative accuracy
                    const float cl = (float)(rr - dist2) / (rf * (rf + sqrtf((float)dist2)));
                    const float o = s_o[j];
                    const float e = (float)((double)o * zz / a.gamma);
                    if (e > m) {  // online form of raster.py:382-387
                        const float sc = expf(m - e);
                        denom *= sc;
#pragma unroll
                        for (int i = 0; i < DP; ++i) num[i] *= sc;
                        m = e;
                    }
                    const float oc = o * cl;
                    const float x = e - m;
                    const float term = oc * expf(x);
                    denom += term;
#pragma unroll
                    for (int i = 0; i < DP; ++i) num[i] = fmaf(term, s_f[j * DP + i], num[i]);
                    // store rule term > 0 (raster.py:389) evaluated as the float64 reference
                    // would: float32 underflows ~640 units of exponent earlier.
                    bool store = term > 0.0f;
                    if (!store && oc > 0.0f) store = x + logf(oc) > -745.13f;
                    if (store) top.insert(zz, s_id[j], cl);
                }
            }
        }
    }

    // finalise, raster.py:401-414
    if (valid) {
        const size_t P = (size_t)cam.W * cam.H;
        const size_t pix = (size_t)py * cam.W + px;
        const float ld = m + logf(denom);
        const float w_bg = expf((float)a.eps_over_g - ld);
        const float inv = 1.0f / denom;
#pragma unroll
        for (int i = 0; i < DP; ++i)
            if (i < a.d) a.image[pix * a.d + i] = fmaf(w_bg, a.bg[i], num[i] * inv);
        a.bg_weight[pix] = w_bg;
        if (a.store_buffer) {
#pragma unroll
            for (int k = 0; k < KT; ++k) {
                if (k < a.K) {
                    const bool empty = top.id[k] < 0;
                    a.ids[k * P + pix] = top.id[k];
                    a.z[k * P + pix] = empty ? 0.0f : (float)top.z[k];
                    a.clos[k * P + pix] = top.c[k];
                }
            }
            a.log_denom[pix] = ld;
        }
    }
    if (a.collect_stats) {
        unsigned h = n_hits;
        unsigned st = (valid && done) ? 1u : 0u;
        for (int o = 16; o > 0; o >>= 1) {
            h += __shfl_xor_sync(0xffffffffu, h, o);
            st += __shfl_xor_sync(0xffffffffu, st, o);
        }
        __syncthreads();
        if ((tid & 31) == 0) {
            atomicAdd(&s_stat[1], (unsigned long long)h);
            atomicAdd(&s_stat[2], (unsigned long long)st);
        }
        __syncthreads();
        if (tid == 0) {
            atomicAdd((unsigned long long *)&a.status[ST_TESTED], (unsigned long long)scanned);
            atomicAdd((unsigned long long *)&a.status[ST_HITS], s_stat[1]);
            atomicAdd((unsigned long long *)&a.status[ST_STOPPED], s_stat[2]);
        }
    }
}

template <int DP, int KT>
void launch_mode(const RasterArgs &r, int n_tiles, int mode, cudaStream_t s) {
    if (mode == SS_MODE_PINHOLE) k_raster<DP, KT, SS_MODE_PINHOLE><<<n_tiles, TILE_PX, 0, s>>>(r);
    else k_raster<DP, KT, SS_MODE_ORTHOGRAPHIC><<<n_tiles, TILE_PX, 0, s>>>(r);
}

template <int DP>
void launch_k(const RasterArgs &r, int n_tiles, int mode, cudaStream_t s) {
    if (r.K <= 5) launch_mode<DP, 5>(r, n_tiles, mode, s);
    else if (r.K <= 8) launch_mode<DP, 8>(r, n_tiles, mode, s);
    else if (r.K <= 32) launch_mode<DP, 32>(r, n_tiles, mode, s);
    else launch_mode<DP, 64>(r, n_tiles, mode, s);
}

}  // namespace

cudaError_t launch_raster(const FwdLaunch &a, cudaStream_t s) {
    const Layout &L = a.L;
    RasterArgs r;
    r.cam = a.cam;
    r.tile_start = (const int *)(a.ws + L.tile_start);
    r.pair_id = (const int *)(a.ws + L.pair_id);
    r.rec = (const Rec *)(a.ws + L.rec);
    r.feat = a.feat; r.bg = a.bg;
    r.d = a.dims.feature_dim; r.K = a.dims.top_k; r.chunk = a.blend.chunk;
    r.gamma = a.gamma; r.eps_over_g = a.blend.eps / a.gamma;
    r.tau_on = a.blend.tau > 0.0 ? 1 : 0;
    r.log_tau = r.tau_on ? log(a.blend.tau / (1.0 - a.blend.tau)) : 0.0;
    r.store_buffer = (a.blend.flags & SS_OPT_STORE_BUFFER) ? 1 : 0;
    r.collect_stats = (a.blend.flags & SS_OPT_COLLECT_STATS) ? 1 : 0;
    r.image = a.image; r.bg_weight = a.bg_weight;
    r.ids = a.ids; r.z = a.z; r.clos = a.clos; r.log_denom = a.log_denom;
    r.status = (long long *)(a.ws + L.status);
    const int d = r.d, mode = a.cam.mode;
    ProfScope ps(KID_RASTER, s);
    if (d == 3) launch_k<3>(r, L.n_tiles, mode, s);
    else if (d <= 4) launch_k<4>(r, L.n_tiles, mode, s);
    else if (d <= 16) launch_k<16>(r, L.n_tiles, mode, s);
    else launch_k<32>(r, L.n_tiles, mode, s);
    count_launch();
    return cudaGetLastError();
}

}  // namespace ss
