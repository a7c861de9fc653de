// Backward kernels for sm_100a.
//
//   k_backward   reference _hit_gradients + _accumulate_tiles (grad.py:89-179, :210-259):
//                one thread per pixel re-creates the blend weights of its K stored hits from
//                (z, closeness, opacity, log_denom), forms the Eq.1 partials in float32 and
//                runs the ray-geometry chain in float64 (the reference's |c| ~ 40, dist ~ 0.03
//                cancellation costs float32 2e-4 per hit).  Per-sphere sums go to an AoS row
//                [g_center(3), d_radius | d_opacity, g_focal, g_sensor, count | d_feature(d)]
//                with 128-bit vector reductions (red.global.add.v4.f32).
//   k_finalize   reference accumulate_and_normalize + gate_small_spheres (grad.py:262-320):
//                per-sphere normalisation, rotation to world, gating, and the block-reduced
//                camera sums (translation, dL/dR, focal, sensor) in float64.
#include <math.h>

#include "ss_common.cuh"

namespace ss {

namespace {

struct BackArgs {
    Cam cam;
    const Rec *rec;
    const float *feat, *bg;
    const int *ids; const float *z, *clos, *log_denom, *upstream;
    float *raw; int raw_stride;
    int d, K;
    double gamma, eps_over_g;
};

__device__ __forceinline__ void red_add_v4(float *addr, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}

template <int DP, int MODE>
__global__ void __launch_bounds__(TILE_PX) k_backward(BackArgs a) {
    const Cam &cam = a.cam;
    const int tile = blockIdx.x;
    const int tid = threadIdx.x;
    const int px = (tile % cam.ntx) * TILE + (tid & (TILE - 1));
    const int py = (tile / cam.ntx) * TILE + (tid >> 4);
    if (!(px < cam.W && py < cam.H)) return;
    const size_t P = (size_t)cam.W * cam.H;
    const size_t pix = (size_t)py * cam.W + px;
    const int K = a.K, d = a.d;

    if (a.ids[pix] < 0) {  // slots are filled front to back: an empty slot 0 means no hit
        bool any = false;
        for (int k = 1; k < K; ++k) any |= a.ids[k * P + pix] >= 0;
        if (!any) return;
    }
    const float ld = a.log_denom[pix];
    const float inv_g = (float)(1.0 / a.gamma);
    float up[DP], fhat[DP];
    const float w_bg = expf((float)a.eps_over_g - ld);
#pragma unroll
    for (int i = 0; i < DP; ++i) {
        up[i] = i < d ? a.upstream[pix * d + i] : 0.0f;
        fhat[i] = i < d ? w_bg * a.bg[i] : 0.0f;
    }
    // f_hat from the stored slots only (grad.py:103-108)
    for (int k = 0; k < K; ++k) {
        const int id = a.ids[k * P + pix];
        if (id < 0) continue;
        const float o = a.rec[id].o;
        const float E = expf(o * a.z[k * P + pix] * inv_g - ld);
        const float w = o * a.clos[k * P + pix] * E;
        const float *f = a.feat + (size_t)id * d;
#pragma unroll
        for (int i = 0; i < DP; ++i)
            if (i < d) fhat[i] = fmaf(w, f[i], fhat[i]);
    }

    // ray (camera.py:332-357)
    const double xs = ((px + 0.5) - cam.W / 2.0) * cam.pix;
    const double ys = ((py + 0.5) - cam.H / 2.0) * cam.pix;
    double ux = 0.0, uy = 0.0, uz = 1.0, inv_vnorm = 1.0;
    if (MODE == SS_MODE_PINHOLE) {
        const double vn = sqrt(xs * xs + ys * ys + cam.focal * cam.focal);
        ux = xs / vn; uy = ys / vn; uz = cam.focal / vn; inv_vnorm = 1.0 / vn;
    }

    for (int k = 0; k < K; ++k) {
        const int id = a.ids[k * P + pix];
        if (id < 0) continue;
        const Rec rc = a.rec[id];
        const float o = rc.o;
        const float zk = a.z[k * P + pix], ck = a.clos[k * P + pix];
        const float ez = o * zk * inv_g;
        const float E = expf(ez - ld);
        const float w = o * ck * E;
        const float *f = a.feat + (size_t)id * d;
        float acoef = 0.0f;
#pragma unroll
        for (int i = 0; i < DP; ++i)
            if (i < d) acoef = fmaf(up[i], f[i] - fhat[i], acoef);
        const double dl_dz = (double)(acoef * w * o * inv_g);
        const double dl_dc = (double)(acoef * o * E);
        const float dl_do = acoef * ck * E * (1.0f + ez);

        // geometry chain, float64 (grad.py:117-165)
        const double r = (double)rc.r;
        double t, dvx, dvy, dvz;
        if (MODE == SS_MODE_PINHOLE) {
            t = rc.cx * ux + rc.cy * uy + rc.cz * uz;
            dvx = rc.cx - t * ux; dvy = rc.cy - t * uy; dvz = rc.cz - t * uz;
        } else {
            t = rc.cz;
            dvx = rc.cx - xs; dvy = rc.cy - ys; dvz = 0.0;
        }
        const double dist = sqrt(fmax(dvx * dvx + dvy * dvy + dvz * dvz, 0.0));
        const bool interior = (0.0f < zk) && (zk < 1.0f);
        const double dl_dzeta = interior ? dl_dz * (-cam.inv_range) : 0.0;
        const double dl_ddist = -dl_dc / fmax(r, 1e-300);
        const double d_radius = dl_dc * dist / fmax(r * r, 1e-300);
        const double inv_dist = dist > 1e-12 ? 1.0 / dist : 0.0;
        const double hx = dvx * inv_dist, hy = dvy * inv_dist, hz = dvz * inv_dist;
        double gcx, gcy, gcz, g_focal, g_sensor;
        if (MODE == SS_MODE_PINHOLE) {
            const double zu = dl_dzeta * uz;
            gcx = dl_ddist * hx + zu * ux;
            gcy = dl_ddist * hy + zu * uy;
            gcz = dl_ddist * hz + zu * uz;
            const double s1 = dl_ddist * (-t) * inv_dist + zu;
            const double gux = s1 * rc.cx, guy = s1 * rc.cy, guz = s1 * rc.cz + dl_dzeta * t;
            const double gdu = gux * ux + guy * uy + guz * uz;
            const double prx = gux - gdu * ux, pry = guy - gdu * uy, prz = guz - gdu * uz;
            g_focal = prz * inv_vnorm;
            g_sensor = (prx * xs + pry * ys) * inv_vnorm / cam.sensor_w;
        } else {
            gcx = dl_ddist * hx; gcy = dl_ddist * hy; gcz = dl_ddist * hz + dl_dzeta;
            g_sensor = -(dl_ddist * inv_dist) * (dvx * xs + dvy * ys) / cam.sensor_w;
            g_focal = 0.0;
        }
        float *row = a.raw + (size_t)id * a.raw_stride;
        red_add_v4(row, (float)gcx, (float)gcy, (float)gcz, (float)d_radius);
        red_add_v4(row + 4, dl_do, (float)g_focal, (float)g_sensor, 1.0f);
#pragma unroll
        for (int i = 0; i < DP; i += 4) {
            if (i < d) {  // DP is a multiple of 4 and up[] is zero beyond d
                const float v0 = w * up[i], v1 = w * up[i + 1], v2 = w * up[i + 2], v3 = w * up[i + 3];
                red_add_v4(row + 8 + i, v0, v1, v2, v3);
            }
        }
    }
}

struct FinArgs {
    long long M; int d, raw_stride;
    Cam cam;
    const float *pos;
    const float *raw;
    const double *proj_r;
    float *d_pos, *d_rad, *d_opa, *d_feat; int *pixel_count;
    double *cam_part; double *cam_grad;
    int normalize, gate, cam_grads, accumulate;
};

__global__ void __launch_bounds__(256) k_finalize(FinArgs a) {
    __shared__ double s_part[8][CAM_VALS];
    __shared__ int s_last;
    const Cam &cam = a.cam;
    const double *R = cam.R;
    double acc[14];
#pragma unroll
    for (int j = 0; j < 14; ++j) acc[j] = 0.0;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < a.M; i += stride) {
        const float4 *row = (const float4 *)(a.raw + (size_t)i * a.raw_stride);
        const float4 r0 = row[0], r1 = row[1];
        const float cnt = r1.w;
        float dp0 = 0.f, dp1 = 0.f, dp2 = 0.f, drad = 0.f, dopa = 0.f;
        if (cnt > 0.0f) {
            double div = 1.0, cam_scale = 1.0;
            const double pr = a.proj_r[i];
            if (a.normalize) {
                div = (double)cnt;
                cam_scale = 1e-3 / fmax(3.14159265358979323846 * (pr * pr), 1.0);
            }
            const double gx = r0.x, gy = r0.y, gz = r0.z;
            const double inv_div = 1.0 / div;
            dp0 = (float)((gx * R[0] + gy * R[3] + gz * R[6]) * inv_div);
            dp1 = (float)((gx * R[1] + gy * R[4] + gz * R[7]) * inv_div);
            dp2 = (float)((gx * R[2] + gy * R[5] + gz * R[8]) * inv_div);
            drad = (float)((double)r0.w * inv_div);
            dopa = (float)((double)r1.x * inv_div);
            if (a.gate && pr <= 3.0) { dp0 = dp1 = dp2 = 0.f; drad = 0.f; }  // grad.py:305-320
            const float *fr = a.raw + (size_t)i * a.raw_stride + 8;
            for (int k = 0; k < a.d; ++k) {
                float v = (float)((double)fr[k] * inv_div);
                if (a.accumulate) a.d_feat[(size_t)i * a.d + k] += v; else a.d_feat[(size_t)i * a.d + k] = v;
            }
            if (a.cam_grads) {
                const double sx = cam_scale * gx, sy = cam_scale * gy, sz = cam_scale * gz;
                const double rx = (double)a.pos[3 * i] - cam.t[0], ry = (double)a.pos[3 * i + 1] - cam.t[1],
                             rz = (double)a.pos[3 * i + 2] - cam.t[2];
                acc[0] += sx; acc[1] += sy; acc[2] += sz;
                acc[3] += sx * rx; acc[4] += sx * ry; acc[5] += sx * rz;
                acc[6] += sy * rx; acc[7] += sy * ry; acc[8] += sy * rz;
                acc[9] += sz * rx; acc[10] += sz * ry; acc[11] += sz * rz;
                acc[12] += cam_scale * (double)r1.y;
                acc[13] += cam_scale * (double)r1.z;
            }
        } else if (!a.accumulate) {
            for (int k = 0; k < a.d; ++k) a.d_feat[(size_t)i * a.d + k] = 0.0f;
        }
        if (a.accumulate) {
            if (cnt > 0.0f) {
                a.d_pos[3 * i] += dp0; a.d_pos[3 * i + 1] += dp1; a.d_pos[3 * i + 2] += dp2;
                a.d_rad[i] += drad; a.d_opa[i] += dopa; a.pixel_count[i] += (int)cnt;
            }
        } else {
            a.d_pos[3 * i] = dp0; a.d_pos[3 * i + 1] = dp1; a.d_pos[3 * i + 2] = dp2;
            a.d_rad[i] = drad; a.d_opa[i] = dopa; a.pixel_count[i] = (int)cnt;
        }
    }
    if (!a.cam_grads) return;
    // block reduction of the 14 camera sums, then a fixed-order final pass by the last block
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int j = 0; j < 14; ++j) {
        double v = acc[j];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) s_part[wid][j] = v;
    }
    __syncthreads();
    if (threadIdx.x < 14) {
        double v = 0.0;
        for (int w = 0; w < 8; ++w) v += s_part[w][threadIdx.x];
        a.cam_part[(size_t)blockIdx.x * CAM_VALS + threadIdx.x] = v;
    }
    __threadfence();
    __syncthreads();
    unsigned int *counter = (unsigned int *)(a.cam_part + (size_t)CAM_BLOCKS_MAX * CAM_VALS);
    if (threadIdx.x == 0) s_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    __shared__ double s_tot[14];
    if (threadIdx.x < 14) {
        double v = 0.0;
        for (unsigned b = 0; b < gridDim.x; ++b) v += a.cam_part[(size_t)b * CAM_VALS + threadIdx.x];
        s_tot[threadIdx.x] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        *counter = 0;  // ready for the next call
        for (int j = 0; j < 3; ++j)  // d_translation = -(sum sc) @ R  (grad.py:289)
            a.cam_grad[j] = -(s_tot[0] * R[0 + j] + s_tot[1] * R[3 + j] + s_tot[2] * R[6 + j]);
        for (int j = 0; j < 9; ++j) a.cam_grad[3 + j] = s_tot[3 + j];
        a.cam_grad[12] = s_tot[12];
        a.cam_grad[13] = s_tot[13];
        a.cam_grad[14] = 0.0; a.cam_grad[15] = 0.0;
    }
}

template <int DP>
void launch_bw_mode(const BackArgs &b, int n_tiles, int mode, cudaStream_t s) {
    if (mode == SS_MODE_PINHOLE) k_backward<DP, SS_MODE_PINHOLE><<<n_tiles, TILE_PX, 0, s>>>(b);
    else k_backward<DP, SS_MODE_ORTHOGRAPHIC><<<n_tiles, TILE_PX, 0, s>>>(b);
}

}  // namespace

cudaError_t launch_backward(const BwdLaunch &a, cudaStream_t s) {
    const Layout &L = a.L;
    const long long M = a.dims.num_spheres;
    const bool cam_grads = (a.blend.flags & SS_OPT_CAMERA_GRADS) != 0;
    if (M <= 0) {  // empty scene: zero camera gradients (reference tests/test_grad.py:175-184)
        if (cam_grads && a.cam_grad) return cudaMemsetAsync(a.cam_grad, 0, 16 * sizeof(double), s);
        return cudaSuccess;
    }
    float *raw = (float *)(a.ws + L.raw);
    cudaError_t e;
    {
        ProfScope ps(KID_MEMSET_BWD, s);
        e = cudaMemsetAsync(raw, 0, (size_t)M * L.raw_stride * sizeof(float), s);
        if (e != cudaSuccess) return e;
        e = cudaMemsetAsync(a.ws + L.cam_part + (size_t)CAM_BLOCKS_MAX * CAM_VALS * 8, 0, 16, s);
        if (e != cudaSuccess) return e;
    }
    BackArgs b;
    b.cam = a.cam;
    b.rec = (const Rec *)(a.ws + L.rec);
    b.feat = a.feat; b.bg = a.bg;
    b.ids = a.ids; b.z = a.z; b.clos = a.clos; b.log_denom = a.log_denom; b.upstream = a.upstream;
    b.raw = raw; b.raw_stride = L.raw_stride;
    b.d = a.dims.feature_dim; b.K = a.dims.top_k;
    b.gamma = a.gamma; b.eps_over_g = a.blend.eps / a.gamma;
    const int d = b.d, mode = a.cam.mode;
    {
        ProfScope ps(KID_BACKWARD, s);
        if (d <= 4) launch_bw_mode<4>(b, L.n_tiles, mode, s);
        else if (d <= 16) launch_bw_mode<16>(b, L.n_tiles, mode, s);
        else launch_bw_mode<32>(b, L.n_tiles, mode, s);
    }

    FinArgs f;
    f.M = M; f.d = d; f.raw_stride = L.raw_stride;
    f.cam = a.cam; f.pos = a.pos; f.raw = raw;
    f.proj_r = (const double *)(a.ws + L.proj_r);
    f.d_pos = a.d_pos; f.d_rad = a.d_rad; f.d_opa = a.d_opa; f.d_feat = a.d_feat;
    f.pixel_count = a.pixel_count;
    f.cam_part = (double *)(a.ws + L.cam_part);
    f.cam_grad = a.cam_grad;
    f.normalize = (a.blend.flags & SS_OPT_NORMALIZE) ? 1 : 0;
    f.gate = (a.blend.flags & SS_OPT_GATE) ? 1 : 0;
    f.cam_grads = cam_grads ? 1 : 0;
    f.accumulate = (a.blend.flags & SS_OPT_ACCUMULATE) ? 1 : 0;
    long long blocks = (M + 255) / 256;
    int grid = (int)(blocks < CAM_BLOCKS_MAX ? blocks : CAM_BLOCKS_MAX);
    {
        ProfScope ps(KID_FINALIZE, s);
        k_finalize<<<grid, 256, 0, s>>>(f);
    }
    count_launch(2);
    return cudaGetLastError();
}

}  // namespace ss
