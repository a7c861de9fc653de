// the step either side of the render path in every training iteration
// (reference softsphere/optim.py), as two HBM-bound elementwise kernels:
//
//   k_photometric  photometric_loss (optim.py:87-97): mean |rendered - target| and its subgradient
//                  image sign(diff) / n, which is the `upstream` of ss_backward.
//   k_fit_step     consumes k_finalize's output directly: opacity-depth regulariser gradients
//                  (optim.py:100-121) added to d_position / d_opacity, visibility += pixel_count
//                  (optim.py:307), and the four per-group bias-corrected Adam updates with the radius
//                  floor (optim.py:142-154, :309-329) -- one pass over the M spheres instead of ~12.
//   k_adam_flat    adam_step on one flat array (camera vectors, parity with the reference function).
#include <math.h>

#include "ss_common.cuh"

namespace ss {

namespace {

__global__ void __launch_bounds__(256) k_photometric(const float *__restrict__ image,
                                                     const float *__restrict__ target, float *upstream,
                                                     long long n, double inv_n, double *loss_sum) {
    __shared__ double s_w[8];
    const float inv_nf = (float)inv_n;
    double acc = 0.0;
    const long long stride = (long long)gridDim.x * blockDim.x * 4;
    for (long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < n; i += stride) {
        if (i + 3 < n) {
            const float4 a = *reinterpret_cast<const float4 *>(image + i);
            const float4 b = *reinterpret_cast<const float4 *>(target + i);
            const float d0 = a.x - b.x, d1 = a.y - b.y, d2 = a.z - b.z, d3 = a.w - b.w;
            acc += (double)(fabsf(d0) + fabsf(d1)) + (double)(fabsf(d2) + fabsf(d3));
            float4 u;
            u.x = (d0 > 0.f) ? inv_nf : (d0 < 0.f ? -inv_nf : 0.f);
            u.y = (d1 > 0.f) ? inv_nf : (d1 < 0.f ? -inv_nf : 0.f);
            u.z = (d2 > 0.f) ? inv_nf : (d2 < 0.f ? -inv_nf : 0.f);
            u.w = (d3 > 0.f) ? inv_nf : (d3 < 0.f ? -inv_nf : 0.f);
            *reinterpret_cast<float4 *>(upstream + i) = u;
        } else {
            for (long long j = i; j < n; ++j) {
                const float dj = image[j] - target[j];
                acc += (double)fabsf(dj);
                upstream[j] = (dj > 0.f) ? inv_nf : (dj < 0.f ? -inv_nf : 0.f);
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double v = 0.0;
        for (int w = 0; w < 8; ++w) v += s_w[w];
        atomicAdd(loss_sum, v * inv_n);
    }
}

struct Betas { float b1, b2, omb1, omb2; };  // 1 - beta is rounded from float64: 1.0f - 0.999f is off by 1.3e-5

__device__ __forceinline__ float adam_update(float p, float g, float &m, float &v, Betas b, float lr_over_bc1,
                                             float inv_sqrt_bc2, float eps) {
    m = b.b1 * m + b.omb1 * g;
    v = b.b2 * v + b.omb2 * g * g;
    // p - lr * (m / bc1) / (sqrt(v / bc2) + eps)
    return p - lr_over_bc1 * m / (sqrtf(v) * inv_sqrt_bc2 + eps);
}

struct FitArgs {
    long long M; int d;
    float *pos, *rad, *opa, *feat;
    const float *d_pos, *d_rad, *d_opa, *d_feat;
    const int *pixel_count; int *visibility;
    float *m_pos, *v_pos, *m_rad, *v_rad, *m_opa, *v_opa, *m_feat, *v_feat;
    float lr_over_bc1[4], inv_sqrt_bc2[4];
    int active[4];
    Betas betas; float eps, radius_min;
    double lambda_od, near_, far_, inv_range;
    double t[3], Rz[3];  // camera position and third row of R (optical axis in world coordinates)
    double *energy;
};

__global__ void __launch_bounds__(256) k_fit_step(FitArgs a) {
    __shared__ double s_w[8];
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    double energy = 0.0;
    if (i < a.M) {
        float p0 = a.pos[3 * i], p1 = a.pos[3 * i + 1], p2 = a.pos[3 * i + 2];
        const float o_raw = a.opa[i];
        float g0 = a.d_pos[3 * i], g1 = a.d_pos[3 * i + 1], g2 = a.d_pos[3 * i + 2];
        float go = a.d_opa[i];
        if (a.lambda_od != 0.0) {  // opacity-depth regulariser, optim.py:100-121
            const double zeta = ((double)p0 - a.t[0]) * a.Rz[0] + ((double)p1 - a.t[1]) * a.Rz[1] +
                                ((double)p2 - a.t[2]) * a.Rz[2];
            const double zc = fmin(fmax(zeta, a.near_), a.far_);
            const double z = (a.far_ - zc) * a.inv_range;
            const double o = fmin(fmax((double)o_raw, 0.0), 1.0);
            energy = a.lambda_od * (-z * o);
            const bool interior = zeta > a.near_ && zeta < a.far_;
            const double dzeta = interior ? a.lambda_od * o * a.inv_range : 0.0;
            g0 += (float)(dzeta * a.Rz[0]); g1 += (float)(dzeta * a.Rz[1]); g2 += (float)(dzeta * a.Rz[2]);
            go += (float)(-a.lambda_od * z);
        }
        if (a.visibility) {  // saturating: the reference sums in int64 (optim.py:307); prune only asks "> 0"
            const long long v = (long long)a.visibility[i] + (long long)a.pixel_count[i];
            a.visibility[i] = v > 0x7fffffffLL ? 0x7fffffff : (int)v;
        }
        if (a.active[0]) {
            float m0 = a.m_pos[3 * i], m1 = a.m_pos[3 * i + 1], m2 = a.m_pos[3 * i + 2];
            float v0 = a.v_pos[3 * i], v1 = a.v_pos[3 * i + 1], v2 = a.v_pos[3 * i + 2];
            p0 = adam_update(p0, g0, m0, v0, a.betas, a.lr_over_bc1[0], a.inv_sqrt_bc2[0], a.eps);
            p1 = adam_update(p1, g1, m1, v1, a.betas, a.lr_over_bc1[0], a.inv_sqrt_bc2[0], a.eps);
            p2 = adam_update(p2, g2, m2, v2, a.betas, a.lr_over_bc1[0], a.inv_sqrt_bc2[0], a.eps);
            a.pos[3 * i] = p0; a.pos[3 * i + 1] = p1; a.pos[3 * i + 2] = p2;
            a.m_pos[3 * i] = m0; a.m_pos[3 * i + 1] = m1; a.m_pos[3 * i + 2] = m2;
            a.v_pos[3 * i] = v0; a.v_pos[3 * i + 1] = v1; a.v_pos[3 * i + 2] = v2;
        }
        if (a.active[1]) {
            float m = a.m_rad[i], v = a.v_rad[i];
            const float r = adam_update(a.rad[i], a.d_rad[i], m, v, a.betas, a.lr_over_bc1[1],
                                        a.inv_sqrt_bc2[1], a.eps);
            a.rad[i] = fmaxf(r, a.radius_min);  // optim.py:315-319
            a.m_rad[i] = m; a.v_rad[i] = v;
        }
        if (a.active[2]) {
            float m = a.m_opa[i], v = a.v_opa[i];
            a.opa[i] = adam_update(o_raw, go, m, v, a.betas, a.lr_over_bc1[2], a.inv_sqrt_bc2[2], a.eps);
            a.m_opa[i] = m; a.v_opa[i] = v;
        }
        if (a.active[3]) {
            for (int k = 0; k < a.d; ++k) {
                const size_t j = (size_t)i * a.d + k;
                float m = a.m_feat[j], v = a.v_feat[j];
                a.feat[j] = adam_update(a.feat[j], a.d_feat[j], m, v, a.betas, a.lr_over_bc1[3],
                                        a.inv_sqrt_bc2[3], a.eps);
                a.m_feat[j] = m; a.v_feat[j] = v;
            }
        }
    }
    if (a.energy && a.lambda_od != 0.0) {
        for (int o = 16; o > 0; o >>= 1) energy += __shfl_xor_sync(0xffffffffu, energy, o);
        if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = energy;
        __syncthreads();
        if (threadIdx.x == 0) {
            double v = 0.0;
            for (int w = 0; w < 8; ++w) v += s_w[w];
            if (v != 0.0) atomicAdd(a.energy, v);
        }
    }
}

__global__ void __launch_bounds__(256) k_adam_flat(float *p, const float *__restrict__ g, float *m, float *v,
                                                   long long n, Betas betas, float lr_over_bc1,
                                                   float inv_sqrt_bc2, float eps, float floor_value, int use_floor) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float mi = m[i], vi = v[i];
    float x = adam_update(p[i], g[i], mi, vi, betas, lr_over_bc1, inv_sqrt_bc2, eps);
    if (use_floor) x = fmaxf(x, floor_value);
    p[i] = x; m[i] = mi; v[i] = vi;
}

}  // namespace

}  // namespace ss

using namespace ss;

extern "C" {

int ss_photometric_loss(const float *image, const float *target, float *upstream, int64_t n, double *loss_out,
                        void *stream) {
    if (!image || !target || !upstream || !loss_out) return SS_ERR_NULL;
    if (n < 0) return SS_ERR_DIMS;
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(loss_out, 0, sizeof(double), s);
    if (e != cudaSuccess) return SS_ERR_CUDA;
    if (n > 0) {
        long long blocks = (n / 4 + 255) / 256;
        int grid = (int)(blocks < 148 * 16 ? (blocks > 0 ? blocks : 1) : 148 * 16);
        k_photometric<<<grid, 256, 0, s>>>(image, target, upstream, n, 1.0 / (double)n, loss_out);
        count_launch();
    }
    return cudaGetLastError() == cudaSuccess ? SS_OK : SS_ERR_CUDA;
}

int ss_fit_step(const SsFitStepArgs *a, void *stream) {
    if (!a) return SS_ERR_NULL;
    if (a->num_spheres < 0 || a->feature_dim < 1 || a->feature_dim > SS_MAX_FEATURE_DIM) return SS_ERR_DIMS;
    if (!(a->beta1 >= 0.0 && a->beta1 < 1.0) || !(a->beta2 >= 0.0 && a->beta2 < 1.0) || !(a->adam_eps >= 0.0))
        return SS_ERR_PARAMS;
    if (a->num_spheres == 0) {
        if (a->energy) return cudaMemsetAsync(a->energy, 0, sizeof(double), (cudaStream_t)stream) == cudaSuccess ? SS_OK : SS_ERR_CUDA;
        return SS_OK;
    }
    if (!a->pos || !a->rad || !a->opa || !a->feat || !a->d_pos || !a->d_rad || !a->d_opa || !a->d_feat) return SS_ERR_NULL;
    if (a->visibility && !a->pixel_count) return SS_ERR_NULL;
    FitArgs f;
    f.M = a->num_spheres; f.d = a->feature_dim;
    f.pos = a->pos; f.rad = a->rad; f.opa = a->opa; f.feat = a->feat;
    f.d_pos = a->d_pos; f.d_rad = a->d_rad; f.d_opa = a->d_opa; f.d_feat = a->d_feat;
    f.pixel_count = a->pixel_count; f.visibility = a->visibility;
    f.m_pos = a->m_pos; f.v_pos = a->v_pos; f.m_rad = a->m_rad; f.v_rad = a->v_rad;
    f.m_opa = a->m_opa; f.v_opa = a->v_opa; f.m_feat = a->m_feat; f.v_feat = a->v_feat;
    float *ms[4] = {a->m_pos, a->m_rad, a->m_opa, a->m_feat};
    float *vs[4] = {a->v_pos, a->v_rad, a->v_opa, a->v_feat};
    for (int g = 0; g < 4; ++g) {
        f.active[g] = a->lr[g] > 0.0 ? 1 : 0;  // lr = 0 freezes the group (optim.py:309-329)
        if (f.active[g]) {
            if (!ms[g] || !vs[g] || a->step[g] < 1) return SS_ERR_PARAMS;
            const double bc1 = 1.0 - pow(a->beta1, (double)a->step[g]);
            const double bc2 = 1.0 - pow(a->beta2, (double)a->step[g]);
            f.lr_over_bc1[g] = (float)(a->lr[g] / bc1);
            f.inv_sqrt_bc2[g] = (float)(1.0 / sqrt(bc2));
        } else {
            f.lr_over_bc1[g] = 0.f; f.inv_sqrt_bc2[g] = 1.f;
        }
    }
    f.betas = Betas{(float)a->beta1, (float)a->beta2, (float)(1.0 - a->beta1), (float)(1.0 - a->beta2)};
    f.eps = (float)a->adam_eps;
    f.radius_min = (float)a->radius_min;
    f.lambda_od = a->lambda_od; f.near_ = a->cam.near_; f.far_ = a->cam.far_;
    f.inv_range = 1.0 / (a->cam.far_ - a->cam.near_);
    for (int j = 0; j < 3; ++j) { f.t[j] = a->cam.t[j]; f.Rz[j] = a->cam.R[6 + j]; }
    f.energy = a->energy;
    cudaStream_t s = (cudaStream_t)stream;
    if (a->energy) {
        if (cudaMemsetAsync(a->energy, 0, sizeof(double), s) != cudaSuccess) return SS_ERR_CUDA;
    }
    k_fit_step<<<(unsigned)((f.M + 255) / 256), 256, 0, s>>>(f);
    count_launch();
    return cudaGetLastError() == cudaSuccess ? SS_OK : SS_ERR_CUDA;
}

int ss_adam_flat(float *params, const float *grads, float *m, float *v, int64_t n, double lr, double beta1,
                 double beta2, double adam_eps, int64_t step, int use_floor, double floor_value, void *stream) {
    if (n < 0) return SS_ERR_DIMS;
    if (n == 0) return SS_OK;
    if (!params || !grads || !m || !v) return SS_ERR_NULL;
    if (step < 1 || !(beta1 >= 0.0 && beta1 < 1.0) || !(beta2 >= 0.0 && beta2 < 1.0)) return SS_ERR_PARAMS;
    const double bc1 = 1.0 - pow(beta1, (double)step), bc2 = 1.0 - pow(beta2, (double)step);
    k_adam_flat<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        params, grads, m, v, n, Betas{(float)beta1, (float)beta2, (float)(1.0 - beta1), (float)(1.0 - beta2)},
        (float)(lr / bc1), (float)(1.0 / sqrt(bc2)),
        (float)adam_eps, (float)floor_value, use_floor);
    count_launch();
    return cudaGetLastError() == cudaSuccess ? SS_OK : SS_ERR_CUDA;
}

}  // extern "C"
