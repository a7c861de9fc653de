// the per-pixel shading stage that consumes the feature map (reference
// softsphere/shade.py), forward and backward, as HBM-bound per-pixel kernels:
//
//   k_shade_identity[_bwd]  shade_identity / shade_identity_backward      shade.py:66-77
//   k_shade_diffuse[_bwd]   shade_diffuse / shade_diffuse_backward        shade.py:84-131  ([albedo:3, normal:3])
//   k_shade_linear          shade_linear (optionally view-conditioned)    shade.py:148-157
//   k_shade_linear_bwd      shade_linear_backward: d_features per pixel, d_weight = x^T up and d_bias = sum up
//                           reduced in shared memory / registers by persistent CTAs, one float64 atomic per entry and CTA
//                                                                         shade.py:160-171
//   k_view_dirs             view_direction_plane                          shade.py:138-142, camera.py:332-357
//
// Arithmetic is float32 (the feature map is float32); the clamp masks use the same closed interval [0, 1]
// as the reference's _clamp01_mask.  Bytes per pixel: identity 24 / 36 (fwd / bwd), diffuse 36 / 60,
// linear 4 (d [+3]) + 12 / 4 (2 d [+3]) + 12.
#include <math.h>

#include "ss_common.cuh"

namespace ss {

namespace {

constexpr int MAX_LIGHTS = 8;
struct Lights {
    float nx[MAX_LIGHTS], ny[MAX_LIGHTS], nz[MAX_LIGHTS];  // -direction (unit)
    float intensity[MAX_LIGHTS], ambient[MAX_LIGHTS];
    int n;
};

__device__ __forceinline__ float clamp01(float x) { return fminf(fmaxf(x, 0.0f), 1.0f); }
__device__ __forceinline__ bool in01(float x) { return x >= 0.0f && x <= 1.0f; }

__global__ void __launch_bounds__(256) k_shade_identity(const float *__restrict__ f, float *out, long long n) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = clamp01(f[i]);
}

__global__ void __launch_bounds__(256) k_shade_identity_bwd(const float *__restrict__ f,
                                                            const float *__restrict__ up, float *d_f, long long n) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        d_f[i] = in01(f[i]) ? up[i] : 0.0f;
}

struct DiffuseParts {
    float ax, ay, az, hx, hy, hz, norm, shade;
    bool ok;
};

__device__ __forceinline__ DiffuseParts diffuse_parts(const float *__restrict__ f, const Lights &L) {
    DiffuseParts p;
    p.ax = f[0]; p.ay = f[1]; p.az = f[2];
    const float nx = f[3], ny = f[4], nz = f[5];
    p.norm = sqrtf(nx * nx + ny * ny + nz * nz);
    p.ok = p.norm > 1e-12f;
    const float inv = p.ok ? 1.0f / p.norm : 0.0f;
    p.hx = nx * inv; p.hy = ny * inv; p.hz = nz * inv;
    float s = 0.0f;
    for (int l = 0; l < L.n; ++l)
        s += L.ambient[l] + L.intensity[l] * fmaxf(0.0f, p.hx * L.nx[l] + p.hy * L.ny[l] + p.hz * L.nz[l]);
    p.shade = s;
    return p;
}

__global__ void __launch_bounds__(256) k_shade_diffuse(const float *__restrict__ img, long long n_px, Lights L,
                                                       float *out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_px) return;
    const DiffuseParts p = diffuse_parts(img + i * 6, L);
    out[i * 3] = clamp01(p.ax * p.shade);
    out[i * 3 + 1] = clamp01(p.ay * p.shade);
    out[i * 3 + 2] = clamp01(p.az * p.shade);
}

__global__ void __launch_bounds__(256) k_shade_diffuse_bwd(const float *__restrict__ img,
                                                           const float *__restrict__ up, long long n_px, Lights L,
                                                           float *d_img) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_px) return;
    const DiffuseParts p = diffuse_parts(img + i * 6, L);
    const float u0 = in01(p.ax * p.shade) ? up[i * 3] : 0.0f;
    const float u1 = in01(p.ay * p.shade) ? up[i * 3 + 1] : 0.0f;
    const float u2 = in01(p.az * p.shade) ? up[i * 3 + 2] : 0.0f;
    const float d_shade = u0 * p.ax + u1 * p.ay + u2 * p.az;
    float gx = 0.0f, gy = 0.0f, gz = 0.0f;  // d loss / d n_hat
    for (int l = 0; l < L.n; ++l) {
        const bool lit = p.hx * L.nx[l] + p.hy * L.ny[l] + p.hz * L.nz[l] > 0.0f;
        const float s = lit ? d_shade * L.intensity[l] : 0.0f;
        gx += s * L.nx[l]; gy += s * L.ny[l]; gz += s * L.nz[l];
    }
    // through n_hat = n / |n|
    const float dot = gx * p.hx + gy * p.hy + gz * p.hz;
    const float inv = p.ok ? 1.0f / p.norm : 0.0f;
    float *o = d_img + i * 6;
    o[0] = u0 * p.shade; o[1] = u1 * p.shade; o[2] = u2 * p.shade;
    o[3] = (gx - dot * p.hx) * inv; o[4] = (gy - dot * p.hy) * inv; o[5] = (gz - dot * p.hz) * inv;
}

constexpr int MAX_IN = SS_MAX_FEATURE_DIM + 3;

__global__ void __launch_bounds__(256) k_shade_linear(const float *__restrict__ img,
                                                      const float *__restrict__ view, long long n_px, int d,
                                                      const float *__restrict__ weight,
                                                      const float *__restrict__ bias, float *out) {
    __shared__ float s_w[MAX_IN * 3 + 3];
    const int d_in = d + (view ? 3 : 0);
    for (int e = threadIdx.x; e < d_in * 3; e += blockDim.x) s_w[e] = weight[e];
    if (threadIdx.x < 3) s_w[MAX_IN * 3 + threadIdx.x] = bias[threadIdx.x];
    __syncthreads();
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_px) return;
    float a0 = s_w[MAX_IN * 3], a1 = s_w[MAX_IN * 3 + 1], a2 = s_w[MAX_IN * 3 + 2];
    const float *x = img + i * d;
    if ((d & 3) == 0) {  // 128-bit loads: a pixel's row is 4 d contiguous bytes
        for (int k = 0; k < d; k += 4) {
            const float4 q = *reinterpret_cast<const float4 *>(x + k);
            const float v[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                a0 = fmaf(v[j], s_w[3 * (k + j)], a0); a1 = fmaf(v[j], s_w[3 * (k + j) + 1], a1);
                a2 = fmaf(v[j], s_w[3 * (k + j) + 2], a2);
            }
        }
    } else {
        for (int k = 0; k < d; ++k) {
            const float v = x[k];
            a0 = fmaf(v, s_w[3 * k], a0); a1 = fmaf(v, s_w[3 * k + 1], a1); a2 = fmaf(v, s_w[3 * k + 2], a2);
        }
    }
    if (view) {
        for (int k = 0; k < 3; ++k) {
            const float v = view[i * 3 + k];
            a0 = fmaf(v, s_w[3 * (d + k)], a0); a1 = fmaf(v, s_w[3 * (d + k) + 1], a1);
            a2 = fmaf(v, s_w[3 * (d + k) + 2], a2);
        }
    }
    out[i * 3] = clamp01(a0); out[i * 3 + 1] = clamp01(a1); out[i * 3 + 2] = clamp01(a2);
}

__global__ void __launch_bounds__(256) k_shade_linear_bwd(const float *__restrict__ img,
                                                          const float *__restrict__ view, long long n_px, int d,
                                                          const float *__restrict__ weight,
                                                          const float *__restrict__ bias,
                                                          const float *__restrict__ up, float *d_img,
                                                          double *d_weight, double *d_bias) {
    extern __shared__ float s_dyn[];
    __shared__ float s_w[MAX_IN * 3 + 3];
    const int d_in = d + (view ? 3 : 0);
    const int xst = d_in | 1;             // odd row stride: a thread's row starts in its own bank
    float *s_x = s_dyn;                   // [256][xst]   inputs of this block's pixels
    float *s_u = s_dyn + 256 * xst;       // [256][3]     masked upstream
    for (int e = threadIdx.x; e < d_in * 3; e += blockDim.x) s_w[e] = weight[e];
    if (threadIdx.x < 3) s_w[MAX_IN * 3 + threadIdx.x] = bias[threadIdx.x];
    __syncthreads();
    // entry (k, c) of x^T up (entries d_in*3 .. +2: the bias sums), split over the 256 threads as (entry,
    // pixel-slice) pairs.  The CTA walks its pixel blocks and keeps the partial sums in registers: one float64
    // atomic per entry, slice and CTA at the very end (an atomic per 256-pixel block would put 16 K same-address
    // atomics on each of the ~50 entries and the kernel would wait on the L2: measured 136 us vs 40 us).
    const int t = threadIdx.x;
    const int n_ent = d_in * 3 + 3;
    const int slices = 256 / n_ent >= 8 ? 8 : (256 / n_ent >= 4 ? 4 : (256 / n_ent >= 2 ? 2 : 1));
    const int ent = t / slices, sl = t - ent * slices;
    const int ek = ent / 3, ec = ent - 3 * ek;
    float acc = 0.0f;
    float *xs = s_x + t * xst;
    const long long n_blocks = (n_px + 255) / 256;
    for (long long blk = blockIdx.x; blk < n_blocks; blk += gridDim.x) {
        const long long i = blk * 256 + t;
        const bool in = i < n_px;
        float u0 = 0.0f, u1 = 0.0f, u2 = 0.0f;
        if (in) {
            float a0 = s_w[MAX_IN * 3], a1 = s_w[MAX_IN * 3 + 1], a2 = s_w[MAX_IN * 3 + 2];
            const bool vec = (d & 3) == 0;
            if (vec)
                for (int k = 0; k < d; k += 4) {
                    const float4 q = *reinterpret_cast<const float4 *>(img + i * d + k);
                    xs[k] = q.x; xs[k + 1] = q.y; xs[k + 2] = q.z; xs[k + 3] = q.w;
                }
            for (int k = 0; k < d_in; ++k) {
                const float v = k < d ? (vec ? xs[k] : img[i * d + k]) : view[i * 3 + (k - d)];
                xs[k] = v;
                a0 = fmaf(v, s_w[3 * k], a0); a1 = fmaf(v, s_w[3 * k + 1], a1); a2 = fmaf(v, s_w[3 * k + 2], a2);
            }
            u0 = in01(a0) ? up[i * 3] : 0.0f;
            u1 = in01(a1) ? up[i * 3 + 1] : 0.0f;
            u2 = in01(a2) ? up[i * 3 + 2] : 0.0f;
            if (vec) {
                for (int k = 0; k < d; k += 4) {
                    float4 q;
                    q.x = u0 * s_w[3 * k] + u1 * s_w[3 * k + 1] + u2 * s_w[3 * k + 2];
                    q.y = u0 * s_w[3 * k + 3] + u1 * s_w[3 * k + 4] + u2 * s_w[3 * k + 5];
                    q.z = u0 * s_w[3 * k + 6] + u1 * s_w[3 * k + 7] + u2 * s_w[3 * k + 8];
                    q.w = u0 * s_w[3 * k + 9] + u1 * s_w[3 * k + 10] + u2 * s_w[3 * k + 11];
                    *reinterpret_cast<float4 *>(d_img + i * d + k) = q;
                }
            } else {
                for (int k = 0; k < d; ++k)
                    d_img[i * d + k] = u0 * s_w[3 * k] + u1 * s_w[3 * k + 1] + u2 * s_w[3 * k + 2];
            }
        } else {
            for (int k = 0; k < d_in; ++k) xs[k] = 0.0f;
        }
        if (!d_weight) continue;
        s_u[t * 3] = u0; s_u[t * 3 + 1] = u1; s_u[t * 3 + 2] = u2;
        __syncthreads();
        if (ent < n_ent) {
            if (ek < d_in) {
                for (int p = sl; p < 256; p += slices) acc = fmaf(s_x[p * xst + ek], s_u[p * 3 + ec], acc);
            } else {
                for (int p = sl; p < 256; p += slices) acc += s_u[p * 3 + ec];
            }
        }
        __syncthreads();
    }
    if (d_weight && ent < n_ent && acc != 0.0f) {
        if (ek < d_in) atomicAdd(d_weight + ent, (double)acc);
        else atomicAdd(d_bias + ec, (double)acc);
    }
}

__global__ void __launch_bounds__(256) k_view_dirs(Cam cam, float *out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)cam.W * cam.H) return;
    const int px = (int)(i % cam.W), py = (int)(i / cam.W);
    double ux = 0.0, uy = 0.0, uz = 1.0;
    if (cam.mode == SS_MODE_PINHOLE) {
        const double xs = ((px + 0.5) - cam.W / 2.0) * cam.pix;
        const double ys = ((py + 0.5) - cam.H / 2.0) * cam.pix;
        const double vn = sqrt(xs * xs + ys * ys + cam.focal * cam.focal);
        ux = xs / vn; uy = ys / vn; uz = cam.focal / vn;
    }
    out[i * 3] = (float)ux; out[i * 3 + 1] = (float)uy; out[i * 3 + 2] = (float)uz;
}

inline int rc_of(cudaError_t e) { return e == cudaSuccess ? SS_OK : SS_ERR_CUDA; }

int make_lights(const SsLight *lights, int n, Lights &L) {
    if (n < 0 || n > MAX_LIGHTS) return SS_ERR_DIMS;
    if (n > 0 && !lights) return SS_ERR_NULL;
    L.n = n;
    for (int l = 0; l < n; ++l) {
        const double *dv = lights[l].direction;
        const double nn = sqrt(dv[0] * dv[0] + dv[1] * dv[1] + dv[2] * dv[2]);
        if (!(nn >= 1e-12) || lights[l].intensity < 0.0 || !(lights[l].ambient >= 0.0 && lights[l].ambient <= 1.0))
            return SS_ERR_PARAMS;  // ValidationError, shade.py:39-45
        L.nx[l] = (float)(-dv[0] / nn); L.ny[l] = (float)(-dv[1] / nn); L.nz[l] = (float)(-dv[2] / nn);
        L.intensity[l] = (float)lights[l].intensity; L.ambient[l] = (float)lights[l].ambient;
    }
    return SS_OK;
}

inline unsigned grid_for(long long n) {
    long long b = (n + 255) / 256;
    return (unsigned)(b < 148 * 32 ? (b > 0 ? b : 1) : 148 * 32);
}

}  // namespace

}  // namespace ss

using namespace ss;

extern "C" {

int ss_shade_identity(const float *image, int64_t n_values, float *out, void *stream) {
    if (n_values < 0) return SS_ERR_DIMS;
    if (n_values == 0) return SS_OK;
    if (!image || !out) return SS_ERR_NULL;
    k_shade_identity<<<grid_for(n_values), 256, 0, (cudaStream_t)stream>>>(image, out, n_values);
    count_launch();
    return rc_of(cudaGetLastError());
}

int ss_shade_identity_backward(const float *image, const float *upstream, int64_t n_values, float *d_image,
                               void *stream) {
    if (n_values < 0) return SS_ERR_DIMS;
    if (n_values == 0) return SS_OK;
    if (!image || !upstream || !d_image) return SS_ERR_NULL;
    k_shade_identity_bwd<<<grid_for(n_values), 256, 0, (cudaStream_t)stream>>>(image, upstream, d_image, n_values);
    count_launch();
    return rc_of(cudaGetLastError());
}

int ss_shade_diffuse(const float *image, int64_t n_pixels, const SsLight *lights, int32_t n_lights, float *out,
                     void *stream) {
    if (n_pixels < 0) return SS_ERR_DIMS;
    Lights L;
    const int rc = make_lights(lights, n_lights, L);
    if (rc != SS_OK) return rc;
    if (n_pixels == 0) return SS_OK;
    if (!image || !out) return SS_ERR_NULL;
    k_shade_diffuse<<<(unsigned)((n_pixels + 255) / 256), 256, 0, (cudaStream_t)stream>>>(image, n_pixels, L, out);
    count_launch();
    return rc_of(cudaGetLastError());
}

int ss_shade_diffuse_backward(const float *image, const float *upstream, int64_t n_pixels, const SsLight *lights,
                              int32_t n_lights, float *d_image, void *stream) {
    if (n_pixels < 0) return SS_ERR_DIMS;
    Lights L;
    const int rc = make_lights(lights, n_lights, L);
    if (rc != SS_OK) return rc;
    if (n_pixels == 0) return SS_OK;
    if (!image || !upstream || !d_image) return SS_ERR_NULL;
    k_shade_diffuse_bwd<<<(unsigned)((n_pixels + 255) / 256), 256, 0, (cudaStream_t)stream>>>(image, upstream,
                                                                                                n_pixels, L, d_image);
    count_launch();
    return rc_of(cudaGetLastError());
}

int ss_shade_linear(const float *image, const float *view_dirs, int64_t n_pixels, int32_t d, const float *weight,
                    const float *bias, float *out, void *stream) {
    if (n_pixels < 0 || d < 1 || d > SS_MAX_FEATURE_DIM) return SS_ERR_DIMS;
    if (n_pixels == 0) return SS_OK;
    if (!image || !weight || !bias || !out) return SS_ERR_NULL;
    k_shade_linear<<<(unsigned)((n_pixels + 255) / 256), 256, 0, (cudaStream_t)stream>>>(image, view_dirs, n_pixels,
                                                                                           d, weight, bias, out);
    count_launch();
    return rc_of(cudaGetLastError());
}

int ss_shade_linear_backward(const float *image, const float *view_dirs, int64_t n_pixels, int32_t d,
                             const float *weight, const float *bias, const float *upstream, float *d_image,
                             double *d_weight, double *d_bias, void *stream) {
    if (n_pixels < 0 || d < 1 || d > SS_MAX_FEATURE_DIM) return SS_ERR_DIMS;
    if ((d_weight == nullptr) != (d_bias == nullptr)) return SS_ERR_NULL;
    cudaStream_t s = (cudaStream_t)stream;
    const int d_in = d + (view_dirs ? 3 : 0);
    if (d_weight) {
        if (cudaMemsetAsync(d_weight, 0, sizeof(double) * d_in * 3, s) != cudaSuccess) return SS_ERR_CUDA;
        if (cudaMemsetAsync(d_bias, 0, sizeof(double) * 3, s) != cudaSuccess) return SS_ERR_CUDA;
    }
    if (n_pixels == 0) return SS_OK;
    if (!image || !weight || !bias || !upstream || !d_image) return SS_ERR_NULL;
    const size_t smem = (size_t)256 * ((d_in | 1) + 3) * sizeof(float);
    const long long n_blocks = (n_pixels + 255) / 256;
    const unsigned grid = (unsigned)(n_blocks < 148 * 4 ? n_blocks : 148 * 4);  // persistent: 4 CTAs per SM
    k_shade_linear_bwd<<<grid, 256, smem, s>>>(image, view_dirs, n_pixels, d, weight,
                                                                              bias, upstream, d_image, d_weight,
                                                                              d_bias);
    count_launch();
    return rc_of(cudaGetLastError());
}

int ss_view_directions(const SsCamera *cam, float *out, void *stream) {
    if (!cam || !out) return SS_ERR_NULL;
    if (cam->width < 1 || cam->height < 1 || !(cam->focal > 0.0) || !(cam->sensor_w > 0.0)) return SS_ERR_CAMERA;
    const Cam c = make_cam(*cam);
    const long long n = (long long)c.W * c.H;
    k_view_dirs<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(c, out);
    count_launch();
    return rc_of(cudaGetLastError());
}

}  // extern "C"
