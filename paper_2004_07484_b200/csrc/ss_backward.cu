// Backward kernels for sm_100a.
//
//   k_backward   reference _hit_gradients + _accumulate_tiles (grad.py:89-179, :210-259):
//                one thread per pixel re-creates the blend weights of its K stored hits from
//                (z, closeness, opacity, log_denom), forms the Eq.1 partials in float32 and
//                runs the ray-geometry chain in float64 (the reference's |c| ~ 40, dist ~ 0.03
//                cancellation costs float32 2e-4 per hit).  Per-sphere sums go to an AoS row
//                [g_center(3), d_radius | d_opacity, g_focal, g_sensor, count | d_feature(d)]
//                with 128-bit vector reductions (red.global.add.v4.f32), after the lanes of a warp
//                that hold the same sphere in a slot have been summed (match.any + pointer jumping).
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
    unsigned long long *clean_tag;
    int d, K;
    double gamma, eps_over_g;
    // SS_OPT_DETERMINISTIC: 0 = float32 L2 reductions (default); 1 = first pass, per-sphere max |addend|
    // (atomicMax on the float bits: order-independent); 2 = second pass, 64-bit fixed-point accumulation on the
    // per-sphere power-of-two grid derived from that max (integer addition is associative: bit-reproducible)
    int det;
    unsigned *det_max;
    long long *raw64;
};

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float sqrt_approx_f(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float ex2_approx_f(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Draw record through the read-only (non-coherent) path: the compiler may then hoist these loads over the
// shared-memory stores and reductions of earlier slots (a generic pointer could alias them).
__device__ __forceinline__ Rec ldg_rec(const Rec *p) {
    const double2 a = __ldg(reinterpret_cast<const double2 *>(p));
    const float4 b = __ldg(reinterpret_cast<const float4 *>(p) + 1);
    Rec r;
    r.cx = a.x; r.cy = a.y;
    r.cz = __hiloint2double(__float_as_int(b.y), __float_as_int(b.x));
    r.r = b.z; r.o = b.w;
    return r;
}

#ifndef SS_BACKWARD_MERGE
#define SS_BACKWARD_MERGE 1
#endif

__device__ __forceinline__ void red_add_v4(float *addr, float a, float b, float c, float d) {
#ifdef SS_EXPERIMENT_NO_RED  // measurement only: floor of the kernel without the reductions
    if (a == 123456.f) *addr = b + c + d;
    return;
#endif
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
                 : "memory");
}

// Deterministic accumulation of one (merged) row of NV floats into sphere `id` (see BackArgs::det).  The merged
// float sums themselves are reproducible (the warp merge depends on the data only); what is not is the ORDER
// in which different warps reach the L2.  Grid: with m = max |addend| of the sphere (2^(e-127) <= m < 2^(e-126),
// e the biased exponent), every addend is rounded to a multiple of q = 2^(e - 126 - 38); the sum of up to
// 2^24 addends (W * H <= 2^24 is enforced) stays below 2^62 quanta.
template <int NV>
__device__ __forceinline__ void det_emit(const BackArgs &a, int id, const float *v) {
    if (a.det == 1) {
        float m = 0.0f;
#pragma unroll
        for (int j = 0; j < NV; ++j)
            if (j != 7) m = fmaxf(m, fabsf(v[j]));
        atomicMax(a.det_max + id, __float_as_uint(m));
        return;
    }
    const int e = (int)(a.det_max[id] >> 23);
    const double inv_q = __hiloint2double((1023 + 164 - e) << 20, 0);  // 2^(164 - e) = 1 / q
    unsigned long long *row = reinterpret_cast<unsigned long long *>(a.raw64) + (size_t)id * a.raw_stride;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const long long iv = j == 7 ? (long long)v[7] : __double2ll_rn((double)v[j] * inv_q);
        if (iv != 0) atomicAdd(row + j, (unsigned long long)iv);
    }
}

// Per-warp accumulator cache of the any-K path (n_track up to 64).  With long records a sphere sits at DIFFERENT
// slot indices in neighbouring pixels, so the lockstep merge below finds few peers (C5: 1.8 lanes per group) and
// the 16-byte L2 reductions dominate the kernel (225 M of them, 1.8 of 3.9 ms).  Each warp therefore keeps CACHE_ROWS
// partial rows in shared memory, direct-mapped by a hash of the sphere id: a group leader adds its sums to the
// cached row of its sphere (plain shared-memory read-modify-write: one owner lane per row and instruction, the warp
// runs the slots in lockstep) and only an evicted or finally flushed row goes to the L2 as reductions.
// Rows per warp cache (8 .. 64) and resident CTAs per SM of the any-K instantiations.  Measured at C5 (k_backward, ms):
// 64 rows / 2 CTAs 3.71, 32 / 2: 3.59, 32 / 3: 3.49, 16 / 3: 3.37, 8 / 3: 3.39, no cache / 3: 4.37, 16 / 4 (64 registers,
// spills): 4.81 -- a smaller cache still catches the repeats of neighbouring slots, and the shared memory it gives back
// goes to the L1 that serves the record and feature gathers; 80 registers hold the kernel without spills.
#ifndef SS_BWD_CACHE_ROWS
#define SS_BWD_CACHE_ROWS 16
#endif
#ifndef SS_BWD_CACHE
#define SS_BWD_CACHE 1
#endif
#ifndef SS_BWD_ANYK_MINB
#define SS_BWD_ANYK_MINB 3    // resident CTAs per SM the any-K instantiation (d <= 16) is compiled for
#endif
constexpr int CACHE_ROWS = SS_BWD_CACHE_ROWS;
template <int DP>
constexpr int cache_stride() { return (8 + ((DP + 3) & ~3)) % 8 == 0 ? 8 + ((DP + 3) & ~3) + 4 : 8 + ((DP + 3) & ~3); }
struct RowCache {
    int *tag;     // [CACHE_ROWS] sphere id or -1
    float *rows;  // [CACHE_ROWS][stride]
    int stride;   // floats per row, = 4 mod 8 (rows of different lanes start in different bank groups)
};

// Per-hit gradient pieces for one stored slot (grad.py:110-179); accumulates into the sphere's row.
// acoef = <upstream, f_k - f_hat> (grad.py:110) is formed by the caller.
template <int DP, int MODE, bool MERGE = false, bool CACHE = false>
__device__ __forceinline__ void slot_gradient_acoef(const BackArgs &a, const Rec &rc, int id, float zk, float ck,
                                                    float E, float inv_g, const float *up, float acoef, int d,
                                                    double xs, double ys, double ux, double uy, double uz,
                                                    double inv_vnorm, const RowCache *cache = nullptr) {
    const Cam &cam = a.cam;
    const float o = rc.o;
    const float ez = o * zk * inv_g;
    const float w = o * ck * E;  // E = exp(o z / gamma - log_denom), computed once per slot by the caller
    const float dl_dz = acoef * w * o * inv_g;
    const float dl_dc = acoef * o * E;
    const float dl_do = acoef * ck * E * (1.0f + ez);

    // geometry chain (grad.py:117-165).  Only the cancelling part -- t = c.u and d = c - t u with
    // |c| ~ 1e3 |d| -- is float64; everything downstream is float32 on well-conditioned values.
    const float r = rc.r;
    float t, dvx, dvy, dvz, dist;
    if (MODE == SS_MODE_PINHOLE) {
        const double td = rc.cx * ux + rc.cy * uy + rc.cz * uz;
        const double ddx = rc.cx - td * ux, ddy = rc.cy - td * uy, ddz = rc.cz - td * uz;
        t = (float)td; dvx = (float)ddx; dvy = (float)ddy; dvz = (float)ddz;
        dist = sqrt_approx_f((float)(ddx * ddx + ddy * ddy + ddz * ddz));
    } else {
        const double ddx = rc.cx - xs, ddy = rc.cy - ys;
        t = (float)rc.cz; dvx = (float)ddx; dvy = (float)ddy; dvz = 0.0f;
        dist = sqrt_approx_f((float)(ddx * ddx + ddy * ddy));
    }
    const bool interior = (0.0f < zk) && (zk < 1.0f);
    const float dl_dzeta = interior ? -dl_dz * (float)cam.inv_range : 0.0f;
    const float inv_r = rcp_approx(r);
    const float dl_ddist = -dl_dc * inv_r;
    const float d_radius = dl_dc * dist * inv_r * inv_r;
    const float inv_dist = dist > 1e-12f ? rcp_approx(dist) : 0.0f;
    const float hx = dvx * inv_dist, hy = dvy * inv_dist, hz = dvz * inv_dist;
    const float xsf = (float)xs, ysf = (float)ys;
    float gcx, gcy, gcz, g_focal, g_sensor;
    if (MODE == SS_MODE_PINHOLE) {
        const float uxf = (float)ux, uyf = (float)uy, uzf = (float)uz;
        const float zu = dl_dzeta * uzf;
        gcx = fmaf(dl_ddist, hx, zu * uxf);
        gcy = fmaf(dl_ddist, hy, zu * uyf);
        gcz = fmaf(dl_ddist, hz, zu * uzf);
        // intrinsics chain (grad.py:141-154): grad_u = s1 c + dl_dzeta t e_z projected off u.  With
        // c = t u + d the projection is s1 d + dl_dzeta t (e_z - u_z u): same value, no cancellation.
        const float s1 = fmaf(-dl_ddist * t, inv_dist, zu);
        const float zt = dl_dzeta * t;
        const float prx = fmaf(s1, dvx, -zt * uzf * uxf);
        const float pry = fmaf(s1, dvy, -zt * uzf * uyf);
        const float prz = fmaf(s1, dvz, zt * (1.0f - uzf * uzf));
        const float ivn = (float)inv_vnorm;
        g_focal = prz * ivn;
        g_sensor = (prx * xsf + pry * ysf) * ivn * (float)(1.0 / cam.sensor_w);
    } else {
        gcx = dl_ddist * hx; gcy = dl_ddist * hy; gcz = dl_ddist * hz + dl_dzeta;
        g_sensor = -(dl_ddist * inv_dist) * (dvx * xsf + dvy * ysf) * (float)(1.0 / cam.sensor_w);
        g_focal = 0.0f;
    }
    constexpr int DP4 = (DP + 3) & ~3;  // the feature part of the row is padded to whole quads
    float v[8 + DP4];
    v[0] = gcx; v[1] = gcy; v[2] = gcz; v[3] = d_radius;
    v[4] = dl_do; v[5] = g_focal; v[6] = g_sensor; v[7] = 1.0f;
#pragma unroll
    for (int i = 0; i < DP4; ++i) v[8 + i] = i < DP ? w * up[i] : 0.0f;  // up[] is zero beyond d
  if (MERGE) {
    // Warp-level pre-reduction: the L2 processes one 16-byte reduction per lane and instruction (15.7 M of
    // them at C3: ~50 us of this kernel), and neighbouring pixels of the 8x4 block mostly hold the SAME
    // sphere in a slot.  match.any groups the lanes by sphere; the groups are summed by pointer jumping
    // (every lane adds the partial sum of its next peer and then points to that peer's next: after
    // log2(group size) rounds the lowest lane of each group holds the group's sum) and only that lane issues
    // the reductions.  (The caller guarantees that all 32 lanes get here; lanes without a hit carry id -1.)
    const unsigned lane = threadIdx.x & 31u;
    const unsigned peers = __match_any_sync(0xffffffffu, id);
    const unsigned above = peers & (0xfffffffeu << lane);  // peers in higher lanes
    int nxt = above ? __ffs((int)above) - 1 : -1;
    while (__any_sync(0xffffffffu, nxt >= 0)) {
        const int src = nxt >= 0 ? nxt : (int)lane;
#pragma unroll
        for (int j = 0; j < 8 + DP; ++j) {  // (padding beyond DP stays zero)
            if (j == 7) continue;  // the pixel count is the group size (set below)
            const float o = __shfl_sync(0xffffffffu, v[j], src);
            if (nxt >= 0) v[j] += o;
        }
        const int nn = __shfl_sync(0xffffffffu, nxt, src);
        nxt = nxt >= 0 ? nn : -1;
    }
    const bool lead = id >= 0 && (peers & ((1u << lane) - 1u)) == 0u;  // the group's lowest lane
    v[7] = (float)__popc(peers);
    if (a.det) {  // (warp-uniform)
        if (lead) det_emit<8 + DP>(a, id, v);
        return;
    }
    if (CACHE) {
        // one owner per cache row and instruction: leaders whose spheres hash to the same row are ranked, the
        // lowest lane uses the cache, the others (rare) reduce straight into the L2
        constexpr int kHashShift = CACHE_ROWS == 64 ? 26 : CACHE_ROWS == 32 ? 27 : CACHE_ROWS == 16 ? 28 : 29;
        const unsigned h = lead ? ((unsigned)id * 2654435761u) >> kHashShift : (unsigned)CACHE_ROWS + lane;
        static_assert(CACHE_ROWS == 64 || CACHE_ROWS == 32 || CACHE_ROWS == 16 || CACHE_ROWS == 8, "6 .. 3 hash bits");
        const unsigned same = __match_any_sync(0xffffffffu, h);
        const bool owner = lead && (same & ((1u << lane) - 1u)) == 0u;
        if (owner) {
            float4 *crow = reinterpret_cast<float4 *>(cache->rows + h * cache->stride);
            const int tag = cache->tag[h];
            if (tag == id) {
#pragma unroll
                for (int q = 0; q < (8 + DP4) / 4; ++q) {
                    float4 r = crow[q];
                    r.x += v[4 * q]; r.y += v[4 * q + 1]; r.z += v[4 * q + 2]; r.w += v[4 * q + 3];
                    crow[q] = r;
                }
            } else {
                if (tag >= 0) {  // evict: the cached partial sums of another sphere go to its accumulator row
                    float *erow = a.raw + (size_t)tag * a.raw_stride;
#pragma unroll
                    for (int q = 0; q < (8 + DP4) / 4; ++q) {
                        const float4 r = crow[q];
                        if (q < 2 || 4 * (q - 2) < d) red_add_v4(erow + 4 * q, r.x, r.y, r.z, r.w);
                    }
                }
#pragma unroll
                for (int q = 0; q < (8 + DP4) / 4; ++q)
                    crow[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                cache->tag[h] = id;
            }
        }
        __syncwarp();  // the row may be read by another lane in the next slot
        if (!lead || owner) return;
    } else {
        if (!lead) return;
    }
  } else {
    if (id < 0) return;
    if (a.det) { det_emit<8 + DP>(a, id, v); return; }
  }
    float *row = a.raw + (size_t)id * a.raw_stride;
    red_add_v4(row, v[0], v[1], v[2], v[3]);
    red_add_v4(row + 4, v[4], v[5], v[6], v[7]);
#pragma unroll
    for (int i = 0; i < DP4; i += 4)
        if (i < d) red_add_v4(row + 8 + i, v[8 + i], v[9 + i], v[10 + i], v[11 + i]);
}

template <int DP, int MODE, bool MERGE = false>
__device__ __forceinline__ void slot_gradient(const BackArgs &a, const Rec &rc, int id, float zk, float ck,
                                              float E, float inv_g, const float *up, const float *fhat,
                                              const float *f, int d, double xs, double ys, double ux, double uy,
                                              double uz, double inv_vnorm) {
    float acoef = 0.0f;
#pragma unroll
    for (int i = 0; i < DP; ++i)
        if (i < d) acoef = fmaf(up[i], f[i] - fhat[i], acoef);
    slot_gradient_acoef<DP, MODE, MERGE>(a, rc, id, zk, ck, E, inv_g, up, acoef, d, xs, ys, ux, uy, uz, inv_vnorm);
}

// KT > 0: the K <= KT slots of a pixel are unrolled, every load of a phase issued before its first use
// (the kernel is latency-bound on dependent gathers).  KT == 0: any K, slot by slot.
template <int DP, int MODE, int KT>
__global__ void __launch_bounds__(TILE_PX, (KT > 0) ? (KT <= 5 ? 4 : 3) : (DP <= 16 ? SS_BWD_ANYK_MINB : 1)) k_backward(BackArgs a) {
    const Cam &cam = a.cam;
    const int tile = blockIdx.x;
    const int tid = threadIdx.x;
    if (tile == 0 && tid == 0) *a.clean_tag = 0ull;  // accumulators are being written: not clean any more
    const int lane = tid & 31, warp = tid >> 5;
    const int px = (tile % cam.ntx) * TILE + (((warp & 1) << 3) | (lane & 7));  // 8x4 block per warp
    const int py = (tile / cam.ntx) * TILE + (((warp >> 1) << 2) | (lane >> 3));
    const bool valid = px < cam.W && py < cam.H;
    // the warp-level merge needs all 32 lanes in the slot loop; it pays up to d = 16 (C5: 5.3 -> 4.8 ms), not measured beyond
    constexpr bool kMerge = (SS_BACKWARD_MERGE != 0) && DP <= 16;
    if (!kMerge && !valid) return;
    const size_t P = (size_t)cam.W * cam.H;
    const size_t pix = valid ? (size_t)py * cam.W + px : 0;
    const int K = a.K, d = a.d;
    const int *__restrict__ ids = a.ids;
    const float *__restrict__ zb = a.z;
    const float *__restrict__ cb = a.clos;

    constexpr int KR = KT > 0 ? KT : 1;
    int sid[KR]; float zk[KR], ck[KR];
    if (KT > 0) {
#pragma unroll
        for (int k = 0; k < KR; ++k) {
            const bool in = k < K && valid;
            sid[k] = in ? ids[k * P + pix] : -1;
            zk[k] = in ? zb[k * P + pix] : 0.0f;
            ck[k] = in ? cb[k * P + pix] : 0.0f;
        }
        bool any = false;
#pragma unroll
        for (int k = 0; k < KR; ++k) any |= sid[k] >= 0;
        if (kMerge ? !__any_sync(0xffffffffu, any) : !any) return;
    } else {
        bool any = false;
        for (int k = 0; k < K; ++k) any |= valid && ids[k * P + pix] >= 0;
        if (kMerge ? !__any_sync(0xffffffffu, any) : !any) return;
    }
    const float ld = a.log_denom[pix];
    const float inv_g = (float)(1.0 / a.gamma);
    float up[DP], fhat[DP];
    const float w_bg = ex2_approx_f(((float)a.eps_over_g - ld) * 1.4426950408889634f);
#pragma unroll
    for (int i = 0; i < DP; ++i) {
        up[i] = i < d ? a.upstream[pix * d + i] : 0.0f;
        fhat[i] = i < d ? w_bg * a.bg[i] : 0.0f;
    }
    // ray (camera.py:332-357)
    const double xs = ((px + 0.5) - cam.W / 2.0) * cam.pix;
    const double ys = ((py + 0.5) - cam.H / 2.0) * cam.pix;
    double ux = 0.0, uy = 0.0, uz = 1.0, inv_vnorm = 1.0;
    if (MODE == SS_MODE_PINHOLE) {
        // one reciprocal square root instead of sqrt + 4 divisions: the ray only feeds gradient VALUES here
        // (tolerance 1e-4), and the long dependent float64 chains are what this latency-bound kernel waits on
        inv_vnorm = rsqrt(xs * xs + ys * ys + cam.focal * cam.focal);
        ux = xs * inv_vnorm; uy = ys * inv_vnorm; uz = cam.focal * inv_vnorm;
    }

    if (KT > 0) {
        // Register diet: the kernel is bound by the latency of its dependent loads, and holding all K records
        // (8 registers each) plus their features limited it to 2 resident CTAs per SM (121 registers).  Phase 1 keeps
        // only the opacity and the scalar <upstream, f_k> of every slot; phase 2 re-reads the record of slot k (an
        // L1 hit) one slot ahead of its use: 64 registers, 4 resident CTAs, 115 -> 91 us at C3.
        float ok[KR], uf[KR], Ek[KR];
        {
            float f[KR][DP];
#pragma unroll
            for (int k = 0; k < KR; ++k) {
                const int id = sid[k] >= 0 ? sid[k] : 0;
                ok[k] = sid[k] >= 0 ? a.rec[id].o : 0.0f;
#pragma unroll
                for (int i = 0; i < DP; ++i) f[k][i] = (sid[k] >= 0 && i < d) ? a.feat[(size_t)id * d + i] : 0.0f;
            }
#pragma unroll
            for (int k = 0; k < KR; ++k) {
                Ek[k] = sid[k] >= 0 ? ex2_approx_f((ok[k] * zk[k] * inv_g - ld) * 1.4426950408889634f) : 0.0f;
                const float w = ok[k] * ck[k] * Ek[k];
                uf[k] = 0.0f;
#pragma unroll
                for (int i = 0; i < DP; ++i) { fhat[i] = fmaf(w, f[k][i], fhat[i]); uf[k] = fmaf(up[i], f[k][i], uf[k]); }
            }
        }
        float ufh = 0.0f;
#pragma unroll
        for (int i = 0; i < DP; ++i) ufh = fmaf(up[i], fhat[i], ufh);
        Rec nxt; nxt.cx = nxt.cy = nxt.cz = 0.0; nxt.r = 1.0f; nxt.o = 0.0f;
        if (sid[0] >= 0) nxt = a.rec[sid[0]];
#pragma unroll
        for (int k = 0; k < KR; ++k) {
            const Rec cur = nxt;
            if (k + 1 < KR && sid[k + 1 < KR ? k + 1 : k] >= 0) nxt = a.rec[sid[k + 1 < KR ? k + 1 : k]];
            if (kMerge ? __any_sync(0xffffffffu, sid[k] >= 0) : sid[k] >= 0)
                slot_gradient_acoef<DP, MODE, kMerge>(a, cur, sid[k], zk[k], ck[k], Ek[k], inv_g, up, uf[k] - ufh, d, xs,
                                                      ys, ux, uy, uz, inv_vnorm);
        }
    } else {
        // Any K (n_track up to 64) and wide payloads: the feature rows (the bulk of the gather traffic: K x 4 d bytes
        // per pixel) are read ONCE, with 128-bit loads when they are aligned quads.  Pass 1 forms f_hat and keeps the
        // scalar <upstream, f_k> of every slot in shared memory (column per thread); pass 2 re-reads only the slot
        // (ids, z, closeness: coalesced, L1 hits) and the 32-byte record and needs no feature at all:
        // <upstream, f_k - f_hat> = <up, f_k> - <up, f_hat>, d_feature = w * upstream.
        extern __shared__ float s_uf[];  // [K][TILE_PX], then the per-warp accumulator caches
        constexpr int DP4c = (DP + 3) & ~3;
        constexpr int CSTRIDE = cache_stride<DP>();  // floats per cached row (= 4 mod 8)
        RowCache cache;
        cache.stride = CSTRIDE;
        cache.rows = s_uf + (size_t)K * TILE_PX + (size_t)warp * (CACHE_ROWS * CSTRIDE + CACHE_ROWS);
        cache.tag = reinterpret_cast<int *>(cache.rows + CACHE_ROWS * CSTRIDE);
        if (kMerge) {
#pragma unroll
            for (int r = 0; r < (CACHE_ROWS + 31) / 32; ++r)
                if (lane + 32 * r < CACHE_ROWS) cache.tag[lane + 32 * r] = -1;
            __syncwarp();
        }
        const bool quads = (d & 3) == 0 && (reinterpret_cast<unsigned long long>(a.feat) & 15ull) == 0ull;
        for (int k = 0; k < K; ++k) {
            const int id = valid ? __ldg(ids + k * P + pix) : -1;
            if (id < 0) continue;
            const float o = __ldg(&a.rec[id].o);
            const float E = ex2_approx_f((o * __ldg(zb + k * P + pix) * inv_g - ld) * 1.4426950408889634f);
            const float w = o * __ldg(cb + k * P + pix) * E;
            const float *f = a.feat + (size_t)id * d;
            float uf = 0.0f;
            if (quads) {
#pragma unroll
                for (int i = 0; i < DP; i += 4) {
                    if (i < d) {
                        const float4 q = __ldg(reinterpret_cast<const float4 *>(f + i));
                        fhat[i] = fmaf(w, q.x, fhat[i]); uf = fmaf(up[i], q.x, uf);
                        if (i + 1 < DP) { fhat[i + 1] = fmaf(w, q.y, fhat[i + 1]); uf = fmaf(up[i + 1], q.y, uf); }
                        if (i + 2 < DP) { fhat[i + 2] = fmaf(w, q.z, fhat[i + 2]); uf = fmaf(up[i + 2], q.z, uf); }
                        if (i + 3 < DP) { fhat[i + 3] = fmaf(w, q.w, fhat[i + 3]); uf = fmaf(up[i + 3], q.w, uf); }
                    }
                }
            } else {
#pragma unroll
                for (int i = 0; i < DP; ++i)
                    if (i < d) { const float fi = __ldg(f + i); fhat[i] = fmaf(w, fi, fhat[i]); uf = fmaf(up[i], fi, uf); }
            }
            s_uf[k * TILE_PX + tid] = uf;
        }
        float ufh = 0.0f;
#pragma unroll
        for (int i = 0; i < DP; ++i) ufh = fmaf(up[i], fhat[i], ufh);
        // (measured at C5, 10 M spheres / d = 16 / K = 32, 3.9 ms: pass 1 1.25 ms, pass 2 without its reductions
        // 0.9 ms, the 225 M 16-byte L2 reductions 1.8 ms; reading ids four slots ahead, prefetching the rows of
        // slot k + 3 or loading slot k + 1 during slot k changed nothing or cost time -- see profiles/r02_summary.md)
        const Rec rc_none = {0.0, 0.0, 0.0, 1.0f, 0.0f};
        for (int k = 0; k < K; ++k) {
            const int id = valid ? __ldg(ids + k * P + pix) : -1;
            if (kMerge ? !__any_sync(0xffffffffu, id >= 0) : id < 0) continue;
            Rec rc = rc_none;
            float zk1 = 0.0f, ck1 = 0.0f, uf = 0.0f;
            if (id >= 0) {
                rc = ldg_rec(a.rec + id);
                zk1 = __ldg(zb + k * P + pix); ck1 = __ldg(cb + k * P + pix);
                uf = s_uf[k * TILE_PX + tid];
            }
            const float E1 = ex2_approx_f((rc.o * zk1 * inv_g - ld) * 1.4426950408889634f);
            slot_gradient_acoef<DP, MODE, kMerge, kMerge && (SS_BWD_CACHE != 0)>(a, rc, id, zk1, ck1, E1, inv_g, up, uf - ufh, d, xs, ys, ux,
                                                          uy, uz, inv_vnorm, &cache);
        }
        if (kMerge && SS_BWD_CACHE && !a.det) {  // flush the cache: every lane owns two rows
            __syncwarp();
#pragma unroll
            for (int r = 0; r < (CACHE_ROWS + 31) / 32; ++r) {
                const int h = lane + 32 * r;
                const int tag = h < CACHE_ROWS ? cache.tag[h] : -1;
                if (tag >= 0) {
                    const float4 *crow = reinterpret_cast<const float4 *>(cache.rows + h * CSTRIDE);
                    float *erow = a.raw + (size_t)tag * a.raw_stride;
#pragma unroll
                    for (int q = 0; q < (8 + DP4c) / 4; ++q) {
                        const float4 v4 = crow[q];
                        if (q < 2 || 4 * (q - 2) < d) red_add_v4(erow + 4 * q, v4.x, v4.y, v4.z, v4.w);
                    }
                }
            }
        }
    }
}

// ---- clean-accumulator protocol ---------------------------------------------------------------
// The raw accumulator rows (M x raw_stride floats, 48 MB at C3) must be zero when k_backward starts.
// Instead of a memset per call, k_finalize re-zeroes exactly the rows it consumed (the ~1/3 of the
// spheres that were touched) and then stamps the workspace with a tag derived from the layout;
// k_raw_prepare zeroes everything only when the tag is missing (first call, new layout, aborted call).
// A fresh workspace must not carry a stale tag: ss_forward clears it, and the tag also encodes dims.
constexpr int BST_COUNTER = CAM_VALS;      // cam_part[16]: completion counter (as unsigned)
constexpr int BST_TAG = CAM_VALS + 1;      // cam_part[17]: clean tag (as unsigned long long)

__global__ void __launch_bounds__(256) k_raw_prepare(float4 *raw4, size_t n4, double *bst, unsigned long long tag) {
    const bool clean = ((const unsigned long long *)bst)[BST_TAG] == tag;
    if (blockIdx.x == 0 && threadIdx.x <= CAM_VALS) bst[threadIdx.x] = 0.0;  // camera sums + counter
    if (clean) return;
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
        raw4[i] = z;
}

// SS_OPT_DETERMINISTIC: fixed-point rows -> the float accumulator rows k_finalize consumes (every row is written,
// so the clean-accumulator protocol stays valid: k_finalize re-zeroes what it consumes).
__global__ void __launch_bounds__(256) k_det_convert(const long long *raw64, const unsigned *det_max, float *raw,
                                                     long long M, int stride) {
    const long long n = M * stride;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long s = i / stride;
        const int j = (int)(i - s * stride);
        const long long iv = raw64[i];
        float out = 0.0f;
        if (iv != 0) {
            const int e = (int)(det_max[s] >> 23);
            const double q = __hiloint2double((1023 - 164 + e) << 20, 0);  // 2^(e - 164)
            out = j == 7 ? (float)iv : (float)((double)iv * q);
        }
        raw[i] = out;
    }
}

struct FinArgs {
    long long M; int d, raw_stride;
    Cam cam;
    const float *pos;
    float *raw;
    const double *proj_r;
    float *d_pos, *d_rad, *d_opa, *d_feat; int *pixel_count;
    double *cam_part; double *cam_grad;
    unsigned long long tag;
    int normalize, gate, cam_grads, accumulate;
    int det;  // camera sums: one slot per block behind the atomics' area, added up in block order by the last block
};

// One thread per sphere.  The kernel is instruction-bound, not bandwidth-bound (ncu: a staged,
// "coalesced" variant executed 950 instructions per warp and took 58 us), so this version keeps the
// per-thread path short: three 128-bit row loads, float32 per-sphere math (the accumulators are float32
// sums already), float64 only for the 14 camera sums, which are reduced through a shared-memory
// transpose instead of 14 x 5 double shuffles.
__global__ void __launch_bounds__(256) k_finalize(FinArgs a) {
    __shared__ double s_red[14][8];
    const Cam &cam = a.cam;
    const int RS = a.raw_stride, d = a.d;
    const int t = threadIdx.x;
    bool any_touched = false;
    float acc[14];
#pragma unroll
    for (int j = 0; j < 14; ++j) acc[j] = 0.0f;
    // Persistent CTAs: a thread walks <= 8 spheres and keeps its camera partial sums in registers, so the
    // butterfly, the barrier, the float64 atomics, the fence and the (returning) completion-counter atomic at the
    // end are paid once per CTA instead of once per 256 spheres.
    const long long n_blocks = (a.M + 255) / 256;
    const bool feat_quads = (d & 3) == 0 && (reinterpret_cast<unsigned long long>(a.d_feat) & 15ull) == 0ull;
    const float4 zero4 = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 n0 = zero4, n1 = zero4;  // the first two quads of the NEXT sphere's row, loaded one iteration ahead
    {
        const long long i0 = (long long)blockIdx.x * 256 + t;
        if (blockIdx.x < n_blocks && i0 < a.M) {
            const float4 *row0 = (const float4 *)(a.raw + (size_t)i0 * RS);
            n0 = row0[0]; n1 = row0[1];
        }
    }
    for (long long blk = blockIdx.x; blk < n_blocks; blk += gridDim.x) {
        const long long i = blk * 256 + t;
        const float4 r0 = n0, r1 = n1;
        {
            const long long inext = i + (long long)gridDim.x * 256;
            if (blk + gridDim.x < n_blocks && inext < a.M) {
                const float4 *rown = (const float4 *)(a.raw + (size_t)inext * RS);
                n0 = rown[0]; n1 = rown[1];
                // a touched sphere also needs its projected radius and position: the kernel spent half its warp time
                // waiting for those two dependent loads (ncu long-scoreboard samples); request the lines now
                if (a.normalize || a.gate) asm volatile("prefetch.global.L1 [%0];" ::"l"(a.proj_r + inext));
                if (a.cam_grads) asm volatile("prefetch.global.L1 [%0];" ::"l"(a.pos + 3 * inext));
            }
        }
        if (i >= a.M) continue;
        float4 *row = (float4 *)(a.raw + (size_t)i * RS);
        const float cnt = r1.w;
        const bool touched = cnt > 0.0f;
        any_touched |= touched;
        float dp0 = 0.f, dp1 = 0.f, dp2 = 0.f, drad = 0.f, dopa = 0.f, inv_div = 0.f;
        if (touched) {
            const double pr = a.proj_r[i];
            float cam_scale = 1.0f;
            inv_div = 1.0f;
            if (a.normalize) {
                inv_div = 1.0f / cnt;
                cam_scale = 1e-3f / fmaxf(3.14159265358979f * (float)(pr * pr), 1.0f);
            }
            const float R0 = (float)cam.R[0], R1 = (float)cam.R[1], R2 = (float)cam.R[2], R3 = (float)cam.R[3],
                        R4 = (float)cam.R[4], R5 = (float)cam.R[5], R6 = (float)cam.R[6], R7 = (float)cam.R[7],
                        R8 = (float)cam.R[8];
            dp0 = (r0.x * R0 + r0.y * R3 + r0.z * R6) * inv_div;  // d_position = (g_center @ R) / count
            dp1 = (r0.x * R1 + r0.y * R4 + r0.z * R7) * inv_div;
            dp2 = (r0.x * R2 + r0.y * R5 + r0.z * R8) * inv_div;
            drad = r0.w * inv_div;
            dopa = r1.x * inv_div;
            if (a.gate && pr <= 3.0) { dp0 = dp1 = dp2 = 0.f; drad = 0.f; }  // grad.py:305-320
            if (a.cam_grads) {
                const float sx = cam_scale * r0.x, sy = cam_scale * r0.y, sz = cam_scale * r0.z;
                const float rx = (float)((double)a.pos[3 * i] - cam.t[0]), ry = (float)((double)a.pos[3 * i + 1] - cam.t[1]),
                            rz = (float)((double)a.pos[3 * i + 2] - cam.t[2]);
                acc[0] += sx; acc[1] += sy; acc[2] += sz;
                acc[3] = fmaf(sx, rx, acc[3]); acc[4] = fmaf(sx, ry, acc[4]); acc[5] = fmaf(sx, rz, acc[5]);
                acc[6] = fmaf(sy, rx, acc[6]); acc[7] = fmaf(sy, ry, acc[7]); acc[8] = fmaf(sy, rz, acc[8]);
                acc[9] = fmaf(sz, rx, acc[9]); acc[10] = fmaf(sz, ry, acc[10]); acc[11] = fmaf(sz, rz, acc[11]);
                acc[12] = fmaf(cam_scale, r1.y, acc[12]);
                acc[13] = fmaf(cam_scale, r1.z, acc[13]);
            }
        }
        // features: RS - 8 = ceil4(d) floats behind the two fixed quads (whole, aligned rows move as 128-bit words)
        float *df = a.d_feat + (size_t)i * d;
        for (int q = 0; q * 4 < d; ++q) {
            float4 f4 = touched ? row[2 + q] : make_float4(0.f, 0.f, 0.f, 0.f);
            const float v[4] = {f4.x * inv_div, f4.y * inv_div, f4.z * inv_div, f4.w * inv_div};
            if (feat_quads) {
                float4 *dq = reinterpret_cast<float4 *>(df) + q;
                if (a.accumulate) {
                    if (touched) { float4 o = *dq; o.x += v[0]; o.y += v[1]; o.z += v[2]; o.w += v[3]; *dq = o; }
                } else {
                    *dq = make_float4(v[0], v[1], v[2], v[3]);
                }
                continue;
            }
#pragma unroll
            for (int c = 0; c < 4; ++c)
                if (q * 4 + c < d) {
                    if (a.accumulate) { if (touched) df[q * 4 + c] += v[c]; }
                    else df[q * 4 + c] = v[c];
                }
        }
        if (a.accumulate) {
            if (touched) {
                a.d_pos[3 * i] += dp0; a.d_pos[3 * i + 1] += dp1; a.d_pos[3 * i + 2] += dp2;
                a.d_rad[i] += drad; a.d_opa[i] += dopa; a.pixel_count[i] += (int)cnt;
            }
        } else {
            a.d_pos[3 * i] = dp0; a.d_pos[3 * i + 1] = dp1; a.d_pos[3 * i + 2] = dp2;
            a.d_rad[i] = drad; a.d_opa[i] = dopa; a.pixel_count[i] = (int)cnt;
        }
        if (touched) {  // give the row back clean for the next call
            const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int q = 0; q < RS / 4; ++q) row[q] = z;
        }
    }

    // camera sums: float32 butterfly inside the warp (32 terms), float64 from there on: per-warp
    // partials in shared memory, ONE block barrier, then warp 0 alone adds the block's 14 sums to the
    // global accumulators (double atomics), fences and bumps the completion counter; the last block
    // publishes the camera block and the clean tag.
    const int lane = t & 31, wid = t >> 5;
    if (a.cam_grads && __any_sync(0xffffffffu, any_touched)) {
#pragma unroll
        for (int j = 0; j < 14; ++j) {
            float v = acc[j];
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) s_red[j][wid] = (double)v;
        }
    } else if (lane == 0) {
#pragma unroll
        for (int j = 0; j < 14; ++j) s_red[j][wid] = 0.0;
    }
    __syncthreads();
    if (wid != 0) return;
    if (a.cam_grads && lane < 14) {
        double v = 0.0;
#pragma unroll
        for (int e = 0; e < 8; ++e) v += s_red[lane][e];
        if (a.det) a.cam_part[CAM_VALS + 2 + (size_t)blockIdx.x * CAM_VALS + lane] = v;
        else if (v != 0.0) atomicAdd(&a.cam_part[lane], v);
    }
    __syncwarp();
    unsigned last = 0u;
    if (lane == 0) {
        __threadfence();  // orders this block's atomics / slot stores (cumulative over the warp) before the counter
        unsigned int *counter = (unsigned int *)(a.cam_part + BST_COUNTER);
        last = atomicAdd(counter, 1u) == gridDim.x - 1 ? 1u : 0u;
        __threadfence();
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (!last) return;
    if (a.cam_grads && a.det) {  // block-ordered sum of the per-block slots: lane j adds up column j
        if (lane < 14) {
            volatile double *slots = a.cam_part + CAM_VALS + 2;
            double acc = 0.0;
            for (unsigned b = 0; b < gridDim.x; ++b) acc += slots[(size_t)b * CAM_VALS + lane];
            a.cam_part[lane] = acc;
        }
        __threadfence();
        __syncwarp();
    }
    if (lane != 0) return;
    if (a.cam_grads) {
        const double *R = cam.R;
        volatile double *vs = a.cam_part;
        const double t0 = vs[0], t1 = vs[1], t2 = vs[2];
        for (int j = 0; j < 3; ++j)  // d_translation = -(sum sc) @ R  (grad.py:289)
            a.cam_grad[j] = -(t0 * R[0 + j] + t1 * R[3 + j] + t2 * R[6 + j]);
        for (int j = 0; j < 9; ++j) a.cam_grad[3 + j] = vs[3 + j];
        a.cam_grad[12] = vs[12];
        a.cam_grad[13] = vs[13];
        a.cam_grad[14] = 0.0; a.cam_grad[15] = 0.0;
    }
    ((unsigned long long *)a.cam_part)[BST_TAG] = a.tag;  // every consumed row is zero again
}

template <int DP, int KT, int MODE>
void launch_bw_one(const BackArgs &b, int n_tiles, cudaStream_t s) {
    // <up, f_k> columns (64 KB at K = 64) + 8 per-warp accumulator caches (60 KB at d = 16)
    constexpr size_t cache_bytes = DP <= 16 ? 8 * (size_t)CACHE_ROWS * (cache_stride<DP>() + 1) * sizeof(float) : 0;
    const size_t smem = KT > 0 ? 0 : (size_t)b.K * TILE_PX * sizeof(float) + cache_bytes;
    if (KT == 0) {
        static PerDeviceOnce attr_once;  // per instantiation and device
        if (attr_once.first())
            cudaFuncSetAttribute(k_backward<DP, MODE, KT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 SS_MAX_TOP_K * TILE_PX * (int)sizeof(float) + (int)cache_bytes);
    }
    k_backward<DP, MODE, KT><<<n_tiles, TILE_PX, smem, s>>>(b);
}

template <int DP, int KT>
void launch_bw_mode(const BackArgs &b, int n_tiles, int mode, cudaStream_t s) {
    if (mode == SS_MODE_PINHOLE) launch_bw_one<DP, KT, SS_MODE_PINHOLE>(b, n_tiles, s);
    else launch_bw_one<DP, KT, SS_MODE_ORTHOGRAPHIC>(b, n_tiles, s);
}

template <int DP>
void launch_bw_k(const BackArgs &b, int n_tiles, int mode, cudaStream_t s) {
#ifdef SS_EXPERIMENT_BWD_LOOP
    launch_bw_mode<DP, 0>(b, n_tiles, mode, s);
#else
    if (DP <= 4 && b.K <= 5) launch_bw_mode<DP, 5>(b, n_tiles, mode, s);
    else if (DP <= 4 && b.K <= 8) launch_bw_mode<DP, 8>(b, n_tiles, mode, s);
    else launch_bw_mode<DP, 0>(b, n_tiles, mode, s);
#endif
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
    double *bst = (double *)(a.ws + L.cam_part);
    // tag of a clean accumulator region for exactly this layout
    unsigned long long tag = 0x5353424b434c4e31ull;  // "SSBKCLN1"
    tag ^= (unsigned long long)M * 0x9e3779b97f4a7c15ull;
    tag ^= ((unsigned long long)L.raw_stride << 48) ^ ((unsigned long long)L.raw << 8) ^ (unsigned long long)a.dims.max_pairs;
    {
        ProfScope ps(KID_MEMSET_BWD, s);
        const size_t n4 = (size_t)M * L.raw_stride / 4;
        k_raw_prepare<<<148, 256, 0, s>>>((float4 *)raw, n4, bst, tag);  // (grid-stride; usually one block's worth of work)
        count_launch();
    }
    BackArgs b;
    b.cam = a.cam;
    b.rec = (const Rec *)(a.ws + L.rec);
    b.feat = a.feat; b.bg = a.bg;
    b.ids = a.ids; b.z = a.z; b.clos = a.clos; b.log_denom = a.log_denom; b.upstream = a.upstream;
    b.raw = raw; b.raw_stride = L.raw_stride;
    b.clean_tag = (unsigned long long *)bst + BST_TAG;
    b.d = a.dims.feature_dim; b.K = a.dims.top_k;
    b.gamma = a.gamma; b.eps_over_g = a.blend.eps / a.gamma;
    b.det = 0; b.det_max = nullptr; b.raw64 = nullptr;
    const int d = b.d, mode = a.cam.mode;
    auto run_backward = [&]() {
        ProfScope ps(KID_BACKWARD, s);
        if (d == 3) launch_bw_k<3>(b, L.n_tiles, mode, s);  // RGB: one shuffle per merge round less than the d = 4 build
        else if (d <= 4) launch_bw_k<4>(b, L.n_tiles, mode, s);
        else if (d <= 16) launch_bw_k<16>(b, L.n_tiles, mode, s);
        else launch_bw_k<32>(b, L.n_tiles, mode, s);
        count_launch();
    };
    const bool det = a.det_ws != nullptr;
    if (!det) {
        run_backward();
    } else {
        // SS_OPT_DETERMINISTIC: pass 1 finds every sphere's largest addend (order-independent max), pass 2
        // accumulates in 64-bit fixed point on that sphere's grid, k_det_convert hands float rows to k_finalize
        const DetLayout D = make_det_layout(a.dims);
        b.det_max = (unsigned *)(a.det_ws + D.max_bits);
        b.raw64 = (long long *)(a.det_ws + D.raw64);
        cudaError_t e = cudaMemsetAsync(a.det_ws, 0, D.total, s);
        if (e != cudaSuccess) return e;
        b.det = 1;
        run_backward();
        b.det = 2;
        run_backward();
        k_det_convert<<<148 * 8, 256, 0, s>>>(b.raw64, b.det_max, raw, M, L.raw_stride);
        count_launch();
    }

    FinArgs f;
    f.M = M; f.d = d; f.raw_stride = L.raw_stride;
    f.cam = a.cam; f.pos = a.pos; f.raw = raw;
    f.proj_r = (const double *)(a.ws + L.proj_r);
    f.d_pos = a.d_pos; f.d_rad = a.d_rad; f.d_opa = a.d_opa; f.d_feat = a.d_feat;
    f.pixel_count = a.pixel_count;
    f.cam_part = bst;
    f.cam_grad = a.cam_grad;
    f.tag = tag;
    f.normalize = (a.blend.flags & SS_OPT_NORMALIZE) ? 1 : 0;
    f.gate = (a.blend.flags & SS_OPT_GATE) ? 1 : 0;
    f.cam_grads = cam_grads ? 1 : 0;
    f.accumulate = (a.blend.flags & SS_OPT_ACCUMULATE) ? 1 : 0;
    f.det = det ? 1 : 0;
    const long long fin_blocks = (M + 255) / 256;
    long long fin_grid = 148 * 4 > (fin_blocks + 7) / 8 ? 148 * 4 : (fin_blocks + 7) / 8;  // one wave (56 registers: 4 CTAs per SM) or <= 8 spheres per thread
    if (det && fin_grid > CAM_BLOCKS_MAX - 2) fin_grid = CAM_BLOCKS_MAX - 2;  // one camera-sum slot per block
    int grid = (int)(fin_blocks < fin_grid ? fin_blocks : fin_grid);
    {
        ProfScope ps(KID_FINALIZE, s);
        k_finalize<<<grid, 256, 0, s>>>(f);
    }
    count_launch();
    return cudaGetLastError();
}

}  // namespace ss
