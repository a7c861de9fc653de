// Step 0 + tile binning for sm_100a.
//
//   k_project   reference compute_bounds (raster.py:181-236): world->camera, tangent-wedge
//               extents, pixel rectangles, culling, earliest depth, projected radius, input
//               validation (scene.py:91-114) -- float64 per sphere, M-parallel, plus the
//               per-tile candidate COUNT (one atomic per touched tile).
//   k_scan      exclusive prefix sum of the tile counts -> tile_start (raster.py:290-292).
//               k_project also writes the sphere id straight into a fixed-capacity bucket of every touched tile
//               (4096 ids per tile; spheres touching > 4 tiles fill the bucket from its far end), so the common
//               case needs no emit pass at all: the per-tile sort reads its bucket and gathers the keys.
//   k_emit      (fallback, only when some tile holds more than 4096 spheres: SS_FLAG_LIST_FALLBACK)
//               writes each (tile, sphere) pair into its tile's segment, claiming the slot with an atomic on a
//               per-tile cursor (the consumed tile counters, zeroed again by k_scan).  The usual frame pays
//               nothing for it: no per-sphere slot array is written by k_project any more.
//   k_tile_sort per-tile sort of the segment by (earliest float64, sphere index): exactly the
//               order the reference gets from "stable argsort by earliest" (raster.py:243)
//               followed by "stable argsort by tile id" (raster.py:289).  One CTA per tile,
//               bitonic network in shared memory; the global M-wide sort and the T-wide
//               (tile, depth) radix sort of the classic design are not needed.
#include <math.h>

#include "ss_common.cuh"
#include "ss_sort.cuh"

namespace ss {

namespace {

constexpr double kHalfPi = 1.57079632679489661923;
constexpr double kIntHuge = 1073741824.0;  // 1 << 30 (raster.py:34)

__device__ __forceinline__ double clampd(double x, double lo, double hi) {
    return fmin(fmax(x, lo), hi);
}

// raster.py:130-154
__device__ void axis_extent_pinhole(double ca, double cz, double inv_cz, double r, double focal, double &lo,
                                    double &hi, bool &empty) {
    double n2 = ca * ca + cz * cz;
    if (cz > r * 1.000001 && n2 > r * r) {
        // Disc strictly in front of the camera plane: |phi| + beta < pi/2, so the wedge neither crosses
        // the horizon nor is empty or full, and tan(phi -+ beta) has a closed form (same value as the
        // reference's asin/atan2/tan chain to a few ulp).  One rsqrt and one reciprocal per axis:
        // tan(phi - beta) = (tp - tb)(1 - tp tb) / D, tan(phi + beta) = (tp + tb)(1 + tp tb) / D,
        // D = 1 - (tp tb)^2 > 0.
        const double tb = r * rsqrt(n2 - r * r);  // tan(beta), beta = asin(r / n)
        const double tp = ca * inv_cz;            // tan(phi), phi = atan2(ca, cz)
        const double pq = tp * tb;
        const double inv_d = focal / (1.0 - pq * pq);
        lo = (tp - tb) * (1.0 - pq) * inv_d;
        hi = (tp + tb) * (1.0 + pq) * inv_d;
        empty = false;
        return;
    }
    double n = sqrt(n2);
    bool full = n2 <= r * r;
    double beta = asin(clampd(r / fmax(n, 1e-300), 0.0, 1.0));
    double phi = atan2(ca, cz);
    double lo_a = phi - beta, hi_a = phi + beta;
    empty = ((lo_a >= kHalfPi) || (hi_a <= -kHalfPi)) && !full;
    const double cap = kHalfPi - 1e-9;
    lo = (lo_a <= -kHalfPi) ? -INFINITY : focal * tan(clampd(lo_a, -cap, cap));
    hi = (hi_a >= kHalfPi) ? INFINITY : focal * tan(clampd(hi_a, -cap, cap));
    if (full) { lo = -INFINITY; hi = INFINITY; }
}

// raster.py:157-178
template <typename CenterFn>
__device__ __forceinline__ void discretize_extent(double lo_px, double hi_px, CenterFn center_px_fn, int limit,
                                                  int &i_lo, int &i_hi, bool &outside) {
    double pad = 1e-9 * (1.0 + fabs(lo_px));
    double lo_f = clampd(ceil(lo_px - 0.5 - pad), -kIntHuge, kIntHuge);
    pad = 1e-9 * (1.0 + fabs(hi_px));
    double hi_f = clampd(floor(hi_px - 0.5 + pad), -kIntHuge, kIntHuge);
    long long a = (long long)lo_f, b = (long long)hi_f;
    if (a > b) {  // sub-pixel extent: the pixel containing the projected centre (rare; exact division here)
        const double center_px = center_px_fn();
        double c = isfinite(center_px) ? center_px : 0.0;
        long long nearest = (long long)clampd(floor(c), -kIntHuge, kIntHuge);
        a = nearest; b = nearest;
    }
    outside = (b < 0) || (a > limit - 1);
    a = a < 0 ? 0 : (a > limit - 1 ? limit - 1 : a);
    b = b < 0 ? 0 : (b > limit - 1 ? limit - 1 : b);
    i_lo = (int)a; i_hi = (int)b;
}

__device__ __forceinline__ unsigned long long order_key(double e) {
    e += 0.0;  // -0.0 -> +0.0 so that equal values have equal keys
    unsigned long long b = (unsigned long long)__double_as_longlong(e);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

struct ProjectArgs {
    long long M; int d;
    const float *pos, *rad, *opa, *feat, *bg;
    Cam cam;
    Rec *rec; unsigned long long *key; ushort4 *trect; double *proj_r; float4 *flt;
    int *tile_count; int *tile_count_big; int *bucket; long long *status;
    int32_t *rect; uint8_t *on_sensor; double *earliest; double *proj_r_out;
    int records_only; int validate;
};

__global__ void __launch_bounds__(256) k_project(ProjectArgs a) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    bool in = i < a.M;
    bool on = false;
    if (in) {
        const Cam &cam = a.cam;
        float pxf = a.pos[3 * i], pyf = a.pos[3 * i + 1], pzf = a.pos[3 * i + 2];
        float rf = a.rad[i], of = a.opa[i];
        bool bad = false;
        if (a.validate) {
            bad = !(isfinite(pxf) && isfinite(pyf) && isfinite(pzf) && isfinite(rf) && isfinite(of)) ||
                  !(rf > 0.0f);
            const float *f = a.feat + (size_t)i * a.d;
            for (int k = 0; k < a.d; ++k) bad |= !isfinite(f[k]);
            if (i == 0)
                for (int k = 0; k < a.d; ++k) bad |= !isfinite(a.bg[k]);
            if (bad) {
                atomicOr((unsigned long long *)&a.status[ST_FLAGS], (unsigned long long)SS_FLAG_INVALID_INPUT);
                atomicMax(&a.status[ST_FIRST_INVALID], a.M - i);  // decoded by k_scan
            }
        }
        double dx = (double)pxf - cam.t[0], dy = (double)pyf - cam.t[1], dz = (double)pzf - cam.t[2];
        const double *R = cam.R;
        double cx = dx * R[0] + dy * R[1] + dz * R[2];
        double cy = dx * R[3] + dy * R[4] + dz * R[5];
        double cz = dx * R[6] + dy * R[7] + dz * R[8];
        double r = (double)rf;
        Rec rc; rc.cx = cx; rc.cy = cy; rc.cz = cz; rc.r = rf; rc.o = fminf(fmaxf(of, 0.0f), 1.0f);
        a.rec[i] = rc;

        double lo_x, hi_x, lo_y, hi_y;
        bool empty_x = false, empty_y = false;
        const bool behind = (cz + r) <= 0.0;
        const bool pin = cam.mode == SS_MODE_PINHOLE;
        const int w = cam.W, h = cam.H;
        const double inv_cz = cz > 0.0 ? 1.0 / cz : 0.0;  // fast paths only (never feeds an exact quantity)
        if (pin) {
            axis_extent_pinhole(cx, cz, inv_cz, r, cam.focal, lo_x, hi_x, empty_x);
            axis_extent_pinhole(cy, cz, inv_cz, r, cam.focal, lo_y, hi_y, empty_y);
        } else {
            lo_x = cx - r; hi_x = cx + r; lo_y = cy - r; hi_y = cy + r;
        }
        // rectangle, visibility and the histogram atomics come first: the slot indices they return are
        // only needed at the very end, so their latency hides behind the rest of the per-sphere math
        ushort4 tr = make_ushort4(1, 0, 1, 0);
        int sl[4] = {0, 0, 0, 0};
        int nt = 0;
        if (!a.records_only) {
            int x0, x1, y0, y1; bool out_x, out_y;
            const double safe_z = cz > 0.0 ? cz : INFINITY;
            auto u_c = [&]() { return pin ? w / 2.0 + cam.focal * cx / safe_z * cam.ppu : w / 2.0 + cx * cam.ppu; };
            auto v_c = [&]() { return pin ? h / 2.0 + cam.focal * cy / safe_z * cam.ppu : h / 2.0 + cy * cam.ppu; };
            discretize_extent(w / 2.0 + lo_x * cam.ppu, w / 2.0 + hi_x * cam.ppu, u_c, w, x0, x1, out_x);
            discretize_extent(h / 2.0 + lo_y * cam.ppu, h / 2.0 + hi_y * cam.ppu, v_c, h, y0, y1, out_y);
            on = !(behind || empty_x || empty_y || out_x || out_y) && !bad;
            if (a.rect) {
                a.rect[4 * i] = x0; a.rect[4 * i + 1] = x1; a.rect[4 * i + 2] = y0; a.rect[4 * i + 3] = y1;
            }
            if (a.on_sensor) a.on_sensor[i] = on ? 1 : 0;
            if (on) {
                tr.x = (unsigned short)(x0 / TILE); tr.y = (unsigned short)(x1 / TILE);
                tr.z = (unsigned short)(y0 / TILE); tr.w = (unsigned short)(y1 / TILE);
                const int wx = tr.y - tr.x + 1;
                nt = wx * (tr.w - tr.z + 1);
                if (nt <= 4) {  // claim the slots now; k_emit needs no atomics for this sphere
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (j < nt) {  // tile j of the rectangle, row-major (no integer division: nt <= 4)
                            const int ty = (j >= wx) + (j >= 2 * wx) + (j >= 3 * wx);
                            sl[j] = atomicAdd(&a.tile_count[(tr.z + ty) * cam.ntx + tr.x + (j - ty * wx)], 1);
                        }
                } else {
                    for (int ty = tr.z; ty <= tr.w; ++ty)
                        for (int tx = tr.x; tx <= tr.y; ++tx) {
                            const int t = ty * cam.ntx + tx;
                            const int sb = atomicAdd(&a.tile_count_big[t], 1);
                            if (sb < BUCKET_CAP) a.bucket[(size_t)t * BUCKET_CAP + BUCKET_CAP - 1 - sb] = (int)i;
                        }
                }
            }
            a.trect[i] = tr;
        }

        // exact quantities (bit-identical formulas to the reference): earliest depth and projected radius
        double e, pr;
        if (pin) {
            const double d2 = cx * cx + cy * cy + cz * cz;
            e = sqrt(d2) - r;
            pr = (cam.focal * r / sqrt(fmax(d2 - r * r, 1e-300))) * cam.ppu;
            if (d2 <= r * r) pr = (double)(w > h ? w : h);
        } else {
            e = cz - r;
            pr = r * cam.ppu;
        }
        a.proj_r[i] = pr;
        if (a.proj_r_out) a.proj_r_out[i] = pr;
        if (!a.records_only) {
            if (!on) e = INFINITY;
            if (a.earliest) a.earliest[i] = e;
            a.key[i] = order_key(e);
            // Screen-space filter record for k_raster: a pixel can only hit the sphere if it lies in
            // the circle around the projected centre with radius f (tan(theta + alpha) - tan(theta))
            // (theta: centre off the optical axis, alpha = asin(r/|c|)), which bounds the projected
            // outline.  Padded for the float32 evaluation; infinite (always passes) when the sphere
            // reaches the camera plane or contains the camera.
            double pcx = 0.0, pcy = 0.0, rho = INFINITY;
            if (pin) {
                const double n2 = cx * cx + cy * cy + cz * cz, rr = r * r;
                if (cz > r && n2 > rr) {
                    const double tan_t = sqrt(cx * cx + cy * cy) * inv_cz;
                    const double tan_a = pr * cam.inv_f_ppu;  // r / sqrt(|c|^2 - r^2), already computed
                    const double den = 1.0 - tan_t * tan_a;
                    if (den > 1e-6) {
                        rho = cam.focal * ((tan_t + tan_a) / den - tan_t);
                        pcx = cam.focal * cx * inv_cz;
                        pcy = cam.focal * cy * inv_cz;
                    }
                }
            } else {
                pcx = cx; pcy = cy; rho = r;
            }
            const float rho_pad = (float)(rho * (1.0 + 1e-5) + 4e-7 * (fabs(pcx) + fabs(pcy) + cam.sensor_w));
            a.flt[i] = make_float4((float)pcx, (float)pcy, rho_pad * rho_pad * 1.000001f, 0.0f);
            if (on && nt <= 4) {
                const int wx = tr.y - tr.x + 1;
#pragma unroll
                for (int j = 0; j < 4; ++j)  // the slot claimed above is the position inside the tile's bucket
                    if (j < nt && sl[j] < BUCKET_CAP) {
                        const int ty = (j >= wx) + (j >= 2 * wx) + (j >= 3 * wx);
                        a.bucket[(size_t)((tr.z + ty) * cam.ntx + tr.x + (j - ty * wx)) * BUCKET_CAP + sl[j]] = (int)i;
                    }
            }
        }
    }
    if (!a.records_only) {  // one atomic per CTA (31 250 same-address atomics, one per warp, cost 4 us at 1 M spheres)
        const int n_on = __syncthreads_count(on ? 1 : 0);
        if (threadIdx.x == 0 && n_on)
            atomicAdd((unsigned long long *)&a.status[ST_ON_SENSOR], (unsigned long long)n_on);
    }
}

// Single-CTA exclusive scan over the tile counts; also resets the emit cursors, lists the
// tiles whose segment is too long for the small sort kernel, and publishes T / overflow.
__global__ void __launch_bounds__(1024) k_scan(int *tile_count, const int *__restrict__ tile_count_big, int *tile_start,
                                               int *tile_cursor, int *big_tiles, int n_tiles,
                                               long long max_pairs, long long M, long long *status) {
    __shared__ long long warp_sums[32];
    __shared__ long long carry_s;
    __shared__ int n_big, n_over;
    int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) { carry_s = 0; n_big = 0; n_over = 0; }
    __syncthreads();
    // 4 consecutive tiles per thread: 4096 tiles (1024 x 1024 pixels) are one pass with two barriers
    for (int base = 0; base < n_tiles; base += 4096) {
        const int i0 = base + tid * 4;
        int cs[4], c[4];
        long long v = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const bool in = i0 + j < n_tiles;
            cs[j] = in ? tile_count[i0 + j] : 0;
            c[j] = cs[j] + (in ? tile_count_big[i0 + j] : 0);
            v += c[j];
        }
        const long long mine = v;
        for (int o = 1; o < 32; o <<= 1) {
            long long n = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += n;
        }
        if (lane == 31) warp_sums[wid] = v;
        __syncthreads();
        if (wid == 0) {
            long long s = warp_sums[lane];
            for (int o = 1; o < 32; o <<= 1) {
                long long n = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += n;
            }
            warp_sums[lane] = s;
        }
        __syncthreads();
        const long long carry = carry_s;
        long long excl = carry + (wid ? warp_sums[wid - 1] : 0) + v - mine;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (i0 + j < n_tiles) {
                tile_start[i0 + j] = (int)(excl > 0x7fffffffLL ? 0x7fffffffLL : excl);
                tile_cursor[i0 + j] = cs[j];  // ids of spheres touching <= 4 tiles sit at the front of the bucket
                tile_count[i0 + j] = 0;       // consumed: from here on the emit cursor of the fallback path (k_emit)
                if (c[j] > SORT_SMALL) big_tiles[1 + atomicAdd(&n_big, 1)] = i0 + j;
                if (c[j] > BUCKET_CAP) n_over = 1;
            }
            excl += c[j];
        }
        __syncthreads();
        if (tid == 0) carry_s = carry + warp_sums[31];
        __syncthreads();
    }
    if (tid == 0) {
        long long total = carry_s;
        tile_start[n_tiles] = (int)(total > 0x7fffffffLL ? 0x7fffffffLL : total);
        big_tiles[0] = n_big;
        if (n_over) status[ST_FLAGS] |= SS_FLAG_LIST_FALLBACK;  // some bucket overflowed: k_emit builds the lists
        status[ST_PAIRS] = total;
        if (total > max_pairs) status[ST_FLAGS] |= SS_FLAG_PAIR_OVERFLOW;
        long long enc = status[ST_FIRST_INVALID];
        status[ST_FIRST_INVALID] = enc ? M - enc : -1;
    }
}

__global__ void __launch_bounds__(256) k_emit(long long M, const ushort4 *__restrict__ trect,
                                              const unsigned long long *__restrict__ key,
                                              const int *__restrict__ tile_start, int *emit_cursor,
                                              unsigned long long *pair_key, int *pair_id, int ntx,
                                              const long long *__restrict__ status) {
    const long long flags = status[ST_FLAGS];
    if ((flags & SS_FLAG_PAIR_OVERFLOW) || !(flags & SS_FLAG_LIST_FALLBACK)) return;  // the usual case: nothing to do
    // Fallback (some tile holds more than BUCKET_CAP spheres): every (tile, sphere) pair claims its slot in the
    // tile's segment with an atomic on the emit cursor (k_scan left it at zero); the per-tile sort orders the segment.
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < M; i += (long long)gridDim.x * blockDim.x) {
        ushort4 tr = trect[i];
        if (tr.x > tr.y) continue;
        unsigned long long k = key[i];
        for (int ty = tr.z; ty <= tr.w; ++ty)
            for (int tx = tr.x; tx <= tr.y; ++tx) {
                int t = ty * ntx + tx;
                int slot = tile_start[t] + atomicAdd(&emit_cursor[t], 1);
                pair_key[slot] = k;
                pair_id[slot] = (int)i;
            }
    }
}

// The same for segments of up to 4096 pairs (12 position bits, 20 key bits), several 64-blocks per warp, every
// stage through shared memory: keys / ids hold the loaded segment, pk the packed words (4096).
constexpr int PACK_BIG = 4096;
__device__ bool sort_packed4096(int s0, int n, const SegSrc &src, int *pair_id, unsigned long long *keys, int *ids,
                                unsigned *pk) {
    __shared__ unsigned long long s_lo[8], s_hi[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int np2 = 64;
    while (np2 < n) np2 <<= 1;
    const int n_blocks = np2 >> 6;
    unsigned long long lo = ~0ull, hi = 0ull;
    for (int i = tid; i < n; i += blockDim.x) {
        unsigned long long k; int id;
        src.load(i, k, id);
        keys[i] = k; ids[i] = id;
        lo = min(lo, k); hi = max(hi, k);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) { s_lo[warp] = lo; s_hi[warp] = hi; }
    __syncthreads();
#pragma unroll
    for (int w = 0; w < 8; ++w) { lo = min(lo, s_lo[w]); hi = max(hi, s_hi[w]); }
    const int bits = 64 - __clzll((long long)(hi - lo));
    const int shift = bits > 20 ? bits - 20 : 0;
    for (int b = warp; b < n_blocks; b += 8) {
        const int i0 = (b << 6) + lane, i1 = i0 + 32;
        unsigned e0 = i0 < n ? (((unsigned)((keys[i0] - lo) >> shift) << 12) | (unsigned)i0) : 0xffffffffu;
        unsigned e1 = i1 < n ? (((unsigned)((keys[i1] - lo) >> shift) << 12) | (unsigned)i1) : 0xffffffffu;
        u_sort64(e0, e1, lane);
        pk[i0] = e0; pk[i1] = e1;
    }
    __syncthreads();
    const int half = np2 >> 1;
    for (int k = 128; k <= np2; k <<= 1) {
        const int hk = k >> 1;
        for (int c = tid; c < half; c += blockDim.x) {  // flip
            const int q = c & (hk - 1);
            const int l = ((c - q) << 1) + q, r = ((c - q) << 1) + k - 1 - q;
            const unsigned a = pk[l], b = pk[r];
            if (b < a) { pk[l] = b; pk[r] = a; }
        }
        __syncthreads();
        for (int j = hk >> 1; j >= 64; j >>= 1) {  // long-distance disperse stages
            for (int c = tid; c < half; c += blockDim.x) {
                const int q = c & (j - 1);
                const int l = ((c - q) << 1) + q;
                const unsigned a = pk[l], b = pk[l + j];
                if (b < a) { pk[l] = b; pk[l + j] = a; }
            }
            __syncthreads();
        }
        for (int b = warp; b < n_blocks; b += 8) {  // j = 32 .. 1 in registers
            const int i0 = (b << 6) + lane, i1 = i0 + 32;
            unsigned e0 = pk[i0], e1 = pk[i1];
            u_disperse64(e0, e1, lane);
            pk[i0] = e0; pk[i1] = e1;
        }
        __syncthreads();
    }
    return rank_ties_and_write<12>(pk, n, [keys](int i) { return keys[i]; }, ids, pair_id + s0);
}

__global__ void __launch_bounds__(256) k_tile_sort_small(const int *__restrict__ tile_start,
                                                         const unsigned long long *__restrict__ pair_key,
                                                         int *pair_id, const int *__restrict__ bucket,
                                                         const unsigned long long *__restrict__ key,
                                                         const int *__restrict__ tile_cursor,
                                                         const long long *__restrict__ status) {
    __shared__ unsigned long long keys[SORT_SMALL];
    __shared__ int ids[SORT_SMALL];
    __shared__ unsigned pk[PACK_MAX];
    const long long flags = status[ST_FLAGS];
    if (flags & SS_FLAG_PAIR_OVERFLOW) return;
    sort_small_segment(tile_start, pair_key, pair_id, bucket, key, tile_cursor, flags, (int)blockIdx.x, keys, ids, pk);
}

// Segments of 513 .. 4096 pairs in the direct (bucket) path -- every tile of the 10 M-sphere configuration: the
// packed 32-bit sort with the float64 keys held in REGISTERS (<= 16 per thread) instead of a shared-memory
// staging array.  Shared memory per CTA drops from 112 KB (sized for the 8192-pair fallback) to 32 KB (ids +
// packed words), so four CTAs share an SM instead of two: the kernel waits on its random 8-byte key gathers and
// on 78 block barriers, and both hide behind other CTAs.  The few words whose 20-bit key parts tie fetch their
// full keys again for the exact ranking.  A segment with too many ties is left to k_tile_sort_big (its entry in
// big_tiles stays positive); a sorted one is marked done (-1 - tile).
__global__ void __launch_bounds__(256, 4) k_tile_sort_mid(const int *__restrict__ tile_start, int *pair_id,
                                                          const int *__restrict__ bucket,
                                                          const unsigned long long *__restrict__ key,
                                                          const int *__restrict__ tile_cursor, int *big_tiles,
                                                          const long long *__restrict__ status) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    int *ids = (int *)smem_raw;
    unsigned *pk = (unsigned *)(smem_raw + (size_t)PACK_BIG * 4);
    __shared__ unsigned long long s_lo[8], s_hi[8];
    const long long flags = status[ST_FLAGS];
    if (flags & (SS_FLAG_PAIR_OVERFLOW | SS_FLAG_LIST_FALLBACK)) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n_big = big_tiles[0];
    for (int bt = blockIdx.x; bt < n_big; bt += gridDim.x) {
        const int t = big_tiles[1 + bt];
        const int s0 = tile_start[t], n = tile_start[t + 1] - s0;
        if (n > PACK_BIG) continue;
        const int *bk = bucket + (size_t)t * BUCKET_CAP;
        const int c_small = tile_cursor[t];
        __syncthreads();  // previous segment's shared arrays fully consumed
        unsigned long long kr[PACK_BIG / 256];
        unsigned long long lo = ~0ull, hi = 0ull;
#pragma unroll
        for (int j = 0; j < PACK_BIG / 256; ++j) {
            const int i = tid + 256 * j;
            kr[j] = ~0ull;
            if (i < n) {
                const int id = bk[i < c_small ? i : BUCKET_CAP - 1 - (i - c_small)];
                ids[i] = id;
                kr[j] = key[id];
            }
        }
#pragma unroll
        for (int j = 0; j < PACK_BIG / 256; ++j)
            if (tid + 256 * j < n) { lo = min(lo, kr[j]); hi = max(hi, kr[j]); }
        for (int o = 16; o > 0; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (lane == 0) { s_lo[warp] = lo; s_hi[warp] = hi; }
        __syncthreads();
#pragma unroll
        for (int w = 0; w < 8; ++w) { lo = min(lo, s_lo[w]); hi = max(hi, s_hi[w]); }
        const int bits = 64 - __clzll((long long)(hi - lo));
        const int shift = bits > 20 ? bits - 20 : 0;
        int np2 = 64;
        while (np2 < n) np2 <<= 1;
        const int n_blocks = np2 >> 6;
#pragma unroll
        for (int j = 0; j < PACK_BIG / 256; ++j) {
            const int i = tid + 256 * j;
            if (i < np2) pk[i] = i < n ? (((unsigned)((kr[j] - lo) >> shift) << 12) | (unsigned)i) : 0xffffffffu;
        }
        __syncthreads();
        for (int b = warp; b < n_blocks; b += 8) {
            const int i0 = (b << 6) + lane, i1 = i0 + 32;
            unsigned e0 = pk[i0], e1 = pk[i1];
            u_sort64(e0, e1, lane);
            pk[i0] = e0; pk[i1] = e1;
        }
        __syncthreads();
        const int half = np2 >> 1;
        for (int k = 128; k <= np2; k <<= 1) {
            const int hk = k >> 1;
            for (int c = tid; c < half; c += blockDim.x) {  // flip
                const int q = c & (hk - 1);
                const int l = ((c - q) << 1) + q, r = ((c - q) << 1) + k - 1 - q;
                const unsigned a = pk[l], b = pk[r];
                if (b < a) { pk[l] = b; pk[r] = a; }
            }
            __syncthreads();
            for (int j = hk >> 1; j >= 64; j >>= 1) {  // long-distance disperse stages
                for (int c = tid; c < half; c += blockDim.x) {
                    const int q = c & (j - 1);
                    const int l = ((c - q) << 1) + q;
                    const unsigned a = pk[l], b = pk[l + j];
                    if (b < a) { pk[l] = b; pk[l + j] = a; }
                }
                __syncthreads();
            }
            for (int b = warp; b < n_blocks; b += 8) {  // j = 32 .. 1 in registers
                const int i0 = (b << 6) + lane, i1 = i0 + 32;
                unsigned e0 = pk[i0], e1 = pk[i1];
                u_disperse64(e0, e1, lane);
                pk[i0] = e0; pk[i1] = e1;
            }
            __syncthreads();
        }
        const bool ok = rank_ties_and_write<12>(pk, n, [key, ids](int i) { return key[ids[i]]; }, ids, pair_id + s0);
        if (ok && tid == 0) big_tiles[1 + bt] = -1 - t;
    }
}

// Persistent over the list of long segments (> SORT_SMALL pairs).  <= 4096: packed 32-bit sort, input from the tile's
// bucket (or from the emitted pairs in the fallback path); <= SORT_BIG: 64-bit network in dynamic smem; longer: in
// place in global memory.  Segments beyond 4096 only exist in the fallback path (they overflow the bucket).
__global__ void __launch_bounds__(256) k_tile_sort_big(const int *__restrict__ tile_start,
                                                       unsigned long long *pair_key, int *pair_id,
                                                       const int *__restrict__ bucket,
                                                       const unsigned long long *__restrict__ key,
                                                       const int *__restrict__ tile_cursor,
                                                       const int *__restrict__ big_tiles,
                                                       const long long *__restrict__ status) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    unsigned long long *keys = (unsigned long long *)smem_raw;
    int *ids = (int *)(smem_raw + (size_t)SORT_BIG * 8);
    unsigned *pk = (unsigned *)(smem_raw + (size_t)SORT_BIG * 12);
    const long long flags = status[ST_FLAGS];
    if (flags & SS_FLAG_PAIR_OVERFLOW) return;
    int n_big = big_tiles[0];
    for (int b = blockIdx.x; b < n_big; b += gridDim.x) {
        int t = big_tiles[1 + b];
        if (t < 0) continue;  // sorted by k_tile_sort_mid
        int s0 = tile_start[t], n = tile_start[t + 1] - s0;
        SegSrc src;
        src.direct = !(flags & SS_FLAG_LIST_FALLBACK);
        src.pair_key = pair_key + s0; src.pair_id = pair_id + s0;
        src.bucket = bucket + (size_t)t * BUCKET_CAP; src.key = key;
        src.c_small = tile_cursor[t];
        __syncthreads();  // previous segment's shared arrays fully consumed
        if (n <= PACK_BIG && sort_packed4096(s0, n, src, pair_id, keys, ids, pk)) continue;
        if (n <= SORT_BIG) {
            __syncthreads();
            for (int i = threadIdx.x; i < n; i += blockDim.x) src.load(i, keys[i], ids[i]);
            __syncthreads();
            bitonic_sort_cta(keys, ids, n);
            for (int i = threadIdx.x; i < n; i += blockDim.x) pair_id[s0 + i] = ids[i];
        } else {
            bitonic_sort_cta(pair_key + s0, pair_id + s0, n);  // global memory, one CTA: slow but exact
        }
    }
}

}  // namespace

cudaError_t launch_project(const FwdLaunch &a, bool records_only, cudaStream_t s) {
    long long M = a.dims.num_spheres;
    char *ws = a.ws;
    const Layout &L = a.L;
    if (!records_only) {
        // status + tile_count + tile_count_big are contiguous: one memset
        ProfScope ps(KID_MEMSET_FWD, s);
        cudaError_t e = cudaMemsetAsync(ws + L.status, 0, L.tile_start - L.status, s);
        if (e != cudaSuccess) return e;
    }
    if (M > 0) {
        ProjectArgs p;
        p.M = M; p.d = a.dims.feature_dim;
        p.pos = a.pos; p.rad = a.rad; p.opa = a.opa; p.feat = a.feat; p.bg = a.bg;
        p.cam = a.cam;
        p.rec = (Rec *)(ws + L.rec); p.key = (unsigned long long *)(ws + L.key);
        p.trect = (ushort4 *)(ws + L.trect); p.proj_r = (double *)(ws + L.proj_r);
        p.flt = (float4 *)(ws + L.flt);
        p.tile_count = (int *)(ws + L.tile_count); p.tile_count_big = (int *)(ws + L.tile_count_big);
        p.bucket = (int *)(ws + L.bucket); p.status = (long long *)(ws + L.status);
        p.rect = a.rect; p.on_sensor = a.on_sensor; p.earliest = a.earliest; p.proj_r_out = a.proj_r_out;
        p.records_only = records_only ? 1 : 0;
        p.validate = (!records_only && !(a.blend.flags & SS_OPT_SKIP_VALIDATE)) ? 1 : 0;
        unsigned grid = (unsigned)((M + 255) / 256);
        ProfScope ps(KID_PROJECT, s);
        k_project<<<grid, 256, 0, s>>>(p);
        count_launch();
    }
    return cudaGetLastError();
}

// Long-segment sort kernels on a side stream beside k_tile_sort_small (compile-time experiment, OFF): one view per step
// gains 0.15 % graph-replayed / 1 % stream-launched (the two kernels are early exits there), but the 64-view step,
// whose two pipeline lanes already fill the machine, loses 12 % as a graph replay (2 389 -> 2 101 frames/s: the extra
// branches and joins of 64 forks) and 1.5 % stream-launched.
#ifndef SS_SORT_FORK
#define SS_SORT_FORK 0
#endif
// Two side streams (used alternately) + fork / join events per host thread and device, created on first use and kept for the life of
// the thread (the only CUDA objects this library owns).  Per THREAD: an event re-recorded by another thread between
// this thread's record and wait would hand the wait the wrong dependency.
struct SideStreams {
    cudaStream_t s1 = nullptr;
    cudaEvent_t fork = nullptr, join1 = nullptr;
    bool ok = false, tried = false;
};
struct SideStreamPair {  // consecutive calls alternate: the two lanes of a pipelined multi-view step do not share one
    SideStreams lane[2];
    unsigned calls = 0;
};
static SideStreams *side_streams() {
    static thread_local SideStreamPair per_dev[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    for (SideStreams &x : per_dev[dev].lane) {  // both lanes on first use (a warm-up call then covers a later capture)
        if (x.tried) continue;
        x.tried = true;
        x.ok = cudaStreamCreateWithFlags(&x.s1, cudaStreamNonBlocking) == cudaSuccess &&
               cudaEventCreateWithFlags(&x.fork, cudaEventDisableTiming) == cudaSuccess &&
               cudaEventCreateWithFlags(&x.join1, cudaEventDisableTiming) == cudaSuccess;
        if (!x.ok) (void)cudaGetLastError();
    }
    SideStreams &x = per_dev[dev].lane[per_dev[dev].calls++ & 1u];
    return x.ok ? &x : nullptr;
}

bool side_stream(cudaStream_t *side, cudaEvent_t *fork, cudaEvent_t *join) {
    SideStreams *x = side_streams();
    if (!x) return false;
    *side = x->s1; *fork = x->fork; *join = x->join1;
    return true;
}

cudaError_t launch_binning(const FwdLaunch &a, cudaStream_t s) {
    long long M = a.dims.num_spheres;
    char *ws = a.ws;
    const Layout &L = a.L;
    int *tile_start = (int *)(ws + L.tile_start);
    int *tile_cursor = (int *)(ws + L.tile_cursor);
    int *big_tiles = (int *)(ws + L.big_tiles);
    long long *status = (long long *)(ws + L.status);
    unsigned long long *pair_key = (unsigned long long *)(ws + L.pair_key);
    int *pair_id = (int *)(ws + L.pair_id);
    {
        ProfScope ps(KID_SCAN, s);
        k_scan<<<1, 1024, 0, s>>>((int *)(ws + L.tile_count), (const int *)(ws + L.tile_count_big),
                                  tile_start, tile_cursor, big_tiles, L.n_tiles, a.dims.max_pairs, M, status);
    }
    count_launch();
    if (M > 0) {
        unsigned grid = (unsigned)((M + 255) / 256);
        if (grid > 148) grid = 148;  // grid-stride: in the usual (bucket) case the launch is an early exit
        {
            ProfScope ps(KID_EMIT, s);
            k_emit<<<grid, 256, 0, s>>>(M, (const ushort4 *)(ws + L.trect),
                                        (const unsigned long long *)(ws + L.key), tile_start, (int *)(ws + L.tile_count),
                                        pair_key, pair_id, L.ntx, status);
        }
        // The small-segment kernel and the two long-segment kernels work on disjoint tiles (segments of <= 512 pairs
        // against the list of longer ones), and the long-segment kernels are usually a list of a few tiles or an early
        // exit, so those two run on a side stream beside the small-segment kernel (fork after k_emit, join before the
        // raster pass; under stream capture the event waits become graph edges) instead of as two more serial steps
        // of the frame.  k_tile_sort_mid and k_tile_sort_big stay IN ORDER on that one stream: the second one skips
        // the list entries the first one has marked as sorted.
        SideStreams *side = SS_SORT_FORK ? side_streams() : nullptr;
        cudaStream_t s_mid = s, s_big = s;
        if (side) {
            if (cudaEventRecord(side->fork, s) != cudaSuccess || cudaStreamWaitEvent(side->s1, side->fork, 0) != cudaSuccess)
                return cudaGetLastError();
            s_mid = side->s1; s_big = side->s1;
        }
        if (!SS_FUSED_SORT) {
            ProfScope ps(KID_SORT_SMALL, s);
            k_tile_sort_small<<<L.n_tiles, 256, 0, s>>>(tile_start, pair_key, pair_id, (const int *)(ws + L.bucket),
                                                        (const unsigned long long *)(ws + L.key), tile_cursor, status);
        }
        static PerDeviceOnce attr_once;
        size_t big_smem = (size_t)SORT_BIG * 12 + (size_t)PACK_BIG * 4;
        if (attr_once.first()) {
            cudaError_t e = cudaFuncSetAttribute(k_tile_sort_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)big_smem);
            if (e != cudaSuccess) return e;
        }
        {
            static PerDeviceOnce mid_once;
            const size_t mid_smem = (size_t)PACK_BIG * 8;
            if (mid_once.first()) {
                cudaError_t e = cudaFuncSetAttribute(k_tile_sort_mid, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)mid_smem);
                if (e != cudaSuccess) return e;
            }
            const int grid_mid = L.n_tiles < 148 * 4 ? L.n_tiles : 148 * 4;
            ProfScope ps(KID_SORT_BIG, s_mid);
            k_tile_sort_mid<<<grid_mid, 256, mid_smem, s_mid>>>(tile_start, pair_id, (const int *)(ws + L.bucket),
                                                            (const unsigned long long *)(ws + L.key), tile_cursor,
                                                            big_tiles, status);
            count_launch();
        }
        int grid_big = L.n_tiles < 296 ? L.n_tiles : 296;
        {
            ProfScope ps(KID_SORT_BIG, s_big);
            k_tile_sort_big<<<grid_big, 256, big_smem, s_big>>>(tile_start, pair_key, pair_id, (const int *)(ws + L.bucket),
                                                                (const unsigned long long *)(ws + L.key), tile_cursor,
                                                                big_tiles, status);
        }
        count_launch(SS_FUSED_SORT ? 2 : 3);
        if (side) {
            if (cudaEventRecord(side->join1, side->s1) != cudaSuccess || cudaStreamWaitEvent(s, side->join1, 0) != cudaSuccess)
                return cudaGetLastError();
        }
    }
    return cudaGetLastError();
}

}  // namespace ss
