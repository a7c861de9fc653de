// Forward raster kernel for sm_100a (reference _draw_tile, raster.py:328-417).
//
// One 256-thread CTA per 16x16 tile, one thread per pixel, one 8x4 pixel block per warp.  The tile's
// depth-ordered candidate list is streamed in batches of `chunk` (<= 256) records staged in shared memory.
// Per batch a warp (1) compacts the candidates whose bounding circle reaches its pixel block, (2) filters
// them 32 at a time -- all lanes look at the same candidate, so the filter's shared-memory reads are
// broadcasts -- into one bit word per lane, and (3) drains those words: every lane evaluates ITS oldest
// pending candidate exactly, so the divergent hit path runs with most lanes busy.
//
// Precision plan: the float64 reference decides hits with
// dist^2 = |c|^2 - t^2 and orders the per-pixel top-K by float64 NDC depth.  Here a cheap
// float32 screen-space test filters candidates: a pixel can only hit a sphere if it lies inside
// the circle, centred on the projected sphere centre, that bounds the sphere's projected
// outline (radius f (tan(theta + alpha) - tan(theta)), widened for float32 rounding).  Every
// candidate that passes is re-evaluated with the reference's own float64 formula, which alone
// decides hit / miss.  The blend (online softmax of Eq. 1) runs in float32 on a float32 depth; the
// float64 depth that ORDERS the top-K record is only formed for hits that pass a float32 pre-filter
// against the record's worst entry (padded by 4x the float32 error), i.e. for hits that can enter it.
#include <math.h>

#include <type_traits>

#include "ss_common.cuh"
#if SS_FUSED_SORT
#include "ss_sort.cuh"
#endif

namespace ss {

namespace {

struct RasterArgs {
    Cam cam;
    const int *tile_start;
    int *pair_id;  // sorted per-tile lists; written by this kernel when it sorts its own tile (sort_here)
    // inputs of the fused per-tile sort (sort_small_segment)
    const unsigned long long *pair_key, *key;
    const int *bucket, *tile_cursor;
    int sort_here;
    const Rec *rec;
    const float4 *flt;
    const float *feat;
    const float *bg;
    int d, K, chunk;
    int tile0;  // first tile of this launch (ss_forward_banded draws the image in bands of tile rows)
    double gamma, eps_over_g, log_tau;
    // float32 depth used for the blend exponent and as a pre-filter of the top-K (the float64 depth is only
    // formed for hits that can enter the record): far, far - near, 1 / (far - near), error pad of the pre-filter
    float far_f, fmn_f, inv_range_f, zpad;
    float ppu_f, ppu2_f;  // pixels per sensor unit and its square (the filter works in pixel units)
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
    int n;  // filled slots: a new entry starts at slot n, not at the bottom of an empty record
    // The LAST entry (slot n - 1; of a full record: the admission threshold) cached in registers.  With n_track = 32
    // the arrays live in local memory (3 CTAs x 128 KB per SM do not fit the L1): candidates arrive roughly front to
    // back, so while the record fills up the usual insert is an append behind the cached last entry (three local
    // stores, no load), and once it is full the usual hit is rejected against the cache (float32 pre-filter first:
    // wlo, formed without the float64 depth).
    double wz; int wid; float wlo;
    __device__ __forceinline__ void init() {
        // The arrays are NOT cleared: slots at and beyond n are never read (the insert bubbles inside [0, n), the
        // getters answer "empty" there), and clearing 16 KT bytes per pixel was 1 GB of local-memory stores per C5
        // frame, most of it evicted to DRAM.
        n = 0;
        wz = -INFINITY; wid = -1; wlo = -INFINITY;
    }
    __device__ __forceinline__ void bind(unsigned char *, int) {}
    __device__ __forceinline__ double get_z(int k) const { return k < n ? z[k] : -INFINITY; }
    __device__ __forceinline__ int get_id(int k) const { return k < n ? id[k] : -1; }
    __device__ __forceinline__ float get_c(int k) const { return k < n ? c[k] : 0.0f; }
    __device__ __forceinline__ bool may_enter(float zzf) const { return zzf >= wlo; }
    // keep the KT largest by (z desc, id asc) -- raster.py:389-399
    __device__ __forceinline__ void insert(double zz, int sid, float cl, float pad) {
        const bool beats_last = n > 0 && (zz > wz || (zz == wz && sid < wid));
        int k;
        if (n < KT) {
            k = n++;
            if (!beats_last) {  // in order: append, the new entry is the last one
                z[k] = zz; id[k] = sid; c[k] = cl;
                wz = zz; wid = sid;
                if (n == KT) wlo = (float)wz - pad;
                return;
            }
            // out of order: the last entry moves down one slot (and stays the last: the cache is unchanged)
            z[k] = wz; id[k] = wid; c[k] = c[k - 1];
            --k;
        } else {
            if (!beats_last) return;
            k = KT - 1;  // the worst entry drops out
        }
#pragma unroll 1
        while (k > 0) {
            const double zp = z[k - 1];
            const int ip = id[k - 1];
            if (!(zz > zp || (zz == zp && sid < ip))) break;
            z[k] = zp; id[k] = ip; c[k] = c[k - 1];
            --k;
        }
        z[k] = zz; id[k] = sid; c[k] = cl;
        if (n == KT) {  // the record is (or has just become) full: refresh the cached threshold
            wz = z[KT - 1]; wid = id[KT - 1];
            wlo = (float)wz - pad;
        }
    }
};

// Shared-memory variant for K <= 8: the K x 256 record lives in shared memory (column tid), only the
// current worst entry (the admission threshold) is cached in registers.  Frees ~17 registers per
// thread, which lets a fourth CTA fit on each SM.
template <int KT>
struct TopKShared {
    double *z; int *id; float *c;  // this thread's column: slot k at [k * TILE_PX]
    // cached slot KT-1 of a FULL record.  While the record is filling up, wz = -inf admits everything and wid carries
    // the fill count as -1 - n (no extra register): a new entry then starts at slot n instead of bubbling up from the
    // bottom through the empty slots (10 shifts of 6 shared-memory accesses for the first five hits of every pixel),
    // and the columns need no clearing.
    double wz; int wid;
    float wlo;                     // (float)wz - pad: a float32 depth below this cannot enter the record
    __device__ __forceinline__ void bind(unsigned char *base, int tid) {
        z = (double *)base + tid;
        id = (int *)(base + (size_t)KT * TILE_PX * 8) + tid;
        c = (float *)(base + (size_t)KT * TILE_PX * 12) + tid;
    }
    __device__ __forceinline__ void init() { wz = -INFINITY; wid = -1; wlo = -INFINITY; }
    __device__ __forceinline__ int filled() const { return wid < 0 && wz == -INFINITY ? -1 - wid : KT; }
    __device__ __forceinline__ bool may_enter(float zzf) const { return zzf >= wlo; }
    __device__ __forceinline__ void insert(double zz, int sid, float cl, float pad) {
        int k;
        const bool filling = wlo == -INFINITY;  // (pad is finite, so a full record has a finite or NaN-free threshold)
        if (filling) {
            k = -1 - wid;
        } else {
            if (!(zz > wz || (zz == wz && sid < wid))) return;
            k = KT - 1;
        }
        while (k > 0) {
            const double zk = z[(k - 1) * TILE_PX];
            const int ik = id[(k - 1) * TILE_PX];
            if (!(zz > zk || (zz == zk && sid < ik))) break;
            z[k * TILE_PX] = zk; id[k * TILE_PX] = ik; c[k * TILE_PX] = c[(k - 1) * TILE_PX];
            --k;
        }
        z[k * TILE_PX] = zz; id[k * TILE_PX] = sid; c[k * TILE_PX] = cl;
        if (filling && wid > -KT) {  // still not full afterwards: n + 1 < KT
            --wid;
        } else {
            wz = z[(KT - 1) * TILE_PX]; wid = id[(KT - 1) * TILE_PX];
            wlo = (float)wz - pad;
        }
    }
    __device__ __forceinline__ double get_z(int k) const { return k < filled() ? z[k * TILE_PX] : -INFINITY; }
    __device__ __forceinline__ int get_id(int k) const { return k < filled() ? id[k * TILE_PX] : -1; }
    __device__ __forceinline__ float get_c(int k) const { return k < filled() ? c[k * TILE_PX] : 0.0f; }
};

#ifndef SS_RASTER_INT_CVT
// Conversions done with integer instructions instead of F2F in the d <= 4, n_track <= 8 instantiations (bit mask:
// 1 = r -> float64, 2 = dist^2 -> float32, 4 = r^2 - dist^2 -> float32; every combination gives the same values).
// Measured at C3 (k_raster, us): 0: 244.6, 1: 247.5, 2: 245.4, 3: 248.3, 4: 243.7, 5: 246.4, 6: 245.8, 7: 248.0 -- the XU
// pipe and the ALU are balanced after the other changes of the hit path, only the last one pays.
#define SS_RASTER_INT_CVT 4
#endif
#ifndef SS_TOPK_SHARED
#define SS_TOPK_SHARED 1  // K <= 8: top-K record in shared memory (1) or registers (0)
#endif

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// float64 -> float32 of a value that is positive and inside the float32 normal range, truncated instead of rounded
// (1 ulp instead of 1/2 ulp), with integer instructions: F2F.F32.F64 runs on the XU pipe (16 lanes per clock and SM),
// which paces the hit path together with the MUFU operations.  Anything else (negative, zero, below 2^-126) gives 0.
__device__ __forceinline__ float trunc_f64_to_f32(double x) {
    const int hi = __double2hiint(x);
    const unsigned b = __funnelshift_l((unsigned)__double2loint(x), (unsigned)(hi - 0x38000000), 3);
    return hi >= 0x38100000 ? __uint_as_float(b) : 0.0f;
}
// keeps a value in a register: stops the compiler from re-deriving it (e.g. re-converting the
// float64 ray to float32 inside the test loop)
__device__ __forceinline__ float pin_reg(float x) {
    asm volatile("" : "+f"(x));
    return x;
}

// Shared-memory loads through an explicit 32-bit shared-space address.  With generic pointers into the dynamic
// shared array the compiler, at the 64-register cap, re-derives the shared window base (S2R SR_CgaCtaId + 3
// integer instructions) in EVERY drain round instead of keeping it in a register.
__device__ __forceinline__ float4 lds_f4(unsigned a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ double2 lds_d2(unsigned a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ unsigned lds_u8(unsigned a) {
    unsigned v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ unsigned lds_u32(unsigned a) {
    unsigned v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

constexpr float kLn2 = 0.6931471805599453f;
#ifndef SS_RASTER_MINB_WIDE
#define SS_RASTER_MINB_WIDE 3  // d <= 16 or long records
#endif
#ifndef SS_RASTER_MINB
#define SS_RASTER_MINB (SS_TOPK_SHARED ? 4 : 3)  // resident CTAs per SM the register allocation targets (d <= 4, K <= 8)
#endif

// floats per staged hit record: 12 + features, padded so that the stride is not a multiple of 8 words (records
// would otherwise start in only 2 or 4 distinct bank groups and the divergent 128-bit loads would serialise)
template <int DP>
constexpr int rec_stride() {
    // d = 3: 48-byte record [cx, cy | cz, r, id | o, f0, f1, f2] -- |c|^2 and o/gamma are re-formed per hit
    // (3 DFMA + 1 FMUL cost less than a fourth divergent 128-bit load)
    return DP == 3 ? 12 : ((12 + ((DP + 3) & ~3)) % 8 == 0 ? 16 + ((DP + 3) & ~3) : 12 + ((DP + 3) & ~3));
}

template <int DP, int KT, int MODE>
__global__ void __launch_bounds__(TILE_PX, (KT <= 8 && DP <= 4) ? SS_RASTER_MINB : (DP <= 16 ? SS_RASTER_MINB_WIDE : 2)) k_raster(RasterArgs a) {
    constexpr int CAP = SS_MAX_CHUNK;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int RS = rec_stride<DP>();           // floats per staged candidate
    float4 *s_cf = (float4 *)smem_raw;            // float32 filter: centre (ortho: cx, cy, -), widened r^2
    // hit record, one per candidate, read with 128-bit loads by the divergent hit path:
    // [cx, cy] [cz, |c|^2] (float64) [r, clamped opacity o, o / gamma * log2(e), sphere id bits] [features]
    float *s_rec = (float *)(s_cf + CAP);
    unsigned char *s_wmask = (unsigned char *)(s_rec + CAP * RS);  // per candidate: which warps' pixel blocks it can touch
    unsigned char *s_list = s_wmask + CAP;         // per warp: compacted indices of its relevant candidates
    constexpr int LSTRIDE = CAP + 4;
    __shared__ float4 s_rect[8];                   // per warp: sensor-space rectangle of its pixel centres
    __shared__ float2 s_org[8];                    // per warp: sensor coordinates of its first pixel centre
    __shared__ double s_red[8];
    __shared__ unsigned long long s_stat[3];

    const Cam &cam = a.cam;
    const int tile = blockIdx.x + a.tile0;
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    // each warp owns an 8x4 pixel block of the 16x16 tile (2 x 4 blocks): a sphere footprint
    // touches fewer warps than with 16x2 strips, and a warp row is one 32-byte sector
    const int lx = ((warp & 1) << 3) | (lane & 7);
    const int ly = ((warp >> 1) << 2) | (lane >> 3);
    const int px = (tile % cam.ntx) * TILE + lx;
    const int py = (tile / cam.ntx) * TILE + ly;
    const bool valid = px < cam.W && py < cam.H;

    // pixel-centre ray, camera frame (camera.py:332-357)
    const double xs = ((px + 0.5) - cam.W / 2.0) * cam.pix;
    const double ys = ((py + 0.5) - cam.H / 2.0) * cam.pix;
    double ux = 0.0, uy = 0.0, uz = 1.0;
    if (MODE == SS_MODE_PINHOLE) {
        double vn = sqrt(xs * xs + ys * ys + cam.focal * cam.focal);
        ux = xs / vn; uy = ys / vn; uz = cam.focal / vn;
    }
    // sensor-space rectangle spanned by this warp's in-image pixel centres (empty: +inf/-inf).  The centres grow with
    // the pixel index, so the rectangle is the first and the last valid column / row of the block -- computed by lane
    // 0 from the indices (same expression as xs / ys above: same bits) instead of a 20-shuffle min / max butterfly.
    if (lane == 0) {
        const int nx = min(8, cam.W - px), ny = min(4, cam.H - py);  // valid columns / rows of this block (lane 0 = its corner)
        float4 rc4 = make_float4(INFINITY, -INFINITY, INFINITY, -INFINITY);
        if (nx > 0 && ny > 0) {
            rc4.x = (float)xs; rc4.y = (float)((((px + nx - 1) + 0.5) - cam.W / 2.0) * cam.pix);
            rc4.z = (float)ys; rc4.w = (float)((((py + ny - 1) + 0.5) - cam.H / 2.0) * cam.pix);
        }
        s_rect[warp] = rc4;
        s_org[warp] = make_float2((float)xs, (float)ys);  // pixel centre of the block's column 0, row 0
    }
    __syncwarp();

    const long long ws_flags = a.status[ST_FLAGS];
    const bool overflow = (ws_flags & SS_FLAG_PAIR_OVERFLOW) != 0;  // lists not built
    const int s0 = a.tile_start[tile];
    const int n_cand = overflow ? 0 : a.tile_start[tile + 1] - s0;
#if SS_FUSED_SORT
    // Fused per-tile sort (experiment, off by default): a tile with <= 512 candidates orders its own list here, in
    // the staging area of its shared memory, instead of in k_tile_sort_small in front of this kernel -- the idea
    // being that the sort would run in the issue slots the drain rounds of the other resident tiles leave idle.
    // Measured at C3: 302 us against 258 + 41 us for the two kernels, i.e. nothing is hidden: both are bound by the
    // same load/store path (shared-memory wavefronts here, shuffles there), not by issue slots.
    if (a.sort_here && n_cand >= 1 && n_cand <= SORT_SMALL) {
        sort_small_segment(a.tile_start, a.pair_key, a.pair_id, a.bucket, a.key, a.tile_cursor, ws_flags, tile,
                           (unsigned long long *)smem_raw, (int *)(smem_raw + SORT_SMALL * 8),
                           (unsigned *)(smem_raw + SORT_SMALL * 12));
        __syncthreads();  // the sorted ids (global) and the scratch (shared, reused by the staging) are settled
    }
#endif

    // tile-wide minimum ray cosine for the early-stop bound (raster.py:358)
    double tile_cos = 1.0;
    if (a.tau_on && MODE == SS_MODE_PINHOLE && n_cand > 0) {
        // u_z = f / |v| falls with |x_s| and |y_s| (every rounding on the way is monotone), so the minimum over the
        // tile's in-image pixels sits at one of the four corners of its valid part: those (up to) four threads publish
        // their value -- no butterfly over 256 lanes
        const int nxt = min(TILE, cam.W - (px - lx)), nyt = min(TILE, cam.H - (py - ly));
#pragma unroll
        for (int cnr = 0; cnr < 4; ++cnr)
            if (lx == ((cnr & 1) ? nxt - 1 : 0) && ly == ((cnr & 2) ? nyt - 1 : 0)) s_red[cnr] = uz;
        __syncthreads();
        double v = s_red[0];
#pragma unroll
        for (int w = 1; w < 4; ++w) { const double o = s_red[w]; v = o < v ? o : v; }
        tile_cos = v;
    }
    if (tid < 3) s_stat[tid] = 0;

    // blend state in base-2 exponent units: mass = o c 2^(e2), e2 = o z / gamma * log2(e)
    const float m2_bg = (float)(a.eps_over_g * 1.4426950408889634);
    float m2 = m2_bg, denom = 1.0f;
    float num[DP];
#pragma unroll
    for (int i = 0; i < DP; ++i) num[i] = 0.0f;
    constexpr bool kTopShared = (SS_TOPK_SHARED != 0) && KT <= 8;
    typename std::conditional<kTopShared, TopKShared<KT>, TopK<KT>>::type top;
    top.bind(s_list + 8 * LSTRIDE, tid);  // shared variant: KT x 256 x 16 B behind the warp lists
    top.init();
    bool done = !valid;
    unsigned n_hits = 0;
    long long scanned = 0;
    const double near_ = cam.near_, far_ = cam.far_, inv_range = cam.inv_range;
    const float inv_g2 = (float)(1.4426950408889634 / a.gamma);

    // exact hit evaluation for one queued candidate (reference raster.py:307-324, :380-399)
    unsigned s_rec_a = (unsigned)__cvta_generic_to_shared(s_rec);
    asm volatile("" : "+r"(s_rec_a));  // opaque: keep it in a register instead of re-deriving it per round
    auto process = [&](unsigned j) {
        const unsigned ra = s_rec_a + j * (RS * 4);
        const double2 cxy = lds_d2(ra);
        constexpr bool kCompact = DP == 3;
        double2 czn;
        float4 mi;  // r, clamped opacity o, 1 / r, sphere id bits (d = 3: the id stays in the filter record)
        float4 f3 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (kCompact) {
            const float4 q = lds_f4(ra + 16);   // cz (float64), r, 1 / r
            czn.x = __hiloint2double(__float_as_int(q.y), __float_as_int(q.x));
            czn.y = cxy.x * cxy.x + cxy.y * cxy.y + czn.x * czn.x;
            mi = make_float4(q.z, 0.0f, q.w, 0.0f);  // the third quad (o, f0, f1, f2) is read once the hit is decided
        } else {
            czn = lds_d2(ra + 16);
            mi = lds_f4(ra + 32);
        }
        // dist2 is NOT clamped at zero here (raster.py:311 clamps): a slightly negative value (ray through the
        // centre, cancellation noise ~1e-13) leaves the decision hc2 > 0 and every float32 consumer unchanged
        // (d2f is clamped below, the float32 value of hc2 is that of r^2); only the rare t <= 0 branch needs the clamp.
        double t, dist2, zeta;
        if (MODE == SS_MODE_PINHOLE) {
            t = ux * cxy.x + uy * cxy.y + uz * czn.x;
            dist2 = czn.y - t * t;
            zeta = t * uz;
        } else {
            t = czn.x;
            const double dx = cxy.x - xs, dy = cxy.y - ys;
            dist2 = dx * dx + dy * dy;
            zeta = t;
        }
        const float rf = mi.x;
        // r^2 - dist^2 in one rounding: r is a float32 value, so r * r is exact in float64 and the fused form
        // equals the reference's (r * r) - dist2 bit for bit.  The hit path is paced by the XU pipe (conversions that
        // touch a 64-bit value, MUFU, bit scans: 16 lanes per clock and SM) as much as by issue slots; conversions can
        // be moved to the ALU (SS_RASTER_INT_CVT: float -> double of a normal positive radius is three integer
        // instructions), which pays for some of them only, and only in the short-record instantiations at 4 CTAs per
        // SM (with wide payloads / long records the kernel waits on local memory: C5 2.92 -> 2.98 ms with all three).
        constexpr bool kXuDiet = KT <= 8 && DP <= 4;
        double rd = (double)rf;
        if (kXuDiet && (SS_RASTER_INT_CVT & 1)) {
            const unsigned rb = __float_as_uint(rf);
            rd = __hiloint2double((int)((rb >> 3) + 0x38000000u), (int)(rb << 29));
            // zero / subnormal radius: the exact conversion (never at sane scales; volatile so that the compiler
            // branches around it instead of executing it for every candidate and selecting)
            if (rb < 0x00800000u) asm volatile("cvt.f64.f32 %0, %1;" : "=d"(rd) : "f"(rf));
        }
        const double hc2 = fma(rd, rd, -dist2);
        // dist2 < r^2 and t + half_chord > 0
        if (hc2 > 0.0 && (t > 0.0 || t + sqrt(fmin(hc2, rd * rd)) > 0.0)) {
            ++n_hits;
            if (kCompact) { f3 = lds_f4(ra + 32); mi.y = f3.x; }
            // float32 NDC depth for the blend exponent: (far - clip(zeta)) / (far - near); the float64 product t u_z is
            // needed by the top-K insert anyway, so ONE conversion (of zeta) replaces two (t and u_z)
            const float zeta_f = (float)zeta;
            const float zzf = fmaxf(fminf(a.far_f - zeta_f, a.fmn_f), 0.0f) * a.inv_range_f;
            // closeness 1 - dist/r as (r^2 - dist^2) / (r (r + dist)): no cancellation near the rim (1 - dist / r in
            // float32 has an ABSOLUTE error of 2e-7, which a hard-gamma stack turns into 1e-4 of the image).  Both
            // float64 -> float32 conversions go TOWARDS ZERO, either as F2F.RZ (XU pipe) or as an integer truncation
            // (ALU; SS_RASTER_INT_CVT picks per value): the same bits in every instantiation, so that n_track = 8 / 16 /
            // 32 render identical images (reference tests/test_grad.py:147-164).
            constexpr bool kIntD2 = kXuDiet && (SS_RASTER_INT_CVT & 2), kIntHc = kXuDiet && (SS_RASTER_INT_CVT & 4);
            const float d2f = fmaxf(kIntD2 ? trunc_f64_to_f32(dist2) : __double2float_rz(dist2), 1e-37f);
            float hc2f = kIntHc ? trunc_f64_to_f32(hc2) : __double2float_rz(hc2);
            if (!kIntHc && hc2f < 1.17549435e-38f) hc2f = 0.0f;
            const float cl = hc2f * mi.z * rcp_approx(fmaf(d2f, rsqrt_approx(d2f), rf));
            const float e2 = zzf * (mi.y * inv_g2);
            if (e2 > m2) {  // online form of raster.py:382-387
                const float sc = ex2_approx(m2 - e2);
                denom *= sc;
#pragma unroll
                for (int i = 0; i < DP; ++i) num[i] *= sc;
                m2 = e2;
            }
            const float oc = mi.y * cl;
            const float x2 = e2 - m2;
            const float term = oc * ex2_approx(x2);
            denom += term;
            if (kCompact) {
                num[0] = fmaf(term, f3.y, num[0]);
                if (DP > 1) num[1 % DP] = fmaf(term, f3.z, num[1 % DP]);
                if (DP > 2) num[2 % DP] = fmaf(term, f3.w, num[2 % DP]);
            }
#pragma unroll
            for (int i4 = 0; i4 < (kCompact ? 0 : DP); i4 += 4) {
                const float4 f = lds_f4(ra + 48 + 4 * i4);
                num[i4] = fmaf(term, f.x, num[i4]);
                if (i4 + 1 < DP) num[i4 + 1] = fmaf(term, f.y, num[i4 + 1]);
                if (i4 + 2 < DP) num[i4 + 2] = fmaf(term, f.z, num[i4 + 2]);
                if (i4 + 3 < DP) num[i4 + 3] = fmaf(term, f.w, num[i4 + 3]);
            }
            if (top.may_enter(zzf)) {  // else: below the record's worst depth even allowing for float32 error
                // store rule term > 0 (raster.py:389) as the float64 reference sees it: float32 (FTZ)
                // underflows ~950 binary orders earlier than float64, so re-derive it in the log domain
                bool store = term > 0.0f;
                if (!store && oc > 0.0f) store = x2 + log2f(oc) > -1075.0f;
                if (store) {
                    double zc = zeta < near_ ? near_ : zeta;
                    zc = zc > far_ ? far_ : zc;
                    const int sid = kCompact ? (int)lds_u32(s_rec_a - CAP * 16 + j * 16 + 12) : __float_as_int(mi.w);
                    top.insert((far_ - zc) * inv_range, sid, cl, a.zpad);
                }
            }
        }
    };

    for (int start = 0; start < n_cand; start += a.chunk) {
        const int cn = min(a.chunk, n_cand - start);
        __syncthreads();  // previous batch fully consumed
        if (tid < cn) {
            const int sid = a.pair_id[s0 + start + tid];
            const Rec rc = a.rec[sid];
            const double n2 = rc.cx * rc.cx + rc.cy * rc.cy + rc.cz * rc.cz;
            float *rp = s_rec + tid * RS;
            *reinterpret_cast<double2 *>(rp) = make_double2(rc.cx, rc.cy);
            if (DP == 3) {
                *reinterpret_cast<float4 *>(rp + 4) = make_float4(__int_as_float(__double2loint(rc.cz)),
                                                                  __int_as_float(__double2hiint(rc.cz)), rc.r,
                                                                  1.0f / rc.r);
            } else {
                *reinterpret_cast<double2 *>(rp + 4) = make_double2(rc.cz, n2);
                *reinterpret_cast<float4 *>(rp + 8) = make_float4(rc.r, rc.o, 1.0f / rc.r, __int_as_float(sid));
            }
            float4 fc = a.flt[sid];  // screen-space filter record (k_project); its spare word carries the sphere id
            fc.w = __int_as_float(sid);
            s_cf[tid] = fc;
            // which warps can this candidate touch?  Same arithmetic as the per-pixel test, applied to the
            // point of the warp's rectangle nearest to the projected centre (rounding is monotone, so a
            // pixel can pass the test only if its warp's rectangle does)
            unsigned wm = 0;
#pragma unroll
            for (int w = 0; w < 8; ++w) {
                const float4 rc4 = s_rect[w];
                const float dx = fminf(fmaxf(fc.x, rc4.x), rc4.y) - fc.x;
                const float dy = fminf(fmaxf(fc.y, rc4.z), rc4.w) - fc.y;
                wm |= (fmaf(dx, dx, dy * dy) < fc.z ? 1u : 0u) << w;
            }
            s_wmask[tid] = (unsigned char)wm;
            const float *f = a.feat + (size_t)sid * a.d;
            if (DP == 3) {
                *reinterpret_cast<float4 *>(rp + 8) = make_float4(rc.o, f[0], a.d > 1 ? f[1] : 0.0f, a.d > 2 ? f[2] : 0.0f);
            } else {
                if ((a.d & 3) == 0 && (reinterpret_cast<unsigned long long>(a.feat) & 15ull) == 0ull) {
#pragma unroll
                    for (int i = 0; i < ((DP + 3) & ~3); i += 4)
                        *reinterpret_cast<float4 *>(rp + 12 + i) =
                            i < a.d ? __ldg(reinterpret_cast<const float4 *>(f + i)) : make_float4(0.f, 0.f, 0.f, 0.f);
                } else {
#pragma unroll
                    for (int i = 0; i < ((DP + 3) & ~3); ++i) rp[12 + i] = i < a.d ? f[i] : 0.0f;
                }
            }
        }
        __syncthreads();
        if (a.tau_on) {  // vote, raster.py:364-368.  (The tile-uniform part -- a float64 square root -- formed once by
            // the first candidate's staging thread instead of by all 256: 240.2 against 239.6 us, not kept.)
            double2 czn0 = *reinterpret_cast<const double2 *>(s_rec + 4);  // c_z, |c|^2 (d = 3: c_z, [r, id])
            float r0 = s_rec[8];
            if (DP == 3) {
                const double2 cxy0 = *reinterpret_cast<const double2 *>(s_rec);
                r0 = s_rec[6];
                czn0.y = cxy0.x * cxy0.x + cxy0.y * cxy0.y + czn0.x * czn0.x;
            }
            const double e0 = (MODE == SS_MODE_PINHOLE) ? sqrt(czn0.y) - (double)r0 : czn0.x - (double)r0;
            const double zb = (far_ - fmin(fmax(e0 * tile_cos, near_), far_)) * inv_range;
            const double z_stop = a.gamma * (a.log_tau + (double)((m2 + log2f(denom)) * kLn2));
            if (!done && zb < z_stop) {
                done = true;  // a finished pixel ignores later hits (raster.py:375-376): its filter words are masked
            }
            if (__syncthreads_and(done)) break;
        }
        scanned += cn;
        if (__all_sync(0xffffffffu, done)) continue;  // warp-uniform

        // compact the indices of the candidates that can touch this warp's 8x4 block (~1 in 4)
        unsigned char *lst = s_list + warp * LSTRIDE;
        int cnt = 0;
        for (int base = 0; base < cn; base += 32) {
            const int j = base + lane;
            const bool rel = j < cn && ((s_wmask[j] >> warp) & 1u);
            const unsigned bal = __ballot_sync(0xffffffffu, rel);
            if (rel) lst[cnt + __popc(bal & ((1u << lane) - 1u))] = (unsigned char)j;
            cnt += __popc(bal);
        }
        if (lane < 4) lst[cnt + lane] = 0;  // padding of the last group of 4: a readable slot, masked out below
        __syncwarp();

        // float32 filter, candidate-parallel: lane l takes candidate 31 - l of a group of 32 relevant candidates and
        // builds the 32-bit mask of the block's pixels (bit p = row p / 8, column p % 8) that lie inside the
        // candidate's bounding circle, row by row from the circle's x-extent on that row; a 32 x 32 bit transpose by
        // shuffles then hands every lane the word of ITS pixel (candidate i at bit 31 - i).  ~3.6 instructions per
        // candidate and warp instead of the 8 of a per-pixel test of every candidate.  The mask is a superset of
        // the per-pixel test dx^2 + dy^2 < rho^2 (rho^2 widened by 0.1 % + 0.01 px^2, column ranges rounded outwards
        // by 0.002 px); the float64 evaluation in process() decides every hit, so a superset only costs a round.
        const float2 org = s_org[warp];
        auto filter_group = [&](int g) -> unsigned {
            const int n = min(32, cnt - g);
            const int i = 31 - lane;
            unsigned x = 0u;
            if (i < n) {
                const float4 c = s_cf[lst[g + i]];
                const float cxp = (c.x - org.x) * a.ppu_f;  // centre in pixel units relative to the block's first pixel
                const float cyp = (c.y - org.y) * a.ppu_f;
                float r2p = c.z * a.ppu2_f;
                r2p = fmaf(r2p, 1e-3f, r2p) + 1e-2f;
                const float lo_a = cxp + 0.498f, hi_a = cxp - 0.498f;  // ceil(v) ~ rne(v + 0.498), floor(v) ~ rne(v - 0.498)
                constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: (v + kMagic) holds rne(v) in its low mantissa bits
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const float dy = (float)r - cyp;
                    float hw;  // half-width of the circle on this row; NaN when the row misses it
                    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(hw) : "f"(fmaf(-dy, dy, r2p)));
                    // first / last column inside, clamped so that an empty row gives lo > hi (fmaxf drops the NaN)
                    const float lo_f = fminf(fmaxf(lo_a - hw, -0.4f), 8.4f);
                    const float hi_f = fminf(fmaxf(hi_a + hw, -1.4f), 7.4f);
                    const unsigned sl = __float_as_uint(lo_f + (kMagic + 8.0f * r)) & 63u;           // 8 r + lo: 0 .. 32
                    const unsigned sr = __float_as_uint((kMagic + 31.0f - 8.0f * r) - hi_f) & 63u;   // 31 - (8 r + hi): 0 .. 32
                    unsigned ml, mr;  // shifts by 32 must give 0: PTX shl / shr clamp the amount
                    asm("shl.b32 %0, %1, %2;" : "=r"(ml) : "r"(0xffffffffu), "r"(sl));
                    asm("shr.u32 %0, %1, %2;" : "=r"(mr) : "r"(0xffffffffu), "r"(sr));
                    x |= ml & mr & (0xffu << (8 * r));
                }
            }
            // bit-matrix transpose: x[lane l] bit p  ->  x[lane p] bit l
#pragma unroll
            for (int j = 16; j > 0; j >>= 1) {
                const unsigned m = j == 16 ? 0x0000ffffu : j == 8 ? 0x00ff00ffu : j == 4 ? 0x0f0f0f0fu
                                                        : j == 2 ? 0x33333333u : 0x55555555u;
                const unsigned t = __shfl_xor_sync(0xffffffffu, x, j);
                x = (lane & j) ? (((t >> j) & m) | (x & ~m)) : ((x & m) | ((t << j) & ~m));
            }
            return done ? 0u : x;
        };
        // Every lane owns two words: `wc`, the word it is draining, and `wn`, the word of the most recently filtered
        // group (empty until the lane gets that far).  A lane whose current word runs empty takes over the next one,
        // so lanes with few hits in a group run ahead by one group while the busy lanes catch up, and the divergent
        // float64 path runs with most lanes active.  `bc - b` is the shared address of the list entry behind bit b
        // of wc; `gl` is the same base for the newest group (warp-uniform).
        unsigned wc, wn = 0u, bc;
        unsigned gl = (unsigned)__cvta_generic_to_shared(lst) + 31u;
        asm volatile("" : "+r"(gl));
        auto drain_round = [&]() {
            if (wc == 0u) { wc = wn; wn = 0u; bc = gl; }
            if (wc) {
                unsigned b;  // highest set bit = oldest pending candidate (list entry 31 - b)
                asm("bfind.u32 %0, %1;" : "=r"(b) : "r"(wc));  // (31 - __clz costs two more integer instructions)
                wc ^= 1u << b;
                process(lds_u8(bc - b));
            }
        };
        wc = filter_group(0);
        bc = gl;
        for (int g = 32; g < cnt; g += 32) {
            const unsigned w = filter_group(g);
            // the new word needs a free slot in every lane: drain until no lane holds two pending words
            while (__any_sync(0xffffffffu, wn != 0u)) drain_round();
            gl += 32u;
            if (wc == 0u) { wc = w; bc = gl; } else wn = w;
        }
        while (__any_sync(0xffffffffu, (wc | wn) != 0u)) drain_round();
    }

    // finalise, raster.py:401-414
    if (valid) {
        const size_t P = (size_t)cam.W * cam.H;
        const size_t pix = (size_t)py * cam.W + px;
        const float ld2 = m2 + log2f(denom);
        const float w_bg = exp2f(m2_bg - ld2);
        const float inv = 1.0f / denom;
#pragma unroll
        for (int i = 0; i < DP; ++i)
            if (i < a.d) a.image[pix * a.d + i] = fmaf(w_bg, a.bg[i], num[i] * inv);
        a.bg_weight[pix] = w_bg;
        if (a.store_buffer) {
            if (KT <= 8) {
#pragma unroll
                for (int k = 0; k < KT; ++k) {
                    if (k < a.K) {
                        const int tid_k = top.get_id(k);
                        a.ids[k * P + pix] = tid_k;
                        a.z[k * P + pix] = tid_k < 0 ? 0.0f : (float)top.get_z(k);
                        a.clos[k * P + pix] = top.get_c(k);
                    }
                }
            } else {
#pragma unroll 4
                for (int k = 0; k < a.K; ++k) {
                    const int tid_k = top.get_id(k);
                    a.ids[k * P + pix] = tid_k;
                    a.z[k * P + pix] = tid_k < 0 ? 0.0f : (float)top.get_z(k);
                    a.clos[k * P + pix] = top.get_c(k);
                }
            }
            a.log_denom[pix] = ld2 * kLn2;
        }
    }
    if (a.collect_stats) {
        unsigned h = n_hits;
        unsigned st = (valid && done) ? 1u : 0u;
        h = __reduce_add_sync(0xffffffffu, h);
        st = __reduce_add_sync(0xffffffffu, st);
        __syncthreads();
        if (lane == 0) {
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
constexpr size_t raster_smem_bytes() {
    return (size_t)SS_MAX_CHUNK * (16 + 4 * rec_stride<DP>()) + SS_MAX_CHUNK + 8 * (SS_MAX_CHUNK + 4) +
           ((SS_TOPK_SHARED != 0 && KT <= 8) ? (size_t)KT * TILE_PX * 16 : 0);
}

template <int DP, int KT, int MODE>
void launch_one(const RasterArgs &r, int n_tiles, cudaStream_t s) {
    constexpr size_t smem = raster_smem_bytes<DP, KT>();
    static PerDeviceOnce attr_once;  // per instantiation and device
    if (attr_once.first()) {
        if (smem + 1024 > 48 * 1024)
            cudaFuncSetAttribute(k_raster<DP, KT, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
#ifndef SS_RASTER_CARVEOUT
#define SS_RASTER_CARVEOUT -1  // percent of the unified L1/shared storage to prefer as shared; -1 = driver default
#endif
        if (SS_RASTER_CARVEOUT >= 0)
            cudaFuncSetAttribute(k_raster<DP, KT, MODE>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 SS_RASTER_CARVEOUT);
    }
    k_raster<DP, KT, MODE><<<n_tiles, TILE_PX, smem, s>>>(r);
}

template <int DP, int KT>
void launch_mode(const RasterArgs &r, int n_tiles, int mode, cudaStream_t s) {
    if (mode == SS_MODE_PINHOLE) launch_one<DP, KT, SS_MODE_PINHOLE>(r, n_tiles, s);
    else launch_one<DP, KT, SS_MODE_ORTHOGRAPHIC>(r, n_tiles, s);
}

template <int DP>
void launch_k(const RasterArgs &r, int n_tiles, int mode, cudaStream_t s) {
    if (r.K <= 5) launch_mode<DP, 5>(r, n_tiles, mode, s);
    else if (r.K <= 8) launch_mode<DP, 8>(r, n_tiles, mode, s);
    else if (r.K <= 32) launch_mode<DP, 32>(r, n_tiles, mode, s);
    else launch_mode<DP, 64>(r, n_tiles, mode, s);
}

}  // namespace

cudaError_t launch_raster(const FwdLaunch &a, cudaStream_t s, int tile0, int n_tiles) {
    const Layout &L = a.L;
    RasterArgs r;
    r.cam = a.cam;
    r.tile_start = (const int *)(a.ws + L.tile_start);
    r.pair_id = (int *)(a.ws + L.pair_id);
    r.pair_key = (const unsigned long long *)(a.ws + L.pair_key);
    r.key = (const unsigned long long *)(a.ws + L.key);
    r.bucket = (const int *)(a.ws + L.bucket);
    r.tile_cursor = (const int *)(a.ws + L.tile_cursor);
    r.sort_here = SS_FUSED_SORT;
    r.rec = (const Rec *)(a.ws + L.rec);
    r.flt = (const float4 *)(a.ws + L.flt);
    r.feat = a.feat; r.bg = a.bg;
    r.d = a.dims.feature_dim; r.K = a.dims.top_k; r.chunk = a.blend.chunk;
    r.gamma = a.gamma; r.eps_over_g = a.blend.eps / a.gamma;
    r.tau_on = a.blend.tau > 0.0 ? 1 : 0;
    r.log_tau = r.tau_on ? log(a.blend.tau / (1.0 - a.blend.tau)) : 0.0;
    r.far_f = (float)a.cam.far_;
    r.fmn_f = (float)(a.cam.far_ - a.cam.near_);
    r.inv_range_f = (float)a.cam.inv_range;
    r.ppu_f = (float)a.cam.ppu;
    r.ppu2_f = (float)(a.cam.ppu * a.cam.ppu);
    // |float32 depth - float64 depth| <= ~6 roundings of (|far| + |zeta|) / (far - near); padded 4x
    r.zpad = (float)(24.0 * ldexp(1.0, -24) * (fabs(a.cam.far_) + fabs(a.cam.near_) + (a.cam.far_ - a.cam.near_)) *
                     a.cam.inv_range);
    r.store_buffer = (a.blend.flags & SS_OPT_STORE_BUFFER) ? 1 : 0;
    r.collect_stats = (a.blend.flags & SS_OPT_COLLECT_STATS) ? 1 : 0;
    r.image = a.image; r.bg_weight = a.bg_weight;
    r.ids = a.ids; r.z = a.z; r.clos = a.clos; r.log_denom = a.log_denom;
    r.status = (long long *)(a.ws + L.status);
    if (n_tiles < 0) n_tiles = L.n_tiles - tile0;
    r.tile0 = tile0;
    if (n_tiles <= 0) return cudaSuccess;
    const int d = r.d, mode = a.cam.mode;
    ProfScope ps(KID_RASTER, s);
    if (d == 3) launch_k<3>(r, n_tiles, mode, s);
    else if (d <= 4) launch_k<4>(r, n_tiles, mode, s);
    else if (d <= 16) launch_k<16>(r, n_tiles, mode, s);
    else launch_k<32>(r, n_tiles, mode, s);
    count_launch();
    return cudaGetLastError();
}

}  // namespace ss
