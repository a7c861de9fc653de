// Shared device/host declarations for the sm_100a sphere-render kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/softsphere_b200.h"

namespace ss {

// Camera-frame draw record of one sphere (DrawRecords, reference raster.py:58-76), packed
// into one 32-byte sector: centre in float64 (decides hits / depth order exactly like the
// float64 reference), radius and CLAMPED opacity in float32 (exact: inputs are float32).
struct __align__(32) Rec {
    double cx, cy, cz;
    float r;
    float o;
};
static_assert(sizeof(Rec) == 32, "Rec must be one 32-byte sector");

// Camera + derived constants handed to kernels by value.
struct Cam {
    double t[3];
    double R[9];
    double focal, sensor_w, near_, far_;
    double ppu;        // W / sensor_w (pixels per metric unit)
    double pix;        // sensor_w / W
    double inv_range;  // 1 / (far - near)
    double inv_f_ppu;  // 1 / (focal * ppu)
    int W, H, mode;
    int ntx, nty;
};

// Workspace layout (byte offsets, 256-byte aligned).
struct Layout {
    size_t status;       // 16 x int64 (SsStatus)
    size_t tile_count;   // n_tiles + 1 int32 (zeroed with status at forward start): spheres touching <= 4 tiles;
                         // after k_scan: the emit cursor of the fallback path
    size_t tile_count_big;  // n_tiles + 1 int32 (zeroed too): spheres touching > 4 tiles
    size_t tile_start;   // n_tiles + 1 int32
    size_t tile_cursor;  // n_tiles int32
    size_t big_tiles;    // n_tiles + 1 int32: [0] = count, then tile ids with > SORT_SMALL pairs
    size_t rec;          // M Rec
    size_t key;          // M uint64 (order-preserving bits of earliest)
    size_t trect;        // M ushort4 tile rects (tx0, tx1, ty0, ty1); tx0 > tx1 = off sensor
    size_t proj_r;       // M double
    size_t flt;          // M float4: screen-space filter (projected centre x, y, padded rho^2, -)
    size_t bucket;       // n_tiles x BUCKET_CAP int32: sphere ids written straight into their tile by k_project
    size_t pair_key;     // max_pairs uint64
    size_t pair_id;      // max_pairs int32
    size_t raw;          // M * raw_stride float (backward accumulators)
    size_t cam_part;     // CAM_BLOCKS_MAX * 16 double + counter
    size_t total;
    int n_tiles, ntx, nty, raw_stride;
};

#ifndef SS_FUSED_SORT
#define SS_FUSED_SORT 0  // lists of <= 512 pairs sorted by k_tile_sort_small (0) or by k_raster itself (1: measured, no gain)
#endif

constexpr int TILE = SS_TILE;
constexpr int TILE_PX = TILE * TILE;
constexpr int SORT_SMALL = 512;   // per-tile lists up to this length: k_tile_sort_small (one CTA per tile, registers + 8 KB smem)
constexpr int SORT_BIG = 8192;    // up to this length in 96 KB dynamic smem; beyond: in global memory
constexpr int BUCKET_CAP = 4096;  // sphere ids per tile bucket; a fuller tile switches the frame to the emit path
constexpr int CAM_BLOCKS_MAX = 1024;
constexpr int CAM_VALS = 16;  // sum sc (3), G (9), focal, sensor, 2 pad

__host__ __device__ inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

inline int raw_stride_for(int d) { return 8 + ((d + 3) & ~3); }

inline Layout make_layout(const SsDims &dm) {
    Layout L;
    L.ntx = (dm.width + TILE - 1) / TILE;
    L.nty = (dm.height + TILE - 1) / TILE;
    L.n_tiles = L.ntx * L.nty;
    L.raw_stride = raw_stride_for(dm.feature_dim);
    size_t M = (size_t)(dm.num_spheres > 0 ? dm.num_spheres : 1);
    size_t P = (size_t)(dm.max_pairs > 0 ? dm.max_pairs : 1);
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off = align256(off + bytes); return o; };
    L.status = take(16 * sizeof(int64_t));
    L.tile_count = take((size_t)(L.n_tiles + 1) * 4);
    L.tile_count_big = take((size_t)(L.n_tiles + 1) * 4);
    L.tile_start = take((size_t)(L.n_tiles + 1) * 4);
    L.tile_cursor = take((size_t)L.n_tiles * 4);
    L.big_tiles = take((size_t)(L.n_tiles + 1) * 4);
    L.rec = take(M * sizeof(Rec));
    L.key = take(M * 8);
    L.trect = take(M * 8);
    L.proj_r = take(M * 8);
    L.flt = take(M * 16);
    L.bucket = take((size_t)L.n_tiles * BUCKET_CAP * 4);
    L.pair_key = take(P * 8);
    L.pair_id = take(P * 4);
    L.raw = take(M * (size_t)L.raw_stride * 4);
    L.cam_part = take((size_t)(CAM_BLOCKS_MAX * CAM_VALS + 2) * 8);
    L.total = off;
    return L;
}

inline Cam make_cam(const SsCamera &c) {
    Cam k;
    for (int i = 0; i < 3; ++i) k.t[i] = c.t[i];
    for (int i = 0; i < 9; ++i) k.R[i] = c.R[i];
    k.focal = c.focal; k.sensor_w = c.sensor_w; k.near_ = c.near_; k.far_ = c.far_;
    k.ppu = (double)c.width / c.sensor_w;
    k.pix = c.sensor_w / (double)c.width;
    k.inv_range = 1.0 / (c.far_ - c.near_);
    k.inv_f_ppu = 1.0 / (c.focal * k.ppu);
    k.W = c.width; k.H = c.height; k.mode = c.mode;
    k.ntx = (c.width + TILE - 1) / TILE;
    k.nty = (c.height + TILE - 1) / TILE;
    return k;
}

// Status slots (int64 each) -- mirrors SsStatus.
enum { ST_FLAGS = 0, ST_ON_SENSOR = 1, ST_PAIRS = 2, ST_TESTED = 3, ST_HITS = 4, ST_STOPPED = 5,
       ST_FIRST_INVALID = 6 };

// Host-side launchers (one per translation unit).
struct FwdLaunch {
    SsDims dims; Cam cam; SsBlend blend; double gamma;
    const float *pos, *rad, *opa, *feat, *bg;
    char *ws; Layout L;
    float *image, *bg_weight; int32_t *ids; float *z, *clos, *log_denom;
    int32_t *rect; uint8_t *on_sensor; double *earliest, *proj_r_out;
};
struct BwdLaunch {
    SsDims dims; Cam cam; SsBlend blend; double gamma;
    const float *pos, *rad, *opa, *feat, *bg;
    char *ws; Layout L;
    const int32_t *ids; const float *z, *clos, *log_denom, *upstream;
    float *d_pos, *d_rad, *d_opa, *d_feat; int32_t *pixel_count; double *cam_grad;
    char *det_ws;  // SS_OPT_DETERMINISTIC scratch (DetLayout) or nullptr
};

// Scratch of the deterministic backward: per-sphere float bits of max |addend| (first pass), then the 64-bit
// fixed-point accumulator rows (same AoS layout as the float rows).
struct DetLayout {
    size_t max_bits;  // M uint32
    size_t raw64;     // M * raw_stride int64
    size_t total;
};
inline DetLayout make_det_layout(const SsDims &dm) {
    DetLayout D;
    const size_t M = (size_t)(dm.num_spheres > 0 ? dm.num_spheres : 1);
    D.max_bits = 0;
    D.raw64 = align256(M * 4);
    D.total = D.raw64 + align256(M * (size_t)raw_stride_for(dm.feature_dim) * 8);
    return D;
}

cudaError_t launch_project(const FwdLaunch &a, bool records_only, cudaStream_t s);
cudaError_t launch_binning(const FwdLaunch &a, cudaStream_t s);
// draws tiles [tile0, tile0 + n_tiles) (n_tiles < 0: to the last tile)
cudaError_t launch_raster(const FwdLaunch &a, cudaStream_t s, int tile0 = 0, int n_tiles = -1);
// One of this thread's two library-owned side streams (used alternately) with its fork / join events, created on
// first use; false if they could not be created (callers then stay on their own stream).
bool side_stream(cudaStream_t *side, cudaEvent_t *fork, cudaEvent_t *join);
cudaError_t launch_backward(const BwdLaunch &a, cudaStream_t s);

void count_launch(int n = 1);

// Function attributes (dynamic shared memory size, carve-out) are per DEVICE: a process that drives several GPUs
// must set them once on each.  One flag array per call site; returns true the first time the calling thread's
// current device is seen (a benign race sets the attribute twice).
struct PerDeviceOnce {
    bool done[64] = {};
    bool first() {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return true;
        if (done[dev]) return false;
        done[dev] = true;
        return true;
    }
};

// Optional per-kernel CUDA-event timing (ss_profile_*): used by bench.py for the roofline line.
enum KernelId { KID_PROJECT = 0, KID_SCAN, KID_EMIT, KID_SORT_SMALL, KID_SORT_BIG, KID_RASTER, KID_BACKWARD,
                KID_FINALIZE, KID_MEMSET_FWD, KID_MEMSET_BWD, KID_COUNT };
void prof_begin(int kid, cudaStream_t s);
void prof_end(int kid, cudaStream_t s);
struct ProfScope {
    int kid; cudaStream_t s;
    ProfScope(int k, cudaStream_t st) : kid(k), s(st) { prof_begin(kid, s); }
    ~ProfScope() { prof_end(kid, s); }
};

}  // namespace ss
