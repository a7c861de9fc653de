// what changes the sphere set between steps and the on-disk record format,
// on the device (reference softsphere/optim.py and softsphere/scene.py):
//
//   k_prune_flags    prune's keep mask (optim.py:161-183): clip(opacity, 0, 1) >= opacity_min, optional
//                    |feature - background| >= background_dist, visibility > 0 -- float64 comparisons on the
//                    float32 columns, like the reference's float64 arrays of the same values.
//   k_compact_count / k_compact_scan / k_compact_rows
//                    stable stream compaction of any set of per-sphere columns (parameters, Adam moments,
//                    visibility) by that mask: per-block counts, one single-CTA scan, one scatter pass that
//                    moves every column in the same launch.  scene.positions[keep] etc. (optim.py:176-181),
//                    states[name].take(keep) (optim.py:351-352).
//   k_subdivide      FCC x12 subdivision (optim.py:186-213): children at parent + r/sqrt(2) * dir, radius
//                    scale * r, opacity and features inherited; child c of parent p at row 12 p + c.
//   k_psc1_unpack / k_psc1_pack
//                    PSC1 record block <-> SoA columns (scene.py:179-227): records are (5 + d) little-endian
//                    float32 per sphere (position*3, radius, opacity, feature*d).  Staged through shared memory
//                    so that both the AoS side and the SoA side move as full sectors.
//   k_cvt_*          float64 <-> float32 blobs of the PSK1 checkpoint (Adam moments are stored as <f8,
//                    optim.py:397-405).
// All of these are pure HBM-bound byte movers; algorithmic bytes are stated at each launcher.
#include <math.h>

#include "ss_common.cuh"

namespace ss {

namespace {

constexpr int CB = 256;  // spheres per compaction block

// T = float: the device-resident float32 columns; T = double: the reference-signature wrapper's float64 host
// columns (an opacity exactly at the threshold must not flip by float32 rounding, optim.py:169-175)
template <typename T>
__global__ void __launch_bounds__(CB) k_prune_flags(const T *__restrict__ opa, const T *__restrict__ feat,
                                                    const T *__restrict__ bg,
                                                    const int *__restrict__ visibility, long long M, int d,
                                                    double opacity_min, double background_dist,
                                                    unsigned char *keep) {
    const long long i = (long long)blockIdx.x * CB + threadIdx.x;
    if (i >= M) return;
    const double o = fmin(fmax((double)opa[i], 0.0), 1.0);
    bool k = o >= opacity_min;
    if (background_dist > 0.0) {
        double s = 0.0;
        for (int c = 0; c < d; ++c) {
            const double df = (double)feat[(size_t)i * d + c] - (double)bg[c];
            s += df * df;
        }
        k = k && (sqrt(s) >= background_dist);
    }
    if (visibility) k = k && visibility[i] > 0;
    keep[i] = k ? 1 : 0;
}

__global__ void __launch_bounds__(CB) k_compact_count(const unsigned char *__restrict__ keep, long long M,
                                                      int *block_count) {
    const long long i = (long long)blockIdx.x * CB + threadIdx.x;
    const int k = (i < M && keep[i]) ? 1 : 0;
    const int n = __syncthreads_count(k);
    if (threadIdx.x == 0) block_count[blockIdx.x] = n;
}

// exclusive scan of the per-block counts (in place) + total; one CTA, 1024 counts per pass
__global__ void __launch_bounds__(1024) k_compact_scan(int *block_count, int n_blocks, long long *total_out) {
    __shared__ long long warp_sums[32];
    __shared__ long long carry_s;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) carry_s = 0;
    __syncthreads();
    for (int base = 0; base < n_blocks; base += 1024) {
        const int i = base + tid;
        const int c = i < n_blocks ? block_count[i] : 0;
        long long v = c;
        for (int o = 1; o < 32; o <<= 1) {
            const long long n = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += n;
        }
        if (lane == 31) warp_sums[wid] = v;
        __syncthreads();
        if (wid == 0) {
            long long w = warp_sums[lane];
            for (int o = 1; o < 32; o <<= 1) {
                const long long n = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += n;
            }
            warp_sums[lane] = w;
        }
        __syncthreads();
        const long long excl = carry_s + (wid > 0 ? warp_sums[wid - 1] : 0) + v - c;
        if (i < n_blocks) block_count[i] = (int)excl;
        __syncthreads();
        if (tid == 1023) carry_s = excl + c;
        __syncthreads();
    }
    if (tid == 0) *total_out = carry_s;
}

// keep[i] = v[i] != 0 (e.g. pixel_count > 0: the spheres that received gradient)
__global__ void __launch_bounds__(256) k_mask_nonzero(const int *__restrict__ v, long long M, unsigned char *keep) {
    const long long i = (long long)blockIdx.x * 256 + threadIdx.x;
    if (i < M) keep[i] = v[i] != 0 ? 1 : 0;
}

constexpr int MAX_COLS = 16;
struct Columns {
    const unsigned *src[MAX_COLS];
    unsigned *dst[MAX_COLS];
    int words[MAX_COLS];  // 32-bit words per row
    int stride[MAX_COLS]; // 32-bit words between consecutive destination rows (= words when packed)
    int n;
};

// One thread per sphere decides its destination row (block offset + rank among the block's kept rows);
// the block then copies the kept rows of every column word by word, consecutive threads on consecutive
// destination words, so the writes of a block are one contiguous run per column.
__global__ void __launch_bounds__(CB) k_compact_rows(const unsigned char *__restrict__ keep, long long M,
                                                     const int *__restrict__ block_offset, Columns cols) {
    __shared__ int s_src[CB];  // local source row of the r-th kept row of this block
    __shared__ int s_warp[CB / 32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const long long row0 = (long long)blockIdx.x * CB;
    const long long i = row0 + tid;
    const bool k = i < M && keep[i];
    const unsigned bal = __ballot_sync(0xffffffffu, k);
    if (lane == 0) s_warp[wid] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0;
#pragma unroll
    for (int w = 0; w < CB / 32; ++w) {
        const int c = s_warp[w];
        if (w < wid) before += c;
        total += c;
    }
    if (k) s_src[before + __popc(bal & ((1u << lane) - 1u))] = tid;
    __syncthreads();
    const long long dst0 = block_offset[blockIdx.x];
    for (int c = 0; c < cols.n; ++c) {
        const int w = cols.words[c];
        const unsigned *src = cols.src[c] + (size_t)row0 * w;
        const int st = cols.stride[c];
        unsigned *dst = cols.dst[c] + (size_t)dst0 * st;
        const int n_words = total * w;
        for (int e = tid; e < n_words; e += CB) {
            const int r = e / w, j = e - r * w;
            dst[r * st + j] = src[s_src[r] * w + j];
        }
    }
}

// Columns that interleave into ONE array of records (equal destination strides, the columns tiling a record without
// gaps): the block assembles its kept rows as records in shared memory and writes them as one contiguous run, each
// warp store covering one aligned 128-byte line.  Into device memory this saves the strided partial-sector writes of
// the column-by-column pass; into MAPPED PINNED HOST memory it is what makes the pass usable as the download itself
// (full-line PCIe writes, no staging array and no separate copy: HostRenderSession's compact gradient rows).
// cols.stride[c] holds the column's word offset inside the record here; S = words per record.
__global__ void __launch_bounds__(CB) k_compact_records(const unsigned char *__restrict__ keep, long long M,
                                                        const int *__restrict__ block_offset, Columns cols,
                                                        unsigned *__restrict__ base, int S) {
    extern __shared__ unsigned s_rec[];  // CB * S words
    __shared__ int s_src[CB];
    __shared__ int s_warp[CB / 32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const long long row0 = (long long)blockIdx.x * CB;
    const long long i = row0 + tid;
    const bool k = i < M && keep[i];
    const unsigned bal = __ballot_sync(0xffffffffu, k);
    if (lane == 0) s_warp[wid] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0;
#pragma unroll
    for (int w = 0; w < CB / 32; ++w) {
        const int c = s_warp[w];
        if (w < wid) before += c;
        total += c;
    }
    if (k) s_src[before + __popc(bal & ((1u << lane) - 1u))] = tid;
    __syncthreads();
    for (int c = 0; c < cols.n; ++c) {
        const int w = cols.words[c];
        const unsigned *src = cols.src[c] + (size_t)row0 * w;
        const int off = cols.stride[c];
        const int n_words = total * w;
        for (int e = tid; e < n_words; e += CB) {
            const int r = e / w, j = e - r * w;
            s_rec[r * S + off + j] = src[s_src[r] * w + j];
        }
    }
    __syncthreads();
    unsigned *dst = base + (size_t)block_offset[blockIdx.x] * S;
    const int n = total * S;
    const int a = (int)(((size_t)dst >> 2) & 31);  // word offset of the run inside its first 128-byte line
    for (int e = tid - a; e < n; e += CB)
        if (e >= 0) dst[e] = s_rec[e];
}

__constant__ float c_fcc[12][3] = {{1, 1, 0},  {1, -1, 0}, {-1, 1, 0},  {-1, -1, 0}, {1, 0, 1},  {1, 0, -1},
                                   {-1, 0, 1}, {-1, 0, -1}, {0, 1, 1},  {0, 1, -1},  {0, -1, 1}, {0, -1, -1}};

// one thread per child (T = double: float64 columns of the reference-signature wrapper, children exact in float64)
template <typename T>
__global__ void __launch_bounds__(256) k_subdivide(const T *__restrict__ pos, const T *__restrict__ rad,
                                                   const T *__restrict__ opa, const T *__restrict__ feat,
                                                   long long M, int d, double scale, T *pos_o, T *rad_o,
                                                   T *opa_o, T *feat_o) {
    const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= M * 12) return;
    const long long p = c / 12;
    const int k = (int)(c - p * 12);
    const double r = (double)rad[p];
    const double a = r / sqrt(2.0);
    pos_o[3 * c] = (T)((double)pos[3 * p] + a * (double)c_fcc[k][0]);
    pos_o[3 * c + 1] = (T)((double)pos[3 * p + 1] + a * (double)c_fcc[k][1]);
    pos_o[3 * c + 2] = (T)((double)pos[3 * p + 2] + a * (double)c_fcc[k][2]);
    rad_o[c] = (T)(r * scale);
    opa_o[c] = opa[p];
    for (int j = 0; j < d; ++j) feat_o[(size_t)c * d + j] = feat[(size_t)p * d + j];
}

constexpr int PB = 128;  // spheres per PSC1 block; (5 + 32) * 128 * 4 = 18.5 KB of shared memory at most

template <bool UNPACK>
__global__ void __launch_bounds__(PB) k_psc1(float *rec, long long M, int d, float *pos, float *rad, float *opa,
                                             float *feat) {
    extern __shared__ float s_rows[];
    const int w = 5 + d;
    const long long row0 = (long long)blockIdx.x * PB;
    const int rows = (int)min((long long)PB, M - row0);
    const int n = rows * w;
    float *g = rec + (size_t)row0 * w;
    if (UNPACK) {
        for (int e = threadIdx.x; e < n; e += PB) s_rows[e] = g[e];
        __syncthreads();
        for (int e = threadIdx.x; e < rows * 3; e += PB) pos[(size_t)row0 * 3 + e] = s_rows[(e / 3) * w + e % 3];
        for (int e = threadIdx.x; e < rows; e += PB) {
            rad[row0 + e] = s_rows[e * w + 3];
            opa[row0 + e] = s_rows[e * w + 4];
        }
        for (int e = threadIdx.x; e < rows * d; e += PB) feat[(size_t)row0 * d + e] = s_rows[(e / d) * w + 5 + e % d];
    } else {
        for (int e = threadIdx.x; e < rows * 3; e += PB) s_rows[(e / 3) * w + e % 3] = pos[(size_t)row0 * 3 + e];
        for (int e = threadIdx.x; e < rows; e += PB) {
            s_rows[e * w + 3] = rad[row0 + e];
            s_rows[e * w + 4] = opa[row0 + e];
        }
        for (int e = threadIdx.x; e < rows * d; e += PB) s_rows[(e / d) * w + 5 + e % d] = feat[(size_t)row0 * d + e];
        __syncthreads();
        for (int e = threadIdx.x; e < n; e += PB) g[e] = s_rows[e];
    }
}

__global__ void __launch_bounds__(256) k_cvt_f64_f32(const double *__restrict__ in, float *out, long long n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (float)in[i];
}
__global__ void __launch_bounds__(256) k_cvt_f32_f64(const float *__restrict__ in, double *out, long long n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = (double)in[i];
}

inline int rc_of(cudaError_t e) { return e == cudaSuccess ? SS_OK : SS_ERR_CUDA; }

}  // namespace

}  // namespace ss

using namespace ss;

extern "C" {

// bytes moved: M (4 + 4 d [+ 4]) read, M written
int ss_prune_mask(const float *opa, const float *feat, const float *bg, const int32_t *visibility, int64_t M,
                  int32_t d, double opacity_min, double background_dist, uint8_t *keep, void *stream) {
    if (M < 0 || d < 1 || d > SS_MAX_FEATURE_DIM) return SS_ERR_DIMS;
    if (M == 0) return SS_OK;
    if (!opa || !keep || (background_dist > 0.0 && (!feat || !bg))) return SS_ERR_NULL;
    k_prune_flags<float><<<(unsigned)((M + CB - 1) / CB), CB, 0, (cudaStream_t)stream>>>(
        opa, feat, bg, visibility, M, d, opacity_min, background_dist, keep);
    count_launch();
    return rc_of(cudaGetLastError());
}

int ss_prune_mask_f64(const double *opa, const double *feat, const double *bg, const int32_t *visibility, int64_t M,
                      int32_t d, double opacity_min, double background_dist, uint8_t *keep, void *stream) {
    if (M < 0 || d < 1 || d > SS_MAX_FEATURE_DIM) return SS_ERR_DIMS;
    if (M == 0) return SS_OK;
    if (!opa || !keep || (background_dist > 0.0 && (!feat || !bg))) return SS_ERR_NULL;
    k_prune_flags<double><<<(unsigned)((M + CB - 1) / CB), CB, 0, (cudaStream_t)stream>>>(
        opa, feat, bg, visibility, M, d, opacity_min, background_dist, keep);
    count_launch();
    return rc_of(cudaGetLastError());
}

int ss_mask_nonzero_i32(const int32_t *values, int64_t M, uint8_t *keep, void *stream) {
    if (M < 0) return SS_ERR_DIMS;
    if (M == 0) return SS_OK;
    if (!values || !keep) return SS_ERR_NULL;
    k_mask_nonzero<<<(unsigned)((M + 255) / 256), 256, 0, (cudaStream_t)stream>>>(values, M, keep);
    count_launch();
    return rc_of(cudaGetLastError());
}

int ss_compact_workspace_bytes(int64_t M, size_t *out_bytes) {
    if (M < 0 || !out_bytes) return SS_ERR_DIMS;
    *out_bytes = align256((size_t)((M + CB - 1) / CB + 1) * sizeof(int));
    return SS_OK;
}

// bytes moved: M (keep) + per column kept_rows * row_bytes read and written
int ss_compact_rows(const uint8_t *keep, int64_t M, const SsColumn *cols, int32_t n_cols, void *workspace,
                    size_t workspace_bytes, int64_t *count_out, void *stream) {
    if (M < 0 || n_cols < 0 || n_cols > MAX_COLS) return SS_ERR_DIMS;
    if (!count_out) return SS_ERR_NULL;
    cudaStream_t s = (cudaStream_t)stream;
    if (M == 0) return rc_of(cudaMemsetAsync(count_out, 0, sizeof(int64_t), s));
    if (!keep || !workspace || (n_cols > 0 && !cols)) return SS_ERR_NULL;
    size_t need;
    ss_compact_workspace_bytes(M, &need);
    if (workspace_bytes < need) return SS_ERR_WORKSPACE;
    Columns c;
    c.n = n_cols;
    for (int i = 0; i < n_cols; ++i) {
        if (!cols[i].src || !cols[i].dst) return SS_ERR_NULL;
        if (cols[i].row_bytes <= 0 || cols[i].row_bytes % 4 != 0) return SS_ERR_DIMS;
        c.src[i] = (const unsigned *)cols[i].src;
        c.dst[i] = (unsigned *)cols[i].dst;
        c.words[i] = (int)(cols[i].row_bytes / 4);
        if (cols[i].dst_stride_bytes != 0 &&
            (cols[i].dst_stride_bytes < cols[i].row_bytes || cols[i].dst_stride_bytes % 4 != 0))
            return SS_ERR_DIMS;
        c.stride[i] = cols[i].dst_stride_bytes ? (int)(cols[i].dst_stride_bytes / 4) : c.words[i];
    }
    const int n_blocks = (int)((M + CB - 1) / CB);
    int *bc = (int *)workspace;
    // interleaved destination?  (every column with the same stride S, the columns tiling [base, base + S words))
    int S = n_cols > 0 ? c.stride[0] : 0;
    unsigned *base = n_cols > 0 ? c.dst[0] : nullptr;
    bool records = n_cols > 1 && S <= 48;
    int covered = 0;
    for (int i = 0; i < n_cols && records; ++i) {
        records = c.stride[i] == S;
        if (c.dst[i] < base) base = c.dst[i];
        covered += c.words[i];
    }
    records = records && covered == S;
    if (records) {
        unsigned long long used = 0;  // S <= 48 words: one bit per word of the record
        for (int i = 0; i < n_cols && records; ++i) {
            const long long off = c.dst[i] - base;
            if (off < 0 || off + c.words[i] > S) { records = false; break; }
            const unsigned long long m = ((c.words[i] >= 64 ? 0ull : (1ull << c.words[i])) - 1ull) << off;
            if (used & m) records = false;
            used |= m;
        }
    }
    k_compact_count<<<n_blocks, CB, 0, s>>>(keep, M, bc);
    k_compact_scan<<<1, 1024, 0, s>>>(bc, n_blocks, (long long *)count_out);
    if (records) {
        Columns r = c;
        for (int i = 0; i < n_cols; ++i) r.stride[i] = (int)(c.dst[i] - base);
        k_compact_records<<<n_blocks, CB, (size_t)CB * S * sizeof(unsigned), s>>>(keep, M, bc, r, base, S);
    } else {
        k_compact_rows<<<n_blocks, CB, 0, s>>>(keep, M, bc, c);
    }
    count_launch(3);
    return rc_of(cudaGetLastError());
}

// bytes moved: M (20 + 4 d) read, 12 M (20 + 4 d) written
int ss_subdivide(const float *pos, const float *rad, const float *opa, const float *feat, int64_t M, int32_t d,
                 double scale, float *pos_out, float *rad_out, float *opa_out, float *feat_out, void *stream) {
    if (M < 0 || d < 1 || d > SS_MAX_FEATURE_DIM || M > (int64_t)1 << 40) return SS_ERR_DIMS;
    if (M == 0) return SS_OK;
    if (!pos || !rad || !opa || !feat || !pos_out || !rad_out || !opa_out || !feat_out) return SS_ERR_NULL;
    if (!(scale > 0.0)) return SS_ERR_PARAMS;
    const long long n = (long long)M * 12;
    k_subdivide<float><<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        pos, rad, opa, feat, M, d, scale, pos_out, rad_out, opa_out, feat_out);
    count_launch();
    return rc_of(cudaGetLastError());
}

int ss_subdivide_f64(const double *pos, const double *rad, const double *opa, const double *feat, int64_t M,
                     int32_t d, double scale, double *pos_out, double *rad_out, double *opa_out, double *feat_out,
                     void *stream) {
    if (M < 0 || d < 1 || d > SS_MAX_FEATURE_DIM || M > (int64_t)1 << 40) return SS_ERR_DIMS;
    if (M == 0) return SS_OK;
    if (!pos || !rad || !opa || !feat || !pos_out || !rad_out || !opa_out || !feat_out) return SS_ERR_NULL;
    if (!(scale > 0.0)) return SS_ERR_PARAMS;
    const long long n = (long long)M * 12;
    k_subdivide<double><<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        pos, rad, opa, feat, M, d, scale, pos_out, rad_out, opa_out, feat_out);
    count_launch();
    return rc_of(cudaGetLastError());
}

// bytes moved: M (20 + 4 d) read and written
int ss_psc1_unpack(const void *records, int64_t M, int32_t d, float *pos, float *rad, float *opa, float *feat,
                   void *stream) {
    if (M < 0 || d < 1 || d > SS_MAX_FEATURE_DIM) return SS_ERR_DIMS;
    if (M == 0) return SS_OK;
    if (!records || !pos || !rad || !opa || !feat) return SS_ERR_NULL;
    k_psc1<true><<<(unsigned)((M + PB - 1) / PB), PB, (size_t)PB * (5 + d) * 4, (cudaStream_t)stream>>>(
        (float *)records, M, d, pos, rad, opa, feat);
    count_launch();
    return rc_of(cudaGetLastError());
}

int ss_psc1_pack(const float *pos, const float *rad, const float *opa, const float *feat, int64_t M, int32_t d,
                 void *records_out, void *stream) {
    if (M < 0 || d < 1 || d > SS_MAX_FEATURE_DIM) return SS_ERR_DIMS;
    if (M == 0) return SS_OK;
    if (!records_out || !pos || !rad || !opa || !feat) return SS_ERR_NULL;
    k_psc1<false><<<(unsigned)((M + PB - 1) / PB), PB, (size_t)PB * (5 + d) * 4, (cudaStream_t)stream>>>(
        (float *)records_out, M, d, (float *)pos, (float *)rad, (float *)opa, (float *)feat);
    count_launch();
    return rc_of(cudaGetLastError());
}

int ss_convert_f64_f32(const double *in, float *out, int64_t n, void *stream) {
    if (n < 0) return SS_ERR_DIMS;
    if (n == 0) return SS_OK;
    if (!in || !out) return SS_ERR_NULL;
    k_cvt_f64_f32<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(in, out, n);
    count_launch();
    return rc_of(cudaGetLastError());
}

int ss_convert_f32_f64(const float *in, double *out, int64_t n, void *stream) {
    if (n < 0) return SS_ERR_DIMS;
    if (n == 0) return SS_OK;
    if (!in || !out) return SS_ERR_NULL;
    k_cvt_f32_f64<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(in, out, n);
    count_launch();
    return rc_of(cudaGetLastError());
}

}  // extern "C"
