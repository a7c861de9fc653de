// Per-tile sort of the candidate lists (device functions shared by ss_project.cu and ss_raster.cu).
#pragma once
#include "ss_common.cuh"

namespace ss {
namespace {

// ---- per-tile sort -------------------------------------------------------------------
// Bitonic network in the "all comparators ascending" form: merge step k first compares
// i with i ^ (k-1) (flip), then i with i ^ j for j = k/4 ... 1 (disperse).  Because every
// comparator moves the minimum to the lower index, elements beyond n behave like +inf
// without being stored: comparators whose upper index is >= n are skipped.

__device__ __forceinline__ bool pair_less(unsigned long long ka, int ia, unsigned long long kb, int ib) {
    return ka < kb || (ka == kb && ia < ib);
}

template <typename KeyPtr, typename IdPtr>
__device__ __forceinline__ void cas(KeyPtr keys, IdPtr ids, int l, int r) {
    unsigned long long kl = keys[l], kr = keys[r];
    int il = ids[l], ir = ids[r];
    if (pair_less(kr, ir, kl, il)) { keys[l] = kr; keys[r] = kl; ids[l] = ir; ids[r] = il; }
}

template <typename KeyPtr, typename IdPtr>
__device__ void bitonic_sort_cta(KeyPtr keys, IdPtr ids, int n) {
    int np2 = 1;
    while (np2 < n) np2 <<= 1;
    int half = np2 >> 1;
    for (int k = 2; k <= np2; k <<= 1) {
        int hk = k >> 1;
        for (int c = threadIdx.x; c < half; c += blockDim.x) {  // flip
            int p = c & (hk - 1);
            int base = (c - p) << 1;
            int l = base + p, r = base + k - 1 - p;
            if (r < n) cas(keys, ids, l, r);
        }
        __syncthreads();
        for (int j = hk >> 1; j >= 1; j >>= 1) {  // disperse
            for (int c = threadIdx.x; c < half; c += blockDim.x) {
                int p = c & (j - 1);
                int l = ((c - p) << 1) + p, r = l + j;
                if (r < n) cas(keys, ids, l, r);
            }
            __syncthreads();
        }
    }
}

// ---- small segments: hybrid register / shared-memory bitonic sort -------------------------------
// The first version ran all log2(n)(log2(n)+1)/2 stages through shared memory and was bound by
// shared-memory bandwidth and barriers (ncu: l1tex 87 %, barrier stall 4.3).  Here every stage whose
// partner distance is < 64 runs in registers: a warp holds a 64-element block (two per lane) and
// exchanges with shuffles; only the flip and the j >= 64 disperse stages of the k >= 128 merges touch
// shared memory (6 of 45 stages at n = 512).  Segments are padded to a power of two with +inf keys.
struct El { unsigned long long k; int id; };

__device__ __forceinline__ bool el_less(const El &a, const El &b) { return a.k < b.k || (a.k == b.k && a.id < b.id); }
__device__ __forceinline__ El el_shfl_xor(const El &e, int m) {
    El r;
    r.k = __shfl_xor_sync(0xffffffffu, e.k, m);
    r.id = __shfl_xor_sync(0xffffffffu, e.id, m);
    return r;
}
__device__ __forceinline__ void el_keep(El &e, const El &p, bool keep_min) {
    const bool p_less = el_less(p, e);
    if (p_less == keep_min) e = p;  // keep_min: take the partner if it is smaller; else if it is not smaller
}
// partner lane = lane ^ m for both halves
__device__ __forceinline__ void warp_stage(El &e0, El &e1, int m, bool keep_min) {
    const El p0 = el_shfl_xor(e0, m), p1 = el_shfl_xor(e1, m);
    el_keep(e0, p0, keep_min);
    el_keep(e1, p1, keep_min);
}
// disperse stages j = 32, 16, ..., 1 on a 64-element block held as (e0 = block[lane], e1 = block[lane + 32])
__device__ __forceinline__ void warp_disperse64(El &e0, El &e1, int lane) {
    if (el_less(e1, e0)) { const El t = e0; e0 = e1; e1 = t; }  // j = 32
#pragma unroll
    for (int j = 16; j >= 1; j >>= 1) warp_stage(e0, e1, j, (lane & j) == 0);
}
// full sort of the 64-element block: merges k = 2 .. 64
__device__ __forceinline__ void warp_sort64(El &e0, El &e1, int lane) {
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
        warp_stage(e0, e1, k - 1, (lane & (k >> 1)) == 0);  // flip: i <-> i ^ (k - 1)
#pragma unroll
        for (int j = k >> 2; j >= 1; j >>= 1) warp_stage(e0, e1, j, (lane & j) == 0);
    }
    {   // flip of the k = 64 merge: index i <-> 63 - i, i.e. my e0 with e1 of lane ^ 31 and vice versa
        const El p1 = el_shfl_xor(e1, 31), p0 = el_shfl_xor(e0, 31);
        el_keep(e0, p1, true);
        el_keep(e1, p0, false);
    }
#pragma unroll
    for (int j = 16; j >= 1; j >>= 1) warp_stage(e0, e1, j, (lane & j) == 0);
}

// ---- segments of <= 512 pairs (every tile of the benchmark): the same network on ONE 32-bit word ---------
// A (key, id) element costs three shuffles and a two-word comparison per compare-exchange.  Inside one tile the
// order-preserving key bits span a small range, so the element is packed as
//     [ (key - key_min) >> shift : 23 bits | position in the segment : 9 bits ],   shift = max(0, bits(range) - 23):
// a monotone integer map of the key (no floating point), every word distinct, one shuffle and a min/max per
// compare-exchange.  Words whose 23-bit parts tie -- a handful per frame -- are then ranked exactly inside
// their run by the full (key, id) pair; a segment where more than a quarter of the words tie (equal depths,
// one far outlier stretching the range) takes the 64-bit network instead.
__device__ __forceinline__ void u_stage(unsigned &e0, unsigned &e1, int m, bool keep_min) {
    const unsigned p0 = __shfl_xor_sync(0xffffffffu, e0, m), p1 = __shfl_xor_sync(0xffffffffu, e1, m);
    e0 = keep_min ? min(e0, p0) : max(e0, p0);
    e1 = keep_min ? min(e1, p1) : max(e1, p1);
}
__device__ __forceinline__ void u_disperse64(unsigned &e0, unsigned &e1, int lane) {
    if (e1 < e0) { const unsigned t = e0; e0 = e1; e1 = t; }  // j = 32
#pragma unroll
    for (int j = 16; j >= 1; j >>= 1) u_stage(e0, e1, j, (lane & j) == 0);
}
__device__ __forceinline__ void u_sort64(unsigned &e0, unsigned &e1, int lane) {
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
        u_stage(e0, e1, k - 1, (lane & (k >> 1)) == 0);
#pragma unroll
        for (int j = k >> 2; j >= 1; j >>= 1) u_stage(e0, e1, j, (lane & j) == 0);
    }
    {   // flip of the k = 64 merge: index i <-> 63 - i
        const unsigned p1 = __shfl_xor_sync(0xffffffffu, e1, 31), p0 = __shfl_xor_sync(0xffffffffu, e0, 31);
        e0 = min(e0, p1);
        e1 = max(e1, p0);
    }
#pragma unroll
    for (int j = 16; j >= 1; j >>= 1) u_stage(e0, e1, j, (lane & j) == 0);
}

constexpr int PACK_MAX = 512;  // 9 index bits

// Where a tile's unsorted segment comes from: the tile's bucket filled by k_project (+ a gather of the
// per-sphere keys), or -- fallback -- the pairs written by k_emit.
struct SegSrc {
    const unsigned long long *pair_key; const int *pair_id;  // emitted pairs, already offset to the segment
    const int *bucket; const unsigned long long *key;        // this tile's bucket; per-sphere keys
    int c_small;                                             // ids of spheres touching <= 4 tiles sit at the front
    bool direct;
    __device__ __forceinline__ void load(int i, unsigned long long &k, int &id) const {
        if (direct) {
            id = bucket[i < c_small ? i : BUCKET_CAP - 1 - (i - c_small)];
            k = key[id];
        } else {
            k = pair_key[i];
            id = pair_id[i];
        }
    }
};

// pk[0 .. n) is sorted by the key part of the packed words (index part: IDX_BITS low bits).  Words in a run of
// equal key parts are ranked exactly by (key, id); returns false, writing nothing, when more than a quarter of
// the words tie (the caller then runs the 64-bit network).  Block-wide call.
template <int IDX_BITS, typename KeyFn>
__device__ bool rank_ties_and_write(const unsigned *pk, int n, KeyFn keys, const int *ids, int *out) {
    __shared__ int s_ties[8];
    constexpr unsigned IDX_MASK = (1u << IDX_BITS) - 1u;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int total = 0;
    for (int p = tid; p < n; p += blockDim.x) {
        const unsigned q = pk[p] >> IDX_BITS;
        total += (p > 0 && (pk[p - 1] >> IDX_BITS) == q) || (p + 1 < n && (pk[p + 1] >> IDX_BITS) == q);
    }
    total = __reduce_add_sync(0xffffffffu, total);
    if (lane == 0) s_ties[warp] = total;
    __syncthreads();
    total = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) total += s_ties[w];
    __syncthreads();  // s_ties may be rewritten by the next segment of a persistent CTA
    if (total * 4 > n) return false;
    for (int p = tid; p < n; p += blockDim.x) {
        const unsigned w = pk[p];
        const unsigned q = w >> IDX_BITS;
        const int me = (int)(w & IDX_MASK);
        int dst = p;
        if (total > 0 && ((p > 0 && (pk[p - 1] >> IDX_BITS) == q) || (p + 1 < n && (pk[p + 1] >> IDX_BITS) == q))) {
            int a = p;
            while (a > 0 && (pk[a - 1] >> IDX_BITS) == q) --a;
            const unsigned long long km = keys(me);
            const int im = ids[me];
            int rank = 0;
            for (int j = a; j < n && (pk[j] >> IDX_BITS) == q; ++j) {
                const int o = (int)(pk[j] & IDX_MASK);
                rank += pair_less(keys(o), ids[o], km, im) ? 1 : 0;
            }
            dst = a + rank;
        }
        out[dst] = ids[me];
    }
    return true;
}

// Sorts the segment [s0, s0 + n), n <= 512, writing pair_id in place.  keys / ids: shared staging (>= 512 entries);
// pk: 512 words.  Returns false (nothing written) when too many packed words tie.
__device__ bool sort_packed512(int s0, int n, int np2, const SegSrc &src, int *pair_id,
                               unsigned long long *keys, int *ids, unsigned *pk) {
    // The key range is taken from the UPPER words of the keys only (sign, exponent and 20 mantissa bits of the
    // depth): lo = min upper word << 32 <= every key, range = (max upper word : ffffffff) - lo >= the true range.
    // The map stays monotone, and it is the same map whenever the depths of a tile differ in their upper words --
    // always, except for near-equal depths, whose words then tie and take the exact ranking below.  A 32-bit
    // min / max costs a quarter of the instructions of the 64-bit one (10 % of this kernel).
    __shared__ unsigned s_min[8], s_max[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n_blocks = np2 >> 6;  // <= 8: at most one 64-block per warp
    const int i0 = (warp << 6) + lane, i1 = i0 + 32;
    unsigned long long k0 = ~0ull, k1 = ~0ull;
    unsigned lo32 = 0xffffffffu, hi32 = 0u;
    if (warp < n_blocks) {
        int id0, id1;
        if (i0 < n) { src.load(i0, k0, id0); keys[i0] = k0; ids[i0] = id0; lo32 = hi32 = (unsigned)(k0 >> 32); }
        if (i1 < n) {
            src.load(i1, k1, id1); keys[i1] = k1; ids[i1] = id1;
            lo32 = min(lo32, (unsigned)(k1 >> 32)); hi32 = max(hi32, (unsigned)(k1 >> 32));
        }
    }
    lo32 = __reduce_min_sync(0xffffffffu, lo32);  // (REDUX: one instruction each instead of a 5-step butterfly)
    hi32 = __reduce_max_sync(0xffffffffu, hi32);
    if (lane == 0) { s_min[warp] = lo32; s_max[warp] = hi32; }
    __syncthreads();
#pragma unroll
    for (int w = 0; w < 8; ++w) { lo32 = min(lo32, s_min[w]); hi32 = max(hi32, s_max[w]); }
    const unsigned long long lo = (unsigned long long)lo32 << 32;
    const unsigned long long range = (((unsigned long long)hi32 << 32) | 0xffffffffull) - lo;
    const int bits = 64 - __clzll((long long)range);  // >= 32
    const int shift = bits > 23 ? bits - 23 : 0;
    unsigned e0 = 0xffffffffu, e1 = 0xffffffffu;  // padding sorts last
    if (warp < n_blocks) {
        if (i0 < n) e0 = ((unsigned)((k0 - lo) >> shift) << 9) | (unsigned)i0;
        if (i1 < n) e1 = ((unsigned)((k1 - lo) >> shift) << 9) | (unsigned)i1;
        u_sort64(e0, e1, lane);
        if (n_blocks > 1) { pk[i0] = e0; pk[i1] = e1; }
    }
    if (n_blocks > 1) {
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
            if (warp < n_blocks) {  // j = 32 .. 1 in registers
                e0 = pk[i0]; e1 = pk[i1];
                u_disperse64(e0, e1, lane);
                pk[i0] = e0; pk[i1] = e1;
            }
            __syncthreads();
        }
    } else {
        if (warp == 0) { pk[i0] = e0; pk[i1] = e1; }
        __syncthreads();
    }
    return rank_ties_and_write<9>(pk, n, [keys](int i) { return keys[i]; }, ids, pair_id + s0);
}

// Sorts the list of tile t when it holds <= SORT_SMALL pairs (longer lists belong to k_tile_sort_mid / _big), writing
// the sorted sphere ids to pair_id.  Block-wide call (256 threads); keys (512 x 8 B), ids (512 x 4 B) and pk
// (512 x 4 B) are shared-memory scratch.  Called by k_tile_sort_small and -- fused -- by k_raster before it draws
// the tile, where the sort's shuffle / min-max work fills issue slots the other resident tiles' drain rounds leave idle.
__device__ __forceinline__ void sort_small_segment(const int *__restrict__ tile_start,
                                                   const unsigned long long *__restrict__ pair_key, int *pair_id,
                                                   const int *__restrict__ bucket,
                                                   const unsigned long long *__restrict__ key,
                                                   const int *__restrict__ tile_cursor, long long flags, int t,
                                                   unsigned long long *keys, int *ids, unsigned *pk) {
    const int s0 = tile_start[t], n = tile_start[t + 1] - s0;
    SegSrc src;
    src.direct = !(flags & SS_FLAG_LIST_FALLBACK);
    src.pair_key = pair_key + s0; src.pair_id = pair_id + s0;
    src.bucket = bucket + (size_t)t * BUCKET_CAP; src.key = key;
    src.c_small = tile_cursor[t];
    if (n == 1 && src.direct && threadIdx.x == 0) pair_id[s0] = src.bucket[src.c_small ? 0 : BUCKET_CAP - 1];
    if (n < 2 || n > SORT_SMALL) return;
    int np2 = 64;
    while (np2 < n) np2 <<= 1;
    if (np2 <= PACK_MAX) {
        if (sort_packed512(s0, n, np2, src, pair_id, keys, ids, pk)) return;
        __syncthreads();  // too many ties: the 64-bit network below re-reads the untouched segment
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int n_blocks = np2 >> 6;
    // load straight into registers, sort each 64-block (merges k = 2..64), park in shared memory
    for (int b = warp; b < n_blocks; b += 8) {
        const int i0 = (b << 6) + lane, i1 = i0 + 32;
        El e0, e1;
        e0.k = ~0ull; e0.id = 0x7fffffff; e1.k = ~0ull; e1.id = 0x7fffffff;
        if (i0 < n) src.load(i0, e0.k, e0.id);
        if (i1 < n) src.load(i1, e1.k, e1.id);
        warp_sort64(e0, e1, lane);
        if (np2 == 64) {  // done: single block
            if (i0 < n) pair_id[s0 + i0] = e0.id;
            if (i1 < n) pair_id[s0 + i1] = e1.id;
        } else {
            keys[i0] = e0.k; ids[i0] = e0.id; keys[i1] = e1.k; ids[i1] = e1.id;
        }
    }
    if (np2 == 64) return;
    __syncthreads();
    const int half = np2 >> 1;
    for (int k = 128; k <= np2; k <<= 1) {
        const int hk = k >> 1;
        for (int c = threadIdx.x; c < half; c += blockDim.x) {  // flip, shared memory
            const int p = c & (hk - 1);
            const int base = (c - p) << 1;
            cas(keys, ids, base + p, base + k - 1 - p);
        }
        __syncthreads();
        for (int j = hk >> 1; j >= 64; j >>= 1) {  // long-distance disperse stages, shared memory
            for (int c = threadIdx.x; c < half; c += blockDim.x) {
                const int p = c & (j - 1);
                const int l = ((c - p) << 1) + p;
                cas(keys, ids, l, l + j);
            }
            __syncthreads();
        }
        const bool last = (k == np2);
        for (int b = warp; b < n_blocks; b += 8) {  // j = 32 .. 1 in registers
            const int i0 = (b << 6) + lane, i1 = i0 + 32;
            El e0, e1;
            e0.k = keys[i0]; e0.id = ids[i0]; e1.k = keys[i1]; e1.id = ids[i1];
            warp_disperse64(e0, e1, lane);
            if (last) {
                if (i0 < n) pair_id[s0 + i0] = e0.id;
                if (i1 < n) pair_id[s0 + i1] = e1.id;
            } else {
                keys[i0] = e0.k; ids[i0] = e0.id; keys[i1] = e1.k; ids[i1] = e1.id;
            }
        }
        if (!last) __syncthreads();
    }
}


}  // namespace
}  // namespace ss
