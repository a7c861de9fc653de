/*
 * ss_oracle.c -- CPU restatement of the reference sphere renderer hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity oracle for the CUDA path:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it.  The product (paper_2004_07484_b200/) never
 * imports, links or calls anything in oracle/.
 *
 * It restates, in plain scalar float64 C, the algorithm of the reference
 * package `softsphere` (pure NumPy, /root/reference/pkg/src/softsphere):
 *
 *   or_compute_bounds   <- raster.py:181-236 (compute_bounds),
 *                          raster.py:130-154 (_axis_extent_pinhole),
 *                          raster.py:157-178 (_discretize_extent),
 *                          camera.py:190-192 (world_to_camera)
 *   or_sort_order       <- raster.py:239-244 (sort_draw_records)
 *   or_bin_tiles        <- raster.py:267-293 (_bin_tiles), :420-434 (_tile_grid)
 *   or_render_forward   <- raster.py:437-512 (render_forward),
 *                          raster.py:300-325 (_intersect_chunk),
 *                          raster.py:328-417 (_draw_tile),
 *                          camera.py:332-357 (sensor_rays_camera_frame)
 *   or_render_backward  <- grad.py:323-357 (render_backward),
 *                          grad.py:89-179 (_hit_gradients),
 *                          grad.py:210-259 (_accumulate_tiles),
 *                          grad.py:262-302 (accumulate_and_normalize),
 *                          grad.py:305-320 (gate_small_spheres)
 *
 * Parity is PINNED: oracle/pin_against_reference.py runs this library against
 * the imported reference in the build container and writes the golden
 * fixtures under tests/golden/ (ids exact, floats to <= 1e-11).
 *
 * Build: gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC (see oracle/Makefile).
 * -ffp-contract=off keeps a*b+c as two roundings like NumPy's elementwise ops.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_PINHOLE 0
#define OR_ORTHO 1
#define OR_INT_HUGE 1073741824.0 /* 1 << 30, raster.py:34 */
#define OR_GATE_RADIUS_PX 3.0    /* grad.py:42 */

typedef struct {
    double t[3];     /* camera position, world */
    double R[9];     /* row-major, p_cam = R (p - t); camera.py:5 */
    double focal;
    double sensor_w;
    double near_;
    double far_;
    int32_t width;
    int32_t height;
    int32_t mode;    /* 0 pinhole, 1 orthographic */
    int32_t pad;
} OrCamera;

static double clampd(double x, double lo, double hi) {
    return x < lo ? lo : (x > hi ? hi : x);
}

/* ---- Step 0 ------------------------------------------------------------ */

/* raster.py:130-154 */
static void axis_extent_pinhole(double ca, double cz, double r, double focal,
                                double *lo, double *hi, int *empty) {
    const double half = M_PI / 2.0;
    double n2 = ca * ca + cz * cz;
    double n = sqrt(n2);
    int full = n2 <= r * r;
    double nn = n > 1e-300 ? n : 1e-300;
    double beta = asin(clampd(r / nn, 0.0, 1.0));
    double phi = atan2(ca, cz);
    double lo_a = phi - beta, hi_a = phi + beta;
    *empty = ((lo_a >= half) || (hi_a <= -half)) && !full;
    double cap = half - 1e-9;
    *lo = (lo_a <= -half) ? -INFINITY : focal * tan(clampd(lo_a, -cap, cap));
    *hi = (hi_a >= half) ? INFINITY : focal * tan(clampd(hi_a, -cap, cap));
    if (full) { *lo = -INFINITY; *hi = INFINITY; }
}

/* raster.py:157-178 */
static void discretize_extent(double lo_px, double hi_px, double center_px, int limit,
                              int64_t *i_lo_out, int64_t *i_hi_out, int *outside) {
    double pad = 1e-9 * (1.0 + fabs(lo_px));
    double lo_f = clampd(ceil(lo_px - 0.5 - pad), -OR_INT_HUGE, OR_INT_HUGE);
    pad = 1e-9 * (1.0 + fabs(hi_px));
    double hi_f = clampd(floor(hi_px - 0.5 + pad), -OR_INT_HUGE, OR_INT_HUGE);
    int64_t i_lo = (int64_t)lo_f, i_hi = (int64_t)hi_f;
    if (i_lo > i_hi) {
        double c = isfinite(center_px) ? center_px : 0.0;
        int64_t nearest = (int64_t)clampd(floor(c), -OR_INT_HUGE, OR_INT_HUGE);
        i_lo = nearest; i_hi = nearest;
    }
    *outside = (i_hi < 0) || (i_lo > limit - 1);
    if (i_lo < 0) i_lo = 0; if (i_lo > limit - 1) i_lo = limit - 1;
    if (i_hi < 0) i_hi = 0; if (i_hi > limit - 1) i_hi = limit - 1;
    *i_lo_out = i_lo; *i_hi_out = i_hi;
}

static void world_to_camera(const OrCamera *cam, const double *p, double *c) {
    double dx = p[0] - cam->t[0], dy = p[1] - cam->t[1], dz = p[2] - cam->t[2];
    const double *R = cam->R;
    c[0] = dx * R[0] + dy * R[1] + dz * R[2];
    c[1] = dx * R[3] + dy * R[4] + dz * R[5];
    c[2] = dx * R[6] + dy * R[7] + dz * R[8];
}

/* raster.py:181-236.  Validation (scene.py:91-114) is the caller's job and is
 * restated in oracle/oracle.py. */
int or_compute_bounds(int64_t m, const double *pos, const double *rad, const OrCamera *cam,
                      int64_t *x_min, int64_t *x_max, int64_t *y_min, int64_t *y_max,
                      uint8_t *on_sensor, double *proj_r, double *center_cam,
                      double *earliest) {
    int w = cam->width, h = cam->height;
    double ppu = (double)w / cam->sensor_w;
    for (int64_t i = 0; i < m; ++i) {
        double c[3];
        world_to_camera(cam, pos + 3 * i, c);
        double r = rad[i];
        double lo_x, hi_x, lo_y, hi_y, u_c, v_c, e, pr;
        int empty_x = 0, empty_y = 0;
        int behind = (c[2] + r) <= 0.0;
        if (cam->mode == OR_PINHOLE) {
            axis_extent_pinhole(c[0], c[2], r, cam->focal, &lo_x, &hi_x, &empty_x);
            axis_extent_pinhole(c[1], c[2], r, cam->focal, &lo_y, &hi_y, &empty_y);
            double safe_z = c[2] > 0 ? c[2] : INFINITY;
            u_c = w / 2.0 + cam->focal * c[0] / safe_z * ppu;
            v_c = h / 2.0 + cam->focal * c[1] / safe_z * ppu;
            double d2 = c[0] * c[0] + c[1] * c[1] + c[2] * c[2];
            e = sqrt(d2) - r;
            double den = d2 - r * r;
            if (den < 1e-300) den = 1e-300;
            pr = (cam->focal * r / sqrt(den)) * ppu;
            if (d2 <= r * r) pr = (double)(w > h ? w : h);
        } else {
            lo_x = c[0] - r; hi_x = c[0] + r;
            lo_y = c[1] - r; hi_y = c[1] + r;
            u_c = w / 2.0 + c[0] * ppu;
            v_c = h / 2.0 + c[1] * ppu;
            e = c[2] - r;
            pr = r * ppu;
        }
        int out_x, out_y;
        discretize_extent(w / 2.0 + lo_x * ppu, w / 2.0 + hi_x * ppu, u_c, w,
                          &x_min[i], &x_max[i], &out_x);
        discretize_extent(h / 2.0 + lo_y * ppu, h / 2.0 + hi_y * ppu, v_c, h,
                          &y_min[i], &y_max[i], &out_y);
        int on = !(behind || empty_x || empty_y || out_x || out_y);
        on_sensor[i] = (uint8_t)on;
        earliest[i] = on ? e : INFINITY;
        proj_r[i] = pr;
        center_cam[3 * i] = c[0]; center_cam[3 * i + 1] = c[1]; center_cam[3 * i + 2] = c[2];
    }
    return 0;
}

/* ---- sort (raster.py:239-244): stable ascending argsort ------------------ */

static void merge_sort_idx(const double *key, int64_t *idx, int64_t *tmp, int64_t n) {
    for (int64_t width = 1; width < n; width *= 2) {
        for (int64_t lo = 0; lo < n; lo += 2 * width) {
            int64_t mid = lo + width < n ? lo + width : n;
            int64_t hi = lo + 2 * width < n ? lo + 2 * width : n;
            int64_t a = lo, b = mid, o = lo;
            while (a < mid && b < hi) {
                /* stable: take from the left run unless right is strictly smaller */
                if (key[idx[b]] < key[idx[a]]) tmp[o++] = idx[b++];
                else tmp[o++] = idx[a++];
            }
            while (a < mid) tmp[o++] = idx[a++];
            while (b < hi) tmp[o++] = idx[b++];
        }
        memcpy(idx, tmp, (size_t)n * sizeof(int64_t));
    }
}

int or_sort_order(int64_t m, const double *earliest, int64_t *order) {
    int64_t *tmp = (int64_t *)malloc((size_t)(m > 0 ? m : 1) * sizeof(int64_t));
    if (!tmp) return -1;
    for (int64_t i = 0; i < m; ++i) order[i] = i;
    merge_sort_idx(earliest, order, tmp, m);
    free(tmp);
    return 0;
}

/* ---- tile binning (raster.py:267-293) ------------------------------------ */
/* bounds arrays are in SORTED order (first n_active entries are on-sensor).
 * Pass record_seq == NULL to get only tile_starts (and the total in
 * tile_starts[n_tiles]).  Within a tile the order is ascending sorted index,
 * which is what the reference's stable argsort by tile id produces. */
int or_bin_tiles(int64_t n_active, const int64_t *x_min, const int64_t *x_max,
                 const int64_t *y_min, const int64_t *y_max, int tile, int ntx, int nty,
                 int64_t *record_seq, int64_t *tile_starts) {
    int64_t n_tiles = (int64_t)ntx * nty;
    memset(tile_starts, 0, (size_t)(n_tiles + 1) * sizeof(int64_t));
    for (int64_t i = 0; i < n_active; ++i) {
        int64_t tx0 = x_min[i] / tile, tx1 = x_max[i] / tile;
        int64_t ty0 = y_min[i] / tile, ty1 = y_max[i] / tile;
        for (int64_t ty = ty0; ty <= ty1; ++ty)
            for (int64_t tx = tx0; tx <= tx1; ++tx) tile_starts[ty * ntx + tx + 1] += 1;
    }
    for (int64_t t = 0; t < n_tiles; ++t) tile_starts[t + 1] += tile_starts[t];
    if (!record_seq) return 0;
    int64_t *cursor = (int64_t *)malloc((size_t)(n_tiles > 0 ? n_tiles : 1) * sizeof(int64_t));
    if (!cursor) return -1;
    memcpy(cursor, tile_starts, (size_t)n_tiles * sizeof(int64_t));
    for (int64_t i = 0; i < n_active; ++i) {
        int64_t tx0 = x_min[i] / tile, tx1 = x_max[i] / tile;
        int64_t ty0 = y_min[i] / tile, ty1 = y_max[i] / tile;
        for (int64_t ty = ty0; ty <= ty1; ++ty)
            for (int64_t tx = tx0; tx <= tx1; ++tx) record_seq[cursor[ty * ntx + tx]++] = i;
    }
    free(cursor);
    return 0;
}

/* ---- rays (camera.py:332-357) --------------------------------------------- */

typedef struct {
    double ox, oy;       /* origin (ortho) */
    double ux, uy, uz;   /* unit direction */
    double xs, ys;       /* sensor_xy */
    double inv_vnorm;
} OrRay;

static void pixel_ray(const OrCamera *cam, int px, int py, OrRay *ray) {
    double ps = cam->sensor_w / cam->width;
    double xs = ((px + 0.5) - cam->width / 2.0) * ps;
    double ys = ((py + 0.5) - cam->height / 2.0) * ps;
    ray->xs = xs; ray->ys = ys;
    if (cam->mode == OR_PINHOLE) {
        double vn = sqrt(xs * xs + ys * ys + cam->focal * cam->focal);
        ray->ux = xs / vn; ray->uy = ys / vn; ray->uz = cam->focal / vn;
        ray->ox = 0.0; ray->oy = 0.0;
        ray->inv_vnorm = 1.0 / vn;
    } else {
        ray->ux = 0.0; ray->uy = 0.0; ray->uz = 1.0;
        ray->ox = xs; ray->oy = ys;
        ray->inv_vnorm = 1.0;
    }
}

/* ---- forward (raster.py:328-417, :437-512) -------------------------------- */

typedef struct {
    int64_t m;
    int d;
    const double *center_cam, *radius, *opacity, *feature, *earliest; /* ORIGINAL order */
    const int64_t *order;       /* sorted idx -> original idx */
    const int64_t *record_seq;  /* sorted indices grouped by tile */
    const int64_t *tile_starts;
    const double *background;
    const OrCamera *cam;
    double gamma, eps, tau;
    int K, tile, chunk, ntx, nty, store_buffer;
    double *image, *bg_weight;
    int32_t *ids;
    double *z, *clos, *log_denom;
    int64_t *stats_rows; /* (n_tiles, 3) */
} FwdCtx;

static void draw_tile(const FwdCtx *cx, int ti) {
    const OrCamera *cam = cx->cam;
    int tx = ti % cx->ntx, ty = ti / cx->ntx;
    int x0 = tx * cx->tile, y0 = ty * cx->tile;
    int x1 = x0 + cx->tile < cam->width ? x0 + cx->tile : cam->width;
    int y1 = y0 + cx->tile < cam->height ? y0 + cx->tile : cam->height;
    int pw = x1 - x0, ph = y1 - y0, p = pw * ph;
    int d = cx->d, K = cx->K, chunk = cx->chunk;
    double g = cx->gamma, near_ = cam->near_, far_ = cam->far_;
    double inv_range = 1.0 / (far_ - near_);

    OrRay *rays = (OrRay *)malloc((size_t)p * sizeof(OrRay));
    double *mm = (double *)malloc((size_t)p * sizeof(double));
    double *denom = (double *)malloc((size_t)p * sizeof(double));
    double *num = (double *)calloc((size_t)p * d, sizeof(double));
    double *tz = (double *)malloc((size_t)p * K * sizeof(double));
    double *tc = (double *)calloc((size_t)p * K, sizeof(double));
    int32_t *tid = (int32_t *)malloc((size_t)p * K * sizeof(int32_t));
    uint8_t *done = (uint8_t *)calloc((size_t)p, 1);
    /* per-chunk scratch for one pixel */
    double *e_ch = (double *)malloc((size_t)chunk * sizeof(double));
    double *z_ch = (double *)malloc((size_t)chunk * sizeof(double));
    double *c_ch = (double *)malloc((size_t)chunk * sizeof(double));
    double *fsum = (double *)malloc((size_t)d * sizeof(double));

    double tile_cos = 1.0;
    for (int q = 0; q < p; ++q) {
        pixel_ray(cam, x0 + q % pw, y0 + q / pw, &rays[q]);
        mm[q] = cx->eps / g;
        denom[q] = 1.0;
        for (int k = 0; k < K; ++k) { tz[q * K + k] = -INFINITY; tid[q * K + k] = -1; }
    }
    if (cam->mode == OR_PINHOLE) {
        tile_cos = INFINITY;
        for (int q = 0; q < p; ++q) if (rays[q].uz < tile_cos) tile_cos = rays[q].uz;
    }

    int64_t s0 = cx->tile_starts[ti], s1 = cx->tile_starts[ti + 1];
    int64_t n_cand = s1 - s0, scanned = 0, hits_blended = 0;
    double log_tau = cx->tau > 0.0 ? log(cx->tau / (1.0 - cx->tau)) : 0.0;

    for (int64_t start = 0; start < n_cand; start += chunk) {
        int64_t cn = n_cand - start < chunk ? n_cand - start : chunk;
        if (cx->tau > 0.0) { /* raster.py:364-368 */
            int64_t first = cx->order[cx->record_seq[s0 + start]];
            double zb = (far_ - clampd(cx->earliest[first] * tile_cos, near_, far_)) * inv_range;
            int all_done = 1;
            for (int q = 0; q < p; ++q) {
                double z_stop = g * (log_tau + mm[q] + log(denom[q]));
                if (zb < z_stop) done[q] = 1;
                all_done &= done[q];
            }
            if (all_done) break;
        }
        scanned += cn;
        for (int q = 0; q < p; ++q) {
            if (done[q]) continue;
            const OrRay *ry = &rays[q];
            double new_m = mm[q];
            int any = 0;
            for (int64_t j = 0; j < cn; ++j) {
                int64_t sid = cx->order[cx->record_seq[s0 + start + j]];
                const double *c = cx->center_cam + 3 * sid;
                double r = cx->radius[sid];
                double t_along, dist2, zeta;
                if (cam->mode == OR_PINHOLE) { /* raster.py:307-311 */
                    t_along = ry->ux * c[0] + ry->uy * c[1] + ry->uz * c[2];
                    double n2 = c[0] * c[0] + c[1] * c[1] + c[2] * c[2];
                    dist2 = n2 - t_along * t_along;
                    zeta = t_along * ry->uz;
                } else {
                    t_along = c[2];
                    double dx = c[0] - ry->ox, dy = c[1] - ry->oy;
                    dist2 = dx * dx + dy * dy;
                    zeta = t_along;
                }
                if (dist2 < 0.0) dist2 = 0.0;
                double rr = r * r;
                double hc = rr - dist2; if (hc < 0.0) hc = 0.0;
                int hit = (dist2 < rr) && (t_along + sqrt(hc) > 0.0);
                if (!hit) { e_ch[j] = -INFINITY; continue; }
                any = 1;
                hits_blended += 1;
                double o = clampd(cx->opacity[sid], 0.0, 1.0);
                double zz = (far_ - clampd(zeta, near_, far_)) * inv_range;
                z_ch[j] = zz;
                c_ch[j] = 1.0 - sqrt(dist2) / r;
                e_ch[j] = o * zz / g;
                if (e_ch[j] > new_m) new_m = e_ch[j];
            }
            if (!any) continue;
            double scale = exp(mm[q] - new_m);
            double tsum = 0.0;
            for (int i = 0; i < d; ++i) fsum[i] = 0.0;
            for (int64_t j = 0; j < cn; ++j) {
                if (e_ch[j] == -INFINITY) continue;
                int64_t sid = cx->order[cx->record_seq[s0 + start + j]];
                double o = clampd(cx->opacity[sid], 0.0, 1.0);
                double term = o * c_ch[j] * exp(e_ch[j] - new_m);
                tsum += term;
                const double *f = cx->feature + (size_t)sid * d;
                for (int i = 0; i < d; ++i) fsum[i] += term * f[i];
                if (term > 0.0) { /* raster.py:389-399: top-K by (z desc, id asc) */
                    double *pz = tz + (size_t)q * K; double *pc = tc + (size_t)q * K;
                    int32_t *pi = tid + (size_t)q * K;
                    double zz = z_ch[j]; int32_t id = (int32_t)sid;
                    int last = K - 1;
                    if (zz > pz[last] || (zz == pz[last] && id < pi[last])) {
                        int k = last;
                        while (k > 0 && (zz > pz[k - 1] || (zz == pz[k - 1] && id < pi[k - 1]))) {
                            pz[k] = pz[k - 1]; pc[k] = pc[k - 1]; pi[k] = pi[k - 1]; --k;
                        }
                        pz[k] = zz; pc[k] = c_ch[j]; pi[k] = id;
                    }
                }
            }
            denom[q] = denom[q] * scale + tsum;
            for (int i = 0; i < d; ++i) num[(size_t)q * d + i] = num[(size_t)q * d + i] * scale + fsum[i];
            mm[q] = new_m;
        }
    }

    int n_done = 0;
    for (int q = 0; q < p; ++q) { /* raster.py:401-417 */
        int gx = x0 + q % pw, gy = y0 + q / pw;
        size_t pix = (size_t)gy * cam->width + gx;
        double ld = mm[q] + log(denom[q]);
        double w_bg = exp(cx->eps / g - ld);
        for (int i = 0; i < d; ++i)
            cx->image[pix * d + i] = num[(size_t)q * d + i] / denom[q] + w_bg * cx->background[i];
        cx->bg_weight[pix] = w_bg;
        if (cx->store_buffer) {
            for (int k = 0; k < K; ++k) {
                int empty = tz[q * K + k] == -INFINITY;
                cx->ids[pix * K + k] = empty ? -1 : tid[q * K + k];
                cx->z[pix * K + k] = empty ? 0.0 : tz[q * K + k];
                cx->clos[pix * K + k] = tc[q * K + k];
            }
            cx->log_denom[pix] = ld;
        }
        n_done += done[q];
    }
    cx->stats_rows[3 * ti] = scanned;
    cx->stats_rows[3 * ti + 1] = hits_blended;
    cx->stats_rows[3 * ti + 2] = n_done;
    free(rays); free(mm); free(denom); free(num); free(tz); free(tc); free(tid); free(done);
    free(e_ch); free(z_ch); free(c_ch); free(fsum);
}

/* stats: [spheres_total, spheres_on_sensor, candidates_tested, hits_blended,
 *         pixels_early_stopped, tiles]  (raster.py:113-123, :504-511) */
int or_render_forward(int64_t m, int d, const double *pos, const double *rad, const double *opa,
                      const double *feat, const double *bg, const OrCamera *cam, double gamma,
                      double eps, double tau, int K, int tile, int chunk, int store_buffer,
                      int threads, double *image, double *bg_weight, int32_t *ids, double *z,
                      double *clos, double *log_denom, int64_t *stats) {
    int ntx = (cam->width + tile - 1) / tile, nty = (cam->height + tile - 1) / tile;
    int64_t n_tiles = (int64_t)ntx * nty;
    size_t mm = (size_t)(m > 0 ? m : 1);
    int64_t *x_min = malloc(mm * 8), *x_max = malloc(mm * 8), *y_min = malloc(mm * 8),
            *y_max = malloc(mm * 8), *order = malloc(mm * 8);
    int64_t *sx0 = malloc(mm * 8), *sx1 = malloc(mm * 8), *sy0 = malloc(mm * 8), *sy1 = malloc(mm * 8);
    uint8_t *on = malloc(mm);
    double *proj_r = malloc(mm * 8), *cc = malloc(mm * 24), *earliest = malloc(mm * 8);
    int64_t *tile_starts = malloc((size_t)(n_tiles + 1) * 8);
    int64_t *stats_rows = calloc((size_t)n_tiles * 3, 8);
    or_compute_bounds(m, pos, rad, cam, x_min, x_max, y_min, y_max, on, proj_r, cc, earliest);
    or_sort_order(m, earliest, order);
    int64_t n_active = 0;
    for (int64_t i = 0; i < m; ++i) n_active += on[i];
    for (int64_t i = 0; i < m; ++i) {
        sx0[i] = x_min[order[i]]; sx1[i] = x_max[order[i]];
        sy0[i] = y_min[order[i]]; sy1[i] = y_max[order[i]];
    }
    or_bin_tiles(n_active, sx0, sx1, sy0, sy1, tile, ntx, nty, NULL, tile_starts);
    int64_t total = tile_starts[n_tiles];
    int64_t *record_seq = malloc((size_t)(total > 0 ? total : 1) * 8);
    or_bin_tiles(n_active, sx0, sx1, sy0, sy1, tile, ntx, nty, record_seq, tile_starts);

    FwdCtx cx = {m, d, cc, rad, opa, feat, earliest, order, record_seq, tile_starts, bg, cam,
                 gamma, eps, tau, K, tile, chunk, ntx, nty, store_buffer,
                 image, bg_weight, ids, z, clos, log_denom, stats_rows};
    if (threads < 1) threads = 1;
#pragma omp parallel for schedule(dynamic, 4) num_threads(threads)
    for (int64_t ti = 0; ti < n_tiles; ++ti) draw_tile(&cx, (int)ti);

    stats[0] = m; stats[1] = n_active; stats[2] = stats[3] = stats[4] = 0; stats[5] = n_tiles;
    for (int64_t ti = 0; ti < n_tiles; ++ti) {
        stats[2] += stats_rows[3 * ti]; stats[3] += stats_rows[3 * ti + 1];
        stats[4] += stats_rows[3 * ti + 2];
    }
    free(x_min); free(x_max); free(y_min); free(y_max); free(order); free(sx0); free(sx1);
    free(sy0); free(sy1); free(on); free(proj_r); free(cc); free(earliest); free(tile_starts);
    free(stats_rows); free(record_seq);
    return 0;
}

/* ---- backward (grad.py) ---------------------------------------------------- */

typedef struct {
    int n;          /* unique spheres in this tile */
    int32_t *uid;   /* sorted unique ids */
    double *sums;   /* n x ncols */
    int64_t *cnt;   /* n */
} TileAcc;

typedef struct {
    int64_t m; int d, K, tile, ntx, nty, ncols;
    const double *center_cam, *radius, *opacity, *feature, *background;
    const OrCamera *cam;
    double gamma, eps;
    const int32_t *ids; const double *z, *clos, *log_denom, *upstream;
    TileAcc *acc;
} BwdCtx;

typedef struct { int32_t id; int32_t seq; } IdSeq;
static int cmp_idseq(const void *a, const void *b) {
    const IdSeq *x = (const IdSeq *)a, *y = (const IdSeq *)b;
    if (x->id != y->id) return x->id < y->id ? -1 : 1;
    return x->seq < y->seq ? -1 : (x->seq > y->seq);
}

/* grad.py:89-179 for one (pixel, slot); writes ncols = 3+1+1+d+2 values */
static void hit_gradient(const BwdCtx *bx, const OrRay *ry, int32_t id, double zz, double cl,
                         double ld, const double *up, const double *f_hat, double *col) {
    const OrCamera *cam = bx->cam;
    int d = bx->d;
    double g = bx->gamma;
    double o = clampd(bx->opacity[id], 0.0, 1.0);
    const double *f = bx->feature + (size_t)id * d;
    double exp_shift = exp(o * zz / g - ld);
    double wgt = o * cl * exp_shift;
    double a_coef = 0.0;
    for (int i = 0; i < d; ++i) a_coef += up[i] * (f[i] - f_hat[i]);
    double dl_dz = a_coef * wgt * o / g;
    double dl_dc = a_coef * o * exp_shift;
    double dl_do = a_coef * cl * exp_shift * (1.0 + o * zz / g);
    const double *c = bx->center_cam + 3 * (size_t)id;
    double radius = bx->radius[id];
    double t_along, dv[3];
    if (cam->mode == OR_PINHOLE) {
        t_along = c[0] * ry->ux + c[1] * ry->uy + c[2] * ry->uz;
        dv[0] = c[0] - t_along * ry->ux; dv[1] = c[1] - t_along * ry->uy; dv[2] = c[2] - t_along * ry->uz;
    } else {
        t_along = c[2];
        dv[0] = c[0] - ry->ox; dv[1] = c[1] - ry->oy; dv[2] = 0.0;
    }
    double dd = dv[0] * dv[0] + dv[1] * dv[1] + dv[2] * dv[2];
    double dist = sqrt(dd > 0.0 ? dd : 0.0);
    int interior = (0.0 < zz) && (zz < 1.0);
    double dl_dzeta = interior ? dl_dz * (-1.0 / (cam->far_ - cam->near_)) : 0.0;
    double dl_ddist = -dl_dc / (radius > 1e-300 ? radius : 1e-300);
    double rr = radius * radius;
    double d_radius = dl_dc * dist / (rr > 1e-300 ? rr : 1e-300);
    double inv_dist = dist > 1e-12 ? 1.0 / (dist > 1e-300 ? dist : 1e-300) : 0.0;
    double dh[3] = {dv[0] * inv_dist, dv[1] * inv_dist, dv[2] * inv_dist};
    double gc[3], g_focal, g_sensor;
    if (cam->mode == OR_PINHOLE) {
        double u[3] = {ry->ux, ry->uy, ry->uz};
        double zu = dl_dzeta * u[2];
        double gu[3];
        double s1 = dl_ddist * (-t_along) * inv_dist;
        for (int j = 0; j < 3; ++j) {
            gc[j] = dl_ddist * dh[j] + zu * u[j];
            gu[j] = s1 * c[j];
            gu[j] += zu * c[j];
        }
        gu[2] += dl_dzeta * t_along;
        double gdu = gu[0] * u[0] + gu[1] * u[1] + gu[2] * u[2];
        double pr[3] = {gu[0] - gdu * u[0], gu[1] - gdu * u[1], gu[2] - gdu * u[2]};
        g_focal = pr[2] * ry->inv_vnorm;
        g_sensor = (pr[0] * ry->xs + pr[1] * ry->ys) * ry->inv_vnorm / cam->sensor_w;
    } else {
        for (int j = 0; j < 3; ++j) gc[j] = dl_ddist * dh[j];
        gc[2] += dl_dzeta;
        g_sensor = -(dl_ddist * inv_dist) * (dv[0] * ry->xs + dv[1] * ry->ys) / cam->sensor_w;
        g_focal = 0.0;
    }
    col[0] = gc[0]; col[1] = gc[1]; col[2] = gc[2];
    col[3] = d_radius; col[4] = dl_do;
    for (int i = 0; i < d; ++i) col[5 + i] = wgt * up[i];
    col[5 + d] = g_focal; col[6 + d] = g_sensor;
}

static void backward_tile(const BwdCtx *bx, int ti) {
    const OrCamera *cam = bx->cam;
    int tx = ti % bx->ntx, ty = ti / bx->ntx;
    int x0 = tx * bx->tile, y0 = ty * bx->tile;
    int x1 = x0 + bx->tile < cam->width ? x0 + bx->tile : cam->width;
    int y1 = y0 + bx->tile < cam->height ? y0 + bx->tile : cam->height;
    int pw = x1 - x0, ph = y1 - y0, p = pw * ph, K = bx->K, d = bx->d, nc = bx->ncols;
    TileAcc *acc = &bx->acc[ti];
    acc->n = 0; acc->uid = NULL; acc->sums = NULL; acc->cnt = NULL;

    IdSeq *ent = (IdSeq *)malloc((size_t)p * K * sizeof(IdSeq));
    double *cols = (double *)malloc((size_t)p * K * nc * sizeof(double));
    double *f_hat = (double *)malloc((size_t)d * sizeof(double));
    int n_ent = 0;
    for (int q = 0; q < p; ++q) {
        int gx = x0 + q % pw, gy = y0 + q / pw;
        size_t pix = (size_t)gy * cam->width + gx;
        const int32_t *pid = bx->ids + pix * K;
        const double *pz = bx->z + pix * K, *pc = bx->clos + pix * K;
        double ld = bx->log_denom[pix];
        const double *up = bx->upstream + pix * d;
        int any = 0;
        for (int k = 0; k < K; ++k) any |= pid[k] >= 0;
        if (!any) continue;
        OrRay ry;
        pixel_ray(cam, gx, gy, &ry);
        double w_bg = exp(bx->eps / bx->gamma - ld);
        for (int i = 0; i < d; ++i) f_hat[i] = 0.0;
        for (int k = 0; k < K; ++k) { /* grad.py:103-108 */
            if (pid[k] < 0) continue;
            double o = clampd(bx->opacity[pid[k]], 0.0, 1.0);
            double wgt = o * pc[k] * exp(o * pz[k] / bx->gamma - ld);
            const double *f = bx->feature + (size_t)pid[k] * d;
            for (int i = 0; i < d; ++i) f_hat[i] += wgt * f[i];
        }
        for (int i = 0; i < d; ++i) f_hat[i] += w_bg * bx->background[i];
        for (int k = 0; k < K; ++k) {
            if (pid[k] < 0) continue;
            hit_gradient(bx, &ry, pid[k], pz[k], pc[k], ld, up, f_hat, cols + (size_t)n_ent * nc);
            ent[n_ent].id = pid[k]; ent[n_ent].seq = n_ent;
            n_ent++;
        }
    }
    if (n_ent > 0) { /* grad.py:231-234: unique + add.at in pixel-major order */
        qsort(ent, (size_t)n_ent, sizeof(IdSeq), cmp_idseq);
        int nu = 0;
        for (int i = 0; i < n_ent; ++i) if (i == 0 || ent[i].id != ent[i - 1].id) nu++;
        acc->n = nu;
        acc->uid = (int32_t *)malloc((size_t)nu * sizeof(int32_t));
        acc->sums = (double *)calloc((size_t)nu * nc, sizeof(double));
        acc->cnt = (int64_t *)calloc((size_t)nu, sizeof(int64_t));
        int u = -1;
        for (int i = 0; i < n_ent; ++i) {
            if (i == 0 || ent[i].id != ent[i - 1].id) { u++; acc->uid[u] = ent[i].id; }
            const double *col = cols + (size_t)ent[i].seq * nc;
            for (int j = 0; j < nc; ++j) acc->sums[(size_t)u * nc + j] += col[j];
            acc->cnt[u] += 1;
        }
    }
    free(ent); free(cols); free(f_hat);
}

/* Outputs: d_pos (M,3), d_rad, d_opa, d_feat (M,d), pixel_count (M) int64,
 * d_t[3], G[9] (= grad_rot_matrix, d loss / d R, row-major), d_focal, d_sensor.
 * The rotation-parameter VJP (camera.py:57-117) is host math in oracle.py. */
int or_render_backward(int64_t m, int d, const double *pos, const double *rad, const double *opa,
                       const double *feat, const double *bg, const OrCamera *cam, double gamma,
                       double eps, int K, const int32_t *ids, const double *z, const double *clos,
                       const double *log_denom, const double *upstream, int normalize, int gate,
                       int tile, int threads, double *d_pos, double *d_rad, double *d_opa,
                       double *d_feat, int64_t *pixel_count, double *d_t, double *G,
                       double *d_focal, double *d_sensor) {
    int ntx = (cam->width + tile - 1) / tile, nty = (cam->height + tile - 1) / tile;
    int64_t n_tiles = (int64_t)ntx * nty;
    int nc = 3 + 1 + 1 + d + 2;
    size_t mm = (size_t)(m > 0 ? m : 1);
    int64_t *x_min = malloc(mm * 8), *x_max = malloc(mm * 8), *y_min = malloc(mm * 8), *y_max = malloc(mm * 8);
    uint8_t *on = malloc(mm);
    double *proj_r = malloc(mm * 8), *cc = malloc(mm * 24), *earliest = malloc(mm * 8);
    or_compute_bounds(m, pos, rad, cam, x_min, x_max, y_min, y_max, on, proj_r, cc, earliest);

    TileAcc *acc = (TileAcc *)calloc((size_t)n_tiles, sizeof(TileAcc));
    BwdCtx bx = {m, d, K, tile, ntx, nty, nc, cc, rad, opa, feat, bg, cam, gamma, eps,
                 ids, z, clos, log_denom, upstream, acc};
    if (threads < 1) threads = 1;
#pragma omp parallel for schedule(dynamic, 4) num_threads(threads)
    for (int64_t ti = 0; ti < n_tiles; ++ti) backward_tile(&bx, (int)ti);

    double *total = (double *)calloc(mm * nc, sizeof(double));
    memset(pixel_count, 0, (size_t)m * sizeof(int64_t));
    for (int64_t ti = 0; ti < n_tiles; ++ti) { /* grad.py:243-250 fixed tile order */
        TileAcc *a = &acc[ti];
        for (int u = 0; u < a->n; ++u) {
            int32_t id = a->uid[u];
            for (int j = 0; j < nc; ++j) total[(size_t)id * nc + j] += a->sums[(size_t)u * nc + j];
            pixel_count[id] += a->cnt[u];
        }
        free(a->uid); free(a->sums); free(a->cnt);
    }
    free(acc);

    /* grad.py:262-302 */
    const double *R = cam->R;
    double sc_sum[3] = {0, 0, 0}, GG[9] = {0}, gf = 0.0, gs = 0.0;
    for (int64_t i = 0; i < m; ++i) {
        const double *row = total + (size_t)i * nc;
        double div = 1.0, cam_scale = 1.0;
        if (normalize) {
            div = (double)(pixel_count[i] > 1 ? pixel_count[i] : 1);
            double area = M_PI * (proj_r[i] * proj_r[i]);
            if (area < 1.0) area = 1.0;
            cam_scale = 1e-3 / area;
        }
        /* d_position = (center_grad @ rot) / div : row vector times R */
        for (int j = 0; j < 3; ++j)
            d_pos[3 * i + j] = (row[0] * R[0 + j] + row[1] * R[3 + j] + row[2] * R[6 + j]) / div;
        d_rad[i] = row[3] / div;
        d_opa[i] = row[4] / div;
        for (int k = 0; k < d; ++k) d_feat[(size_t)i * d + k] = row[5 + k] / div;
        double sc[3] = {cam_scale * row[0], cam_scale * row[1], cam_scale * row[2]};
        double rel[3] = {pos[3 * i] - cam->t[0], pos[3 * i + 1] - cam->t[1], pos[3 * i + 2] - cam->t[2]};
        for (int a = 0; a < 3; ++a) {
            sc_sum[a] += sc[a];
            for (int b = 0; b < 3; ++b) GG[3 * a + b] += sc[a] * rel[b];
        }
        gf += cam_scale * row[5 + d];
        gs += cam_scale * row[6 + d];
        if (gate && proj_r[i] <= OR_GATE_RADIUS_PX) { /* grad.py:305-320 */
            d_pos[3 * i] = d_pos[3 * i + 1] = d_pos[3 * i + 2] = 0.0;
            d_rad[i] = 0.0;
        }
    }
    for (int j = 0; j < 3; ++j)
        d_t[j] = -(sc_sum[0] * R[0 + j] + sc_sum[1] * R[3 + j] + sc_sum[2] * R[6 + j]);
    for (int j = 0; j < 9; ++j) G[j] = GG[j];
    *d_focal = gf; *d_sensor = gs;
    free(total); free(x_min); free(x_max); free(y_min); free(y_max); free(on); free(proj_r);
    free(cc); free(earliest);
    return 0;
}

int or_num_threads_available(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
