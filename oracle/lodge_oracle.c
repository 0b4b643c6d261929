/*
 * lodge_oracle.c -- CPU restatement of the reference `splatlod` per-frame
 * render path, in fp64, following NumPy's operation order.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker (or the reported CPU baseline).  The product path
 * (paper_2505_23158_b200/) never links or calls it.
 *
 * Parity is pinned: oracle/make_golden.py runs the reference in place
 * (/root/reference/pkg/src) and tests/test_oracle_golden.py checks this file
 * bit-for-bit against the committed vectors under tests/golden/.
 *
 * Operation order (measured on numpy 2.3.5 / OpenBLAS 0.3.30):
 *   - np.einsum with three operands: sequential over the summed indices in
 *     lexical order, each term ((a*b)*c), accumulator starting at 0.
 *   - add.reduce / prod over a length-3 axis: ((a+b)+c), ((a*b)*c).
 *   - BLAS matmul (N>=2 rows) and 1-D np.dot: fma(a2,b2,fma(a1,b1,a0*b0)).
 *   - every other ufunc: one correctly rounded IEEE op, no contraction.
 * Build with -ffp-contract=off (oracle/Makefile) so C never fuses on its own.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define TILE 16
#define SUPPORT_SIGMA 3.0
#define SUPPORT_Q 9.0 /* SUPPORT_SIGMA**2 * 2.0 * 0.5, src/raster.py:27 */

static const double SH_C0 = 0.28209479177387814;
static const double SH_C1 = 0.4886025119029199;
static const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
static const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

typedef struct {
  double R[9];      /* world->camera rotation, row-major (Camera.rotation_matrix) */
  double pos[3];    /* camera position */
  double fx, fy, cx, cy;
  int32_t w, h;
  double near_plane;
} orc_camera;

typedef struct {
  double alpha_clamp, alpha_min, t_min, dilation2d;
} orc_raster_cfg;

/* fma chain used by OpenBLAS dgemm / ddot for 3-term dot products. */
static inline double dot3_blas(const double *a, const double *b) {
  return fma(a[2], b[2], fma(a[1], b[1], a[0] * b[0]));
}

/* ---------------------------------------------------------------------- */
/* a4/a5: nearest_two_chunks + blend_factor (src/blending.py:77-99)        */
/* ---------------------------------------------------------------------- */
void orc_select(const double *centers, int32_t K, const double *pos, int32_t *f,
                int32_t *o, double *t_bar, double *t) {
  /* dist = np.linalg.norm(centers - c, axis=1) = sqrt((s0+s1)+s2) */
  int32_t b0 = -1, b1 = -1;
  double d0 = 0, d1 = 0;
  for (int32_t j = 0; j < K; ++j) {
    double x = centers[3 * j] - pos[0], y = centers[3 * j + 1] - pos[1], z = centers[3 * j + 2] - pos[2];
    double d = sqrt((x * x + y * y) + z * z);
    /* lexsort((arange, dist)): ascending dist, ties to the lower id */
    if (b0 < 0 || d < d0) {
      b1 = b0; d1 = d0; b0 = j; d0 = d;
    } else if (b1 < 0 || d < d1) {
      b1 = j; d1 = d;
    }
  }
  *f = b0;
  *o = (K > 1) ? b1 : -1;
  if (K > 1) {
    const double *mf = centers + 3 * b0, *mo = centers + 3 * b1;
    double fo[3] = {mf[0] - mo[0], mf[1] - mo[1], mf[2] - mo[2]};
    double co[3] = {pos[0] - mo[0], pos[1] - mo[1], pos[2] - mo[2]};
    double d2 = dot3_blas(fo, fo);
    double tb = dot3_blas(co, fo) / d2;
    *t_bar = tb;
    *t = fmin(1.0, fmax(0.0, tb)); /* min(1.0, max(0.0, t_bar)) */
  } else {
    *t_bar = 1.0;
    *t = 1.0;
  }
}

/* ---------------------------------------------------------------------- */
/* a6: compose_active per level (src/blending.py:119-128)                  */
/* union1d(a,b) + modulation {1 both, t only-a, 1-t only-b}.               */
/* Returns the union size.                                                 */
/* ---------------------------------------------------------------------- */
int64_t orc_union(const int64_t *a, int64_t na, const int64_t *b, int64_t nb, double t,
                  int64_t *out_idx, double *out_mod, int8_t *out_tag) {
  int64_t i = 0, j = 0, k = 0;
  const double omt = 1.0 - t;
  while (i < na || j < nb) {
    int64_t v;
    int8_t tag;
    if (j >= nb || (i < na && a[i] < b[j])) { v = a[i++]; tag = 1; }
    else if (i >= na || b[j] < a[i]) { v = b[j++]; tag = 2; }
    else { v = a[i]; ++i; ++j; tag = 3; }
    out_idx[k] = v;
    if (out_mod) out_mod[k] = (tag == 3) ? 1.0 : (tag == 1 ? t : omt);
    if (out_tag) out_tag[k] = tag;
    ++k;
  }
  return k;
}

/* ---------------------------------------------------------------------- */
/* a10: eval_sh for one splat (src/raster.py:136-173)                      */
/* coeffs: (3, terms) row-major.  NumPy evaluates per channel with the     */
/* operation order written in the source; we reproduce it term by term.    */
/* ---------------------------------------------------------------------- */
static void eval_sh1(const double *coeffs, int terms, int degree, double xs, double ys,
                     double zs, double *rgb) {
  double xx = 0, yy = 0, zz = 0, xy = 0, yz = 0, xz = 0;
  double b2[5] = {0}, b3[7] = {0};
  double c1y = SH_C1 * ys, c1z = SH_C1 * zs, c1x = SH_C1 * xs;
  if (degree >= 2) {
    xx = xs * xs; yy = ys * ys; zz = zs * zs;
    xy = xs * ys; yz = ys * zs; xz = xs * zs;
    b2[0] = SH_C2[0] * xy;
    b2[1] = SH_C2[1] * yz;
    b2[2] = SH_C2[2] * (((2 * zz) - xx) - yy);
    b2[3] = SH_C2[3] * xz;
    b2[4] = SH_C2[4] * (xx - yy);
  }
  if (degree >= 3) {
    b3[0] = SH_C3[0] * (ys * ((3 * xx) - yy));
    b3[1] = SH_C3[1] * (xy * zs);
    b3[2] = SH_C3[2] * (ys * (((4 * zz) - xx) - yy));
    b3[3] = SH_C3[3] * (zs * (((2 * zz) - (3 * xx)) - (3 * yy)));
    b3[4] = SH_C3[4] * (xs * (((4 * zz) - xx) - yy));
    b3[5] = SH_C3[5] * (zs * (xx - yy));
    b3[6] = SH_C3[6] * (xs * (xx - (3 * yy)));
  }
  for (int c = 0; c < 3; ++c) {
    const double *k = coeffs + c * terms;
    double out = SH_C0 * k[0];
    if (degree >= 1) {
      out = out - c1y * k[1];
      out = out + c1z * k[2];
      out = out - c1x * k[3];
      if (degree >= 2)
        for (int q = 0; q < 5; ++q) out = out + b2[q] * k[4 + q];
      if (degree >= 3)
        for (int q = 0; q < 7; ++q) out = out + b3[q] * k[9 + q];
    }
    out = out + 0.5;
    rgb[c] = out > 0.0 ? out : 0.0; /* np.maximum(out + 0.5, 0.0) */
    if (out != out) rgb[c] = out;   /* NaN propagates through np.maximum */
  }
}

/* ---------------------------------------------------------------------- */
/* a8: project_scene (src/raster.py:188-291) for one level.                */
/* Scene arrays are SoA fp64: means (N,3) scales (N,3) rots (N,4 wxyz)     */
/* opac (N) fv (N) sh (N,3,terms).  idx: n input indices; mod: n or NULL.  */
/* Outputs (capacity n): survivors in input order.  Returns M.             */
/* cov2d is (M,2,2) row-major, conic (M,3), extent (M,2).                  */
/* rect (M,4) = x0,x1,y0,y1 clipped tile ranges (src/raster.py:303-313).   */
/* ---------------------------------------------------------------------- */
int64_t orc_project(const double *means, const double *scales, const double *rots,
                    const double *opac, const double *fvar, const double *sh, int32_t degree,
                    const int64_t *idx, int64_t n, const double *mod, const orc_camera *cam,
                    const orc_raster_cfg *cfg, int32_t shade, int64_t *src, double *mean2d,
                    double *cov2d_out, double *conic, double *extent, double *depth,
                    double *opacity, double *color, int32_t *rect) {
  const int terms = (degree + 1) * (degree + 1);
  const double *W = cam->R;
  const double fx = cam->fx, fy = cam->fy, cx = cam->cx, cy = cam->cy;
  const int32_t w = cam->w, h = cam->h;
  const double lim_x = 1.3 * 0.5 * (double)w / fx;
  const double lim_y = 1.3 * 0.5 * (double)h / fy;
  const int32_t tiles_x = (w + TILE - 1) / TILE, tiles_y = (h + TILE - 1) / TILE;
  int64_t m = 0;
  for (int64_t e = 0; e < n; ++e) {
    const int64_t g = idx[e];
    const double *mu = means + 3 * g;
    double d[3] = {mu[0] - cam->pos[0], mu[1] - cam->pos[1], mu[2] - cam->pos[2]};
    /* cam_pts = (means - position) @ w2c.T  (BLAS dgemm) */
    double x = dot3_blas(d, W + 0), y = dot3_blas(d, W + 3), z = dot3_blas(d, W + 6);
    if (!(z > cam->near_plane)) continue;
    double mx = ((fx * x) / z) + cx, my = ((fy * y) / z) + cy;
    /* quat_to_matrix (src/scene.py:23-42) */
    const double *q = rots + 4 * g;
    double qw = q[0], qx = q[1], qy = q[2], qz = q[3];
    double r[9];
    r[0] = 1 - 2 * ((qy * qy) + (qz * qz));
    r[1] = 2 * ((qx * qy) - (qw * qz));
    r[2] = 2 * ((qx * qz) + (qw * qy));
    r[3] = 2 * ((qx * qy) + (qw * qz));
    r[4] = 1 - 2 * ((qx * qx) + (qz * qz));
    r[5] = 2 * ((qy * qz) - (qw * qx));
    r[6] = 2 * ((qx * qz) - (qw * qy));
    r[7] = 2 * ((qy * qz) + (qw * qx));
    r[8] = 1 - 2 * ((qx * qx) + (qy * qy));
    const double *sc = scales + 3 * g;
    double s2[3] = {sc[0] * sc[0], sc[1] * sc[1], sc[2] * sc[2]};
    /* cov_world = einsum("nij,nj,nkj->nik") + fv on the diagonal */
    double cw[9];
    for (int i = 0; i < 3; ++i)
      for (int k = 0; k < 3; ++k) {
        double acc = 0.0;
        for (int j = 0; j < 3; ++j) acc = acc + (r[3 * i + j] * s2[j]) * r[3 * k + j];
        cw[3 * i + k] = acc;
      }
    const double fv = fvar[g];
    cw[0] = cw[0] + fv; cw[4] = cw[4] + fv; cw[8] = cw[8] + fv;
    /* cov_cam = einsum("ij,njk,lk->nil", W, cw, W) */
    double cc[9];
    for (int i = 0; i < 3; ++i)
      for (int l = 0; l < 3; ++l) {
        double acc = 0.0;
        for (int j = 0; j < 3; ++j)
          for (int k = 0; k < 3; ++k) acc = acc + (W[3 * i + j] * cw[3 * j + k]) * W[3 * l + k];
        cc[3 * i + l] = acc;
      }
    /* Jacobian at the clamped evaluation point */
    double tx = x / z, ty = y / z;
    tx = tx < -lim_x ? -lim_x : (tx > lim_x ? lim_x : tx);
    ty = ty < -lim_y ? -lim_y : (ty > lim_y ? lim_y : ty);
    double jx = tx * z, jy = ty * z;
    double inv_z = 1.0 / z;
    double J[6] = {fx * inv_z, 0.0, ((-fx * jx) * inv_z) * inv_z,
                   0.0, fy * inv_z, ((-fy * jy) * inv_z) * inv_z};
    /* cov2d = einsum("nij,njk,nlk->nil", J, cc, J) */
    double c2[4];
    for (int i = 0; i < 2; ++i)
      for (int l = 0; l < 2; ++l) {
        double acc = 0.0;
        for (int j = 0; j < 3; ++j)
          for (int k = 0; k < 3; ++k) acc = acc + (J[3 * i + j] * cc[3 * j + k]) * J[3 * l + k];
        c2[2 * i + l] = acc;
      }
    double det_raw = c2[0] * c2[3] - c2[1] * c2[2];
    det_raw = det_raw > 0.0 ? det_raw : 0.0; /* np.maximum(det_raw, 0) */
    c2[0] = c2[0] + cfg->dilation2d;
    c2[3] = c2[3] + cfg->dilation2d;
    double det = c2[0] * c2[3] - c2[1] * c2[2];
    /* filter_opacity_factor (src/raster.py:176-185) */
    double ra = s2[0] / (s2[0] + fv), rb = s2[1] / (s2[1] + fv), rc = s2[2] / (s2[2] + fv);
    double op = opac[g] * sqrt((ra * rb) * rc);
    if (cfg->dilation2d > 0) op = op * sqrt(det_raw / det);
    if (mod) op = op * mod[e];
    double e0 = c2[0] > 0.0 ? c2[0] : 0.0, e1 = c2[3] > 0.0 ? c2[3] : 0.0;
    double ex = SUPPORT_SIGMA * sqrt(e0), ey = SUPPORT_SIGMA * sqrt(e1);
    int ok = det > 1e-12;
    ok = ok && (mx + ex > 0) && (mx - ex < (double)w);
    ok = ok && (my + ey > 0) && (my - ey < (double)h);
    if (!ok) continue;
    double inv_det = 1.0 / det;
    src[m] = e;
    mean2d[2 * m] = mx; mean2d[2 * m + 1] = my;
    if (cov2d_out) { cov2d_out[4 * m] = c2[0]; cov2d_out[4 * m + 1] = c2[1]; cov2d_out[4 * m + 2] = c2[2]; cov2d_out[4 * m + 3] = c2[3]; }
    conic[3 * m] = c2[3] * inv_det;
    conic[3 * m + 1] = (-c2[1]) * inv_det;
    conic[3 * m + 2] = c2[0] * inv_det;
    extent[2 * m] = ex; extent[2 * m + 1] = ey;
    depth[m] = z;
    opacity[m] = op;
    if (rect) {
      int64_t x0 = (int64_t)floor((mx - ex) / TILE), x1 = (int64_t)floor((mx + ex) / TILE);
      int64_t y0 = (int64_t)floor((my - ey) / TILE), y1 = (int64_t)floor((my + ey) / TILE);
      x0 = x0 < 0 ? 0 : (x0 > tiles_x - 1 ? tiles_x - 1 : x0);
      x1 = x1 < 0 ? 0 : (x1 > tiles_x - 1 ? tiles_x - 1 : x1);
      y0 = y0 < 0 ? 0 : (y0 > tiles_y - 1 ? tiles_y - 1 : y0);
      y1 = y1 < 0 ? 0 : (y1 > tiles_y - 1 ? tiles_y - 1 : y1);
      rect[4 * m] = (int32_t)x0; rect[4 * m + 1] = (int32_t)x1;
      rect[4 * m + 2] = (int32_t)y0; rect[4 * m + 3] = (int32_t)y1;
    }
    if (shade) {
      double dd0 = mu[0] - cam->pos[0], dd1 = mu[1] - cam->pos[1], dd2 = mu[2] - cam->pos[2];
      double nrm = sqrt((dd0 * dd0 + dd1 * dd1) + dd2 * dd2);
      eval_sh1(sh + (size_t)g * 3 * terms, terms, degree, dd0 / nrm, dd1 / nrm, dd2 / nrm,
               color + 3 * m);
    } else {
      color[3 * m] = color[3 * m + 1] = color[3 * m + 2] = 0.0;
    }
    ++m;
  }
  return m;
}

/* ---------------------------------------------------------------------- */
/* a14-a16: rasterize (src/raster.py:380-449)                              */
/* ---------------------------------------------------------------------- */
typedef struct {
  double depth;
  int64_t src;
  int64_t row;
} key_t_;

static int cmp_key(const void *pa, const void *pb) {
  const key_t_ *a = (const key_t_ *)pa, *b = (const key_t_ *)pb;
  if (a->depth < b->depth) return -1;
  if (a->depth > b->depth) return 1;
  if (a->src < b->src) return -1;
  if (a->src > b->src) return 1;
  return 0;
}

static void tile_range(double mx, double my, double ex, double ey, int32_t tiles_x,
                       int32_t tiles_y, int64_t *r) {
  int64_t x0 = (int64_t)floor((mx - ex) / TILE), x1 = (int64_t)floor((mx + ex) / TILE);
  int64_t y0 = (int64_t)floor((my - ey) / TILE), y1 = (int64_t)floor((my + ey) / TILE);
  r[0] = x0 < 0 ? 0 : (x0 > tiles_x - 1 ? tiles_x - 1 : x0);
  r[1] = x1 < 0 ? 0 : (x1 > tiles_x - 1 ? tiles_x - 1 : x1);
  r[2] = y0 < 0 ? 0 : (y0 > tiles_y - 1 ? tiles_y - 1 : y0);
  r[3] = y1 < 0 ? 0 : (y1 > tiles_y - 1 ? tiles_y - 1 : y1);
}

/* Returns P (number of tile-splat pairs), or -1 on allocation failure.
 * Optional outputs: tile_offsets (T+1) and tile_src (P, the source index of
 * each member, per-tile lists concatenated in tile order): these are the
 * "sorted per-tile lists" the GPU path must reproduce bit-exactly.  Pass
 * tile_src == NULL to only count. */
int64_t orc_rasterize(int64_t n_inputs, int64_t M, const int64_t *src, const double *mean2d,
                      const double *conic, const double *extent, const double *depth,
                      const double *opacity, const double *color, int32_t w, int32_t h,
                      const orc_raster_cfg *cfg, int32_t need_image, int32_t record_max,
                      double *image, int64_t *tile_count, int64_t *visible, double *maxw,
                      int64_t *tile_offsets, int64_t *tile_src, int64_t tile_src_cap) {
  const int32_t tiles_x = (w + TILE - 1) / TILE, tiles_y = (h + TILE - 1) / TILE;
  const int64_t T = (int64_t)tiles_x * tiles_y;
  if (need_image) memset(image, 0, sizeof(double) * (size_t)w * h * 3);
  memset(visible, 0, sizeof(int64_t) * (size_t)w * h);
  memset(tile_count, 0, sizeof(int64_t) * (size_t)T);
  if (record_max) memset(maxw, 0, sizeof(double) * (size_t)n_inputs);
  if (tile_offsets) memset(tile_offsets, 0, sizeof(int64_t) * (size_t)(T + 1));
  if (M == 0) return 0;

  key_t_ *keys = (key_t_ *)malloc(sizeof(key_t_) * (size_t)M);
  int64_t *rects = (int64_t *)malloc(sizeof(int64_t) * 4 * (size_t)M);
  if (!keys || !rects) { free(keys); free(rects); return -1; }
  for (int64_t i = 0; i < M; ++i) { keys[i].depth = depth[i]; keys[i].src = src[i]; keys[i].row = i; }
  qsort(keys, (size_t)M, sizeof(key_t_), cmp_key); /* np.lexsort((src, depth)) */
  int64_t P = 0;
  for (int64_t r = 0; r < M; ++r) {
    int64_t i = keys[r].row;
    tile_range(mean2d[2 * i], mean2d[2 * i + 1], extent[2 * i], extent[2 * i + 1], tiles_x, tiles_y, rects + 4 * r);
    int64_t *rr = rects + 4 * r;
    for (int64_t ty = rr[2]; ty <= rr[3]; ++ty)
      for (int64_t tx = rr[0]; tx <= rr[1]; ++tx) tile_count[ty * tiles_x + tx]++;
    P += (rr[1] - rr[0] + 1) * (rr[3] - rr[2] + 1);
  }
  int64_t *start = (int64_t *)malloc(sizeof(int64_t) * (size_t)(T + 1));
  int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)T);
  int64_t *members = (int64_t *)malloc(sizeof(int64_t) * (size_t)(P > 0 ? P : 1));
  if (!start || !fill || !members) { free(keys); free(rects); free(start); free(fill); free(members); return -1; }
  start[0] = 0;
  for (int64_t t = 0; t < T; ++t) start[t + 1] = start[t] + tile_count[t];
  memcpy(fill, start, sizeof(int64_t) * (size_t)T);
  /* duplication in global depth order == stable argsort by tile id */
  for (int64_t r = 0; r < M; ++r) {
    int64_t *rr = rects + 4 * r;
    for (int64_t ty = rr[2]; ty <= rr[3]; ++ty)
      for (int64_t tx = rr[0]; tx <= rr[1]; ++tx) members[fill[ty * tiles_x + tx]++] = r;
  }
  if (tile_offsets) memcpy(tile_offsets, start, sizeof(int64_t) * (size_t)(T + 1));
  if (tile_src && P <= tile_src_cap)
    for (int64_t p = 0; p < P; ++p) tile_src[p] = keys[members[p]].src;

  const double amin = cfg->alpha_min, aclamp = cfg->alpha_clamp, tmin = cfg->t_min;
  int64_t nthreads = 1;
#ifdef _OPENMP
  nthreads = omp_get_max_threads();
#endif
  /* per-thread max-weight scratch keeps the result independent of threads */
  double *maxw_t = NULL;
  if (record_max) {
    maxw_t = (double *)calloc((size_t)nthreads * (size_t)n_inputs, sizeof(double));
    if (!maxw_t) { free(keys); free(rects); free(start); free(fill); free(members); return -1; }
  }
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t t = 0; t < T; ++t) {
    int64_t tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    double *mw = record_max ? maxw_t + tid * n_inputs : NULL;
    const int32_t tx = (int32_t)(t % tiles_x), ty = (int32_t)(t / tiles_x);
    const int32_t px0 = tx * TILE, py0 = ty * TILE;
    const int32_t px1 = px0 + TILE < w ? px0 + TILE : w, py1 = py0 + TILE < h ? py0 + TILE : h;
    const int64_t b = start[t], e = start[t + 1];
    for (int32_t py = py0; py < py1; ++py)
      for (int32_t px = px0; px < px1; ++px) {
        const double gx = (double)px + 0.5, gy = (double)py + 0.5;
        double trans = 1.0, cp = 1.0, img0 = 0, img1 = 0, img2 = 0;
        double blk0 = 0, blk1 = 0, blk2 = 0;
        int64_t vis = 0;
        /* _composite_tile: blocks of 1024 members, cumprod within a block
         * (src/raster.py:346-373); reproduced so T_before is bit-exact. */
        for (int64_t k = b; k < e; ++k) {
          if (((k - b) & 1023) == 0 && k != b) {
            trans = cp * trans; cp = 1.0;
            img0 += blk0; img1 += blk1; img2 += blk2; blk0 = blk1 = blk2 = 0;
            if (!(trans >= tmin)) break;
          }
          const int64_t i = keys[members[k]].row;
          const double dx = gx - mean2d[2 * i], dy = gy - mean2d[2 * i + 1];
          const double *cn = conic + 3 * i;
          const double q = ((cn[0] * dx) * dx + ((2.0 * cn[1]) * dx) * dy) + (cn[2] * dy) * dy;
          double alpha = opacity[i] * exp(-0.5 * (q > 0.0 ? q : 0.0));
          alpha = alpha < aclamp ? alpha : aclamp;
          const int skipped = (alpha < amin) || (q > SUPPORT_Q);
          const double a = skipped ? 0.0 : alpha;
          const double before = cp * trans;
          cp = cp * (1.0 - a);
          if (before >= tmin) {
            const double wgt = before * a;
            if (need_image) {
              const double *c = color + 3 * i;
              blk0 += wgt * c[0]; blk1 += wgt * c[1]; blk2 += wgt * c[2];
            }
            if (!skipped) vis++;
            if (mw) { int64_t s = src[i]; if (wgt > mw[s]) mw[s] = wgt; }
          }
        }
        img0 += blk0; img1 += blk1; img2 += blk2;
        const size_t pix = (size_t)py * w + px;
        visible[pix] = vis;
        if (need_image) {
          image[3 * pix] = img0 < 0 ? 0 : (img0 > 1 ? 1 : img0);
          image[3 * pix + 1] = img1 < 0 ? 0 : (img1 > 1 ? 1 : img1);
          image[3 * pix + 2] = img2 < 0 ? 0 : (img2 > 1 ? 1 : img2);
        }
      }
  }
  if (record_max) {
    for (int64_t tt = 0; tt < nthreads; ++tt)
      for (int64_t s = 0; s < n_inputs; ++s)
        if (maxw_t[tt * n_inputs + s] > maxw[s]) maxw[s] = maxw_t[tt * n_inputs + s];
    free(maxw_t);
  }
  free(keys); free(rects); free(start); free(fill); free(members);
  return P;
}

/* Host threads of the OpenMP loops (the bench's CPU arm uses every core even
   when a launcher such as torchrun exported OMP_NUM_THREADS=1). */
void orc_set_threads(int32_t n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int32_t orc_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ---------------------------------------------------------------------- */
/* project_scene over fp32 AoS storage (the asset record layout,           */
/* src/assets.py:240-254: [mean3, scale3, rot4, opacity, fv] + sh), values  */
/* widened to fp64 exactly as the device's fp32 store does.  Parallel over  */
/* contiguous input chunks (each restated by orc_project), concatenated in  */
/* input order, so the result is independent of the thread count.          */
/* ---------------------------------------------------------------------- */
int64_t orc_project_f32(const float *geom, const float *sh, int32_t degree, const int64_t *idx,
                        int64_t n, const double *mod, const orc_camera *cam,
                        const orc_raster_cfg *cfg, int32_t shade, int64_t *src, double *mean2d,
                        double *cov2d_out, double *conic, double *extent, double *depth,
                        double *opacity, double *color, int32_t *rect) {
  const int terms = (degree + 1) * (degree + 1);
  const int64_t chunk = 8192;
  const int64_t nchunks = (n + chunk - 1) / chunk;
  int64_t *mc = (int64_t *)calloc((size_t)(nchunks > 0 ? nchunks : 1), sizeof(int64_t));
  if (!mc) return -1;
  int failed = 0;
  /* pass 1: survivors per chunk (outputs staged in place, compacted later) */
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t c = 0; c < nchunks; ++c) {
    const int64_t b = c * chunk, k = (b + chunk < n ? chunk : n - b);
    double *buf = (double *)malloc(sizeof(double) * (size_t)k * (12 + 3 * terms));
    int64_t *lidx = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
    if (!buf || !lidx) { failed = 1; free(buf); free(lidx); continue; }
    double *mu = buf, *sc = mu + 3 * k, *ro = sc + 3 * k, *op = ro + 4 * k, *fv = op + k,
           *shd = fv + k;
    for (int64_t i = 0; i < k; ++i) {
      const float *g = geom + 12 * idx[b + i];
      for (int d = 0; d < 3; ++d) { mu[3 * i + d] = g[d]; sc[3 * i + d] = g[3 + d]; }
      for (int d = 0; d < 4; ++d) ro[4 * i + d] = g[6 + d];
      op[i] = g[10];
      fv[i] = g[11];
      const float *s = sh + (int64_t)3 * terms * idx[b + i];
      for (int d = 0; d < 3 * terms; ++d) shd[(int64_t)3 * terms * i + d] = s[d];
      lidx[i] = i;
    }
    mc[c] = orc_project(mu, sc, ro, op, fv, shd, degree, lidx, k, mod ? mod + b : NULL, cam, cfg,
                        shade, src + b, mean2d + 2 * b, cov2d_out ? cov2d_out + 4 * b : NULL,
                        conic + 3 * b, extent + 2 * b, depth + b, opacity + b, color + 3 * b,
                        rect ? rect + 4 * b : NULL);
    for (int64_t i = 0; i < mc[c]; ++i) src[b + i] += b;
    free(buf);
    free(lidx);
  }
  if (failed) { free(mc); return -1; }
  /* pass 2: compact the chunks in input order */
  int64_t m = 0;
  for (int64_t c = 0; c < nchunks; ++c) {
    const int64_t b = c * chunk, k = mc[c];
    if (m != b && k > 0) {
      memmove(src + m, src + b, sizeof(int64_t) * k);
      memmove(mean2d + 2 * m, mean2d + 2 * b, sizeof(double) * 2 * k);
      if (cov2d_out) memmove(cov2d_out + 4 * m, cov2d_out + 4 * b, sizeof(double) * 4 * k);
      memmove(conic + 3 * m, conic + 3 * b, sizeof(double) * 3 * k);
      memmove(extent + 2 * m, extent + 2 * b, sizeof(double) * 2 * k);
      memmove(depth + m, depth + b, sizeof(double) * k);
      memmove(opacity + m, opacity + b, sizeof(double) * k);
      memmove(color + 3 * m, color + 3 * b, sizeof(double) * 3 * k);
      if (rect) memmove(rect + 4 * m, rect + 4 * b, sizeof(int32_t) * 4 * k);
    }
    m += k;
  }
  free(mc);
  return m;
}
