/*
 * synth.c -- input fixtures for the bench configs: a
 * deep_street-style corridor scene at arbitrary scale, the LOD level
 * selection proxy, and radius-offset chunk active sets.
 *
 * Restates the value laws of reference src/synthetic.py:81-171 (structure
 * grid, three fine-clutter bands, 40 furniture blobs, SH dc from colour,
 * rest N(0, 0.02)) with a counter-based RNG (splitmix64 of seed, stream,
 * index) so any thread count gives bit-identical output; the random numbers
 * differ from NumPy's generator, the laws do not.  Active sets restate
 * select_active / build_chunk_active_sets (src/lod.py:194-213,
 * src/chunks.py:122-135) in fp64 with NumPy's norm order.
 *
 * Bench/test infrastructure: produces inputs for both the GPU arm and the
 * CPU reference arm; it is not part of the render path.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

typedef struct { uint64_t s; } rng_t;
static inline rng_t rng_at(uint64_t seed, uint64_t stream, uint64_t idx) {
  rng_t r;
  r.s = mix64(seed ^ mix64(stream * 0x632be59bd9b4e019ull ^ mix64(idx)));
  return r;
}
static inline double unif(rng_t *r) {  /* [0, 1) */
  r->s = mix64(r->s);
  return (double)(r->s >> 11) * (1.0 / 9007199254740992.0);
}
static inline double unif_ab(rng_t *r, double a, double b) { return a + (b - a) * unif(r); }
static inline double normal(rng_t *r, double mu, double sd) {
  double u1 = unif(r), u2 = unif(r);
  if (u1 < 1e-300) u1 = 1e-300;
  return mu + sd * sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}
static inline double clampd(double x, double lo, double hi) { return x < lo ? lo : (x > hi ? hi : x); }

static const double C0 = 0.28209479177387814;

static void region_color(double z, double length, double c[3]) {
  double t = z / length;
  c[0] = clampd(0.35 + 0.3 * sin(6.0 * t), 0.05, 0.95);
  c[1] = clampd(0.35 + 0.25 * cos(9.0 * t), 0.05, 0.95);
  c[2] = clampd(0.40 + 0.2 * sin(4.0 * t + 1.0), 0.05, 0.95);
}

static void random_quat(rng_t *r, double q[4]) { /* Shoemake, (w, x, y, z) */
  double u1 = unif(r), u2 = unif(r), u3 = unif(r);
  double a = sqrt(1.0 - u1), b = sqrt(u1);
  q[0] = a * sin(6.283185307179586 * u2);
  q[1] = a * cos(6.283185307179586 * u2);
  q[2] = b * sin(6.283185307179586 * u3);
  q[3] = b * cos(6.283185307179586 * u3);
}

#define N_GROUND (220 * 9)
#define N_WALL (220 * 6)
#define N_BLOBS 40
#define BLOB_M 25

int64_t synth_count(int64_t n_fine) {
  return N_GROUND + 2 * N_WALL + 3 * (n_fine / 3) + N_BLOBS * BLOB_M;
}

static void put(float *geom, float *sh, int terms, int64_t i, const double p[3], const double s[3],
                const double q[4], double op, const double col[3], rng_t *r) {
  float *g = geom + 12 * i;
  g[0] = (float)p[0]; g[1] = (float)p[1]; g[2] = (float)p[2];
  g[3] = (float)s[0]; g[4] = (float)s[1]; g[5] = (float)s[2];
  g[6] = (float)q[0]; g[7] = (float)q[1]; g[8] = (float)q[2]; g[9] = (float)q[3];
  g[10] = (float)clampd(op, 0.0, 1.0);
  g[11] = 0.0f;
  float *k = sh + (int64_t)3 * terms * i;
  for (int c = 0; c < 3; ++c) {
    k[c * terms] = (float)((col[c] - 0.5) / C0);
    for (int t = 1; t < terms; ++t) k[c * terms + t] = (float)normal(r, 0.0, 0.02);
  }
}

/* Scene: geom (N,12) fp32 [mean, scale, rot wxyz, opacity, fv=0];
 * sh (N,3,(deg+1)^2) fp32.  N = synth_count(n_fine). */
void synth_street(uint64_t seed, int64_t n_fine, double length, int32_t degree, float *geom,
                  float *sh) {
  const int terms = (degree + 1) * (degree + 1);
  const double half_w = 6.0, ground_y = -2.0, wall_top = 6.0;
  const int64_t n_each = n_fine / 3;
  const int64_t o_wall = N_GROUND, o_fine = N_GROUND + 2 * N_WALL;
  const int64_t o_blob = o_fine + 3 * n_each;
  const double s2 = 0.7071067811865476;
  /* structure: ground (normal +y) and two walls (normal -+x) */
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < N_GROUND + 2 * N_WALL; ++i) {
    rng_t r = rng_at(seed, 1, (uint64_t)i);
    double p[3], s[3], q[4], col[3];
    int64_t k;
    int nl;
    double side = 0.0;
    if (i < N_GROUND) { k = i; nl = 9; }
    else { k = (i - o_wall) % N_WALL; nl = 6; side = (i - o_wall) < N_WALL ? -1.0 : 1.0; }
    double zz = 1.0 + (length - 1.0) * (double)(k / nl) / 219.0;
    double ll = (double)(k % nl) / (double)(nl - 1);
    if (i < N_GROUND) {
      p[0] = -half_w + 2 * half_w * ll; p[1] = ground_y; p[2] = zz;
      q[0] = s2; q[1] = -s2; q[2] = 0; q[3] = 0;
    } else {
      p[0] = side * half_w; p[1] = ground_y + (wall_top - ground_y) * ll; p[2] = zz;
      q[0] = s2; q[1] = 0; q[2] = -side * s2; q[3] = 0;
    }
    for (int d = 0; d < 3; ++d) p[d] += normal(&r, 0.0, 0.18);
    double t = exp(unif_ab(&r, log(0.7), log(1.1)));
    s[0] = t * unif_ab(&r, 0.7, 1.3); s[1] = t * unif_ab(&r, 0.7, 1.3); s[2] = t * 0.25;
    double op = unif_ab(&r, 0.85, 0.98);
    if (i < N_GROUND) {
      const double base[3] = {0.38, 0.36, 0.35};
      for (int c = 0; c < 3; ++c) col[c] = clampd(base[c] + normal(&r, 0.0, 0.06), 0.02, 1.5);
    } else {
      region_color(zz, length, col);
      for (int c = 0; c < 3; ++c) col[c] += normal(&r, 0.0, 0.05);
    }
    put(geom, sh, terms, i, p, s, q, op, col, &r);
  }
  /* fine clutter: three bands */
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < 3 * n_each; ++i) {
    const int band = (int)(i / n_each);
    rng_t r = rng_at(seed, 2, (uint64_t)i);
    double p[3], s[3], q[4], col[3], base[3];
    double z = length * pow(unif(&r), 0.8);
    if (band == 0) {
      p[0] = unif_ab(&r, -5.0, 5.0); p[1] = unif_ab(&r, ground_y + 0.05, ground_y + 0.9);
      base[0] = 0.38; base[1] = 0.36; base[2] = 0.35;
    } else {
      double side = band == 1 ? -1.0 : 1.0;
      p[0] = side * unif_ab(&r, 3.2, half_w - 0.2); p[1] = unif_ab(&r, ground_y + 0.1, 4.5);
      region_color(z, length, base);
    }
    p[2] = z;
    double size = exp(unif_ab(&r, log(0.04), log(0.8)));
    for (int d = 0; d < 3; ++d) s[d] = size * unif_ab(&r, 0.6, 1.4);
    random_quat(&r, q);
    double op = unif_ab(&r, 0.5, 0.95);
    for (int c = 0; c < 3; ++c) col[c] = clampd(base[c] + normal(&r, 0.0, 0.07), 0.02, 1.2);
    put(geom, sh, terms, o_fine + i, p, s, q, op, col, &r);
  }
  /* street furniture blobs */
  for (int b = 0; b < N_BLOBS; ++b) {
    rng_t rb = rng_at(seed, 3, (uint64_t)b);
    double sx = unif_ab(&rb, 2.0, 4.5) * (unif(&rb) < 0.5 ? -1.0 : 1.0);
    double c[3] = {sx, unif_ab(&rb, -1.5, 1.0), unif_ab(&rb, 4.0, length - 5.0)};
    double bc[3] = {unif_ab(&rb, 0.1, 0.9), unif_ab(&rb, 0.1, 0.9), unif_ab(&rb, 0.1, 0.9)};
    for (int m = 0; m < BLOB_M; ++m) {
      rng_t r = rng_at(seed, 4, (uint64_t)(b * BLOB_M + m));
      double p[3], s[3], q[4], col[3];
      for (int d = 0; d < 3; ++d) p[d] = c[d] + normal(&r, 0.0, 0.5);
      for (int d = 0; d < 3; ++d) s[d] = exp(unif_ab(&r, log(0.08), log(0.3)));
      random_quat(&r, q);
      double op = unif_ab(&r, 0.5, 0.95);
      for (int d = 0; d < 3; ++d) col[d] = clampd(bc[d] + normal(&r, 0.0, 0.08), 0.02, 1.2);
      put(geom, sh, terms, o_blob + b * BLOB_M + m, p, s, q, op, col, &r);
    }
  }
}

/* ------------------------------------------------------------------------
 * Config 4: a Zip-NeRF-style indoor room, 40 x 30 x 4 m
 * (x in [-20, 20], z in [-15, 15], floor y = 0, ceiling y = 4), with
 * deep_street's value laws (src/synthetic.py:81-171): a structure layer of
 * oriented surface splats on jittered grids (floor, ceiling, four walls),
 * three bands of multi-scale fine clutter (floor, along the walls, ceiling
 * fixtures) whose colours track the local structure colour, and furniture
 * blobs on the floor.  Not in the reference: a new seeded generator.
 * ------------------------------------------------------------------------ */
#define RX 20.0
#define RZ 15.0
#define RH 4.0
#define R_FLOOR_NX 81
#define R_FLOOR_NZ 61
#define R_WALL_NH 9
#define R_N_FLOOR (R_FLOOR_NX * R_FLOOR_NZ)
#define R_N_WALLX (R_FLOOR_NX * R_WALL_NH) /* walls z = -+RZ, along x */
#define R_N_WALLZ (R_FLOOR_NZ * R_WALL_NH) /* walls x = -+RX, along z */
#define R_N_STRUCT (2 * R_N_FLOOR + 2 * R_N_WALLX + 2 * R_N_WALLZ)
#define R_N_BLOBS 60

int64_t synth_room_count(int64_t n_fine) {
  return R_N_STRUCT + 3 * (n_fine / 3) + R_N_BLOBS * BLOB_M;
}

static void room_color(double x, double z, double c[3]) {
  const double u = (x + RX) / (2 * RX), v = (z + RZ) / (2 * RZ);
  c[0] = clampd(0.45 + 0.25 * sin(5.0 * u + 0.3), 0.05, 0.95);
  c[1] = clampd(0.40 + 0.20 * cos(7.0 * v), 0.05, 0.95);
  c[2] = clampd(0.38 + 0.22 * sin(3.0 * (u + v) + 1.0), 0.05, 0.95);
}

void synth_room(uint64_t seed, int64_t n_fine, int32_t degree, float *geom, float *sh) {
  const int terms = (degree + 1) * (degree + 1);
  const int64_t n_each = n_fine / 3;
  const int64_t o_fine = R_N_STRUCT, o_blob = o_fine + 3 * n_each;
  const double s2 = 0.7071067811865476;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < R_N_STRUCT; ++i) {
    rng_t r = rng_at(seed, 11, (uint64_t)i);
    double p[3], s[3], q[4], col[3];
    int64_t k = i;
    int part;  /* 0 floor, 1 ceiling, 2/3 walls z = -+RZ, 4/5 walls x = -+RX */
    if (k < R_N_FLOOR) part = 0;
    else if ((k -= R_N_FLOOR) < R_N_FLOOR) part = 1;
    else if ((k -= R_N_FLOOR) < 2 * R_N_WALLX) { part = 2 + (int)(k / R_N_WALLX); k %= R_N_WALLX; }
    else { k -= 2 * R_N_WALLX; part = 4 + (int)(k / R_N_WALLZ); k %= R_N_WALLZ; }
    if (part <= 1) {
      const double x = -RX + 2 * RX * (double)(k / R_FLOOR_NZ) / (R_FLOOR_NX - 1);
      const double z = -RZ + 2 * RZ * (double)(k % R_FLOOR_NZ) / (R_FLOOR_NZ - 1);
      p[0] = x; p[1] = part == 0 ? 0.0 : RH; p[2] = z;
      q[0] = s2; q[1] = part == 0 ? -s2 : s2; q[2] = 0; q[3] = 0;  /* normal -+y */
    } else if (part <= 3) {
      const double x = -RX + 2 * RX * (double)(k / R_WALL_NH) / (R_FLOOR_NX - 1);
      const double y = RH * (double)(k % R_WALL_NH) / (R_WALL_NH - 1);
      p[0] = x; p[1] = y; p[2] = part == 2 ? -RZ : RZ;
      q[0] = 1; q[1] = 0; q[2] = 0; q[3] = 0;  /* thin along z: normal -+z */
    } else {
      const double z = -RZ + 2 * RZ * (double)(k / R_WALL_NH) / (R_FLOOR_NZ - 1);
      const double y = RH * (double)(k % R_WALL_NH) / (R_WALL_NH - 1);
      p[0] = part == 4 ? -RX : RX; p[1] = y; p[2] = z;
      q[0] = s2; q[1] = 0; q[2] = s2; q[3] = 0;  /* thin along x */
    }
    for (int d = 0; d < 3; ++d) p[d] += normal(&r, 0.0, 0.18);
    const double t = exp(unif_ab(&r, log(0.35), log(0.55)));
    s[0] = t * unif_ab(&r, 0.7, 1.3); s[1] = t * unif_ab(&r, 0.7, 1.3); s[2] = t * 0.25;
    const double op = unif_ab(&r, 0.85, 0.98);
    room_color(p[0], p[2], col);
    for (int c = 0; c < 3; ++c) col[c] = clampd(col[c] + normal(&r, 0.0, 0.06), 0.02, 1.5);
    put(geom, sh, terms, i, p, s, q, op, col, &r);
  }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < 3 * n_each; ++i) {
    const int band = (int)(i / n_each);
    rng_t r = rng_at(seed, 12, (uint64_t)i);
    double p[3], s[3], q[4], col[3];
    if (band == 0) {  /* floor clutter */
      p[0] = unif_ab(&r, -RX + 0.3, RX - 0.3); p[1] = unif_ab(&r, 0.05, 0.9);
      p[2] = unif_ab(&r, -RZ + 0.3, RZ - 0.3);
    } else if (band == 1) {  /* along the walls, 0.2 .. 2.8 m in */
      const double u = unif(&r) * 2.0 * (2 * RX + 2 * RZ), in = unif_ab(&r, 0.2, 2.8);
      if (u < 2 * RX) { p[0] = -RX + u; p[2] = -RZ + in; }
      else if (u < 4 * RX) { p[0] = -RX + (u - 2 * RX); p[2] = RZ - in; }
      else if (u < 4 * RX + 2 * RZ) { p[0] = -RX + in; p[2] = -RZ + (u - 4 * RX); }
      else { p[0] = RX - in; p[2] = -RZ + (u - 4 * RX - 2 * RZ); }
      p[1] = unif_ab(&r, 0.1, RH - 0.3);
    } else {  /* ceiling fixtures */
      p[0] = unif_ab(&r, -RX + 0.3, RX - 0.3); p[1] = unif_ab(&r, RH - 0.8, RH - 0.05);
      p[2] = unif_ab(&r, -RZ + 0.3, RZ - 0.3);
    }
    const double size = exp(unif_ab(&r, log(0.02), log(0.4)));
    for (int d = 0; d < 3; ++d) s[d] = size * unif_ab(&r, 0.6, 1.4);
    random_quat(&r, q);
    const double op = unif_ab(&r, 0.5, 0.95);
    room_color(p[0], p[2], col);
    for (int c = 0; c < 3; ++c) col[c] = clampd(col[c] + normal(&r, 0.0, 0.07), 0.02, 1.2);
    put(geom, sh, terms, o_fine + i, p, s, q, op, col, &r);
  }
  for (int b = 0; b < R_N_BLOBS; ++b) {
    rng_t rb = rng_at(seed, 13, (uint64_t)b);
    const double c[3] = {unif_ab(&rb, -RX + 2, RX - 2), unif_ab(&rb, 0.3, 1.1),
                         unif_ab(&rb, -RZ + 2, RZ - 2)};
    const double bc[3] = {unif_ab(&rb, 0.1, 0.9), unif_ab(&rb, 0.1, 0.9), unif_ab(&rb, 0.1, 0.9)};
    for (int m = 0; m < BLOB_M; ++m) {
      rng_t r = rng_at(seed, 14, (uint64_t)(b * BLOB_M + m));
      double p[3], s[3], q[4], col[3];
      for (int d = 0; d < 3; ++d) p[d] = c[d] + normal(&r, 0.0, 0.35);
      for (int d = 0; d < 3; ++d) s[d] = exp(unif_ab(&r, log(0.05), log(0.2)));
      random_quat(&r, q);
      const double op = unif_ab(&r, 0.5, 0.95);
      for (int d = 0; d < 3; ++d) col[d] = clampd(bc[d] + normal(&r, 0.0, 0.08), 0.02, 1.2);
      put(geom, sh, terms, o_blob + b * BLOB_M + m, p, s, q, op, col, &r);
    }
  }
}

/* LOD pruning proxy key: opacity * max(scale)^2. */
void synth_prune_key(const float *geom, int64_t n, float *key) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const float *g = geom + 12 * i;
    float m = g[3] > g[4] ? g[3] : g[4];
    m = m > g[5] ? m : g[5];
    key[i] = g[10] * m * m;
  }
}

/* Gather a level: rows idx of base geometry/SH with filter variance fv. */
void synth_gather_level(const float *geom, const float *sh, int32_t terms, const int64_t *idx,
                        int64_t n, float fv, float *out_geom, float *out_sh) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    memcpy(out_geom + 12 * i, geom + 12 * idx[i], 48);
    out_geom[12 * i + 11] = fv;
    memcpy(out_sh + (int64_t)3 * terms * i, sh + (int64_t)3 * terms * idx[i], 12 * terms);
  }
}

/* Distance-band membership of one level for K query points (chunk centres):
 * level l's set for chunk j is { i : lo[j] <= |mu_i - c_j| < hi[j] } with
 * the norm evaluated as sqrt((dx*dx + dy*dy) + dz*dz) in fp64 (NumPy order).
 * Pass 1 (out == NULL) counts into counts[K]; pass 2 fills out with the
 * sorted indices at offsets[j]. */
void synth_bands(const float *geom, int64_t n, const double *centers, int32_t K, const double *lo,
                 const double *hi, int64_t *counts, const int64_t *offsets, uint32_t *out) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int32_t j = 0; j < K; ++j) {
    const double cx = centers[3 * j], cy = centers[3 * j + 1], cz = centers[3 * j + 2];
    int64_t c = 0;
    uint32_t *dst = out ? out + offsets[j] : NULL;
    for (int64_t i = 0; i < n; ++i) {
      const float *g = geom + 12 * i;
      double dx = (double)g[0] - cx, dy = (double)g[1] - cy, dz = (double)g[2] - cz;
      double d = sqrt((dx * dx + dy * dy) + dz * dz);
      if (d >= lo[j] && d < hi[j]) {
        if (dst) dst[c] = (uint32_t)i;
        ++c;
      }
    }
    if (counts) counts[j] = c;
  }
}

void synth_set_threads(int32_t n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int32_t synth_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
