// K2: EWA projection with the Eq. 3 smoothing-filter opacity factor, 2-D
// dilation, culling and SH colour; one active Gaussian per thread and step
// (persistent CTAs), fp64 arithmetic in the reference's operation order
// (compiled with -fmad=false; every fma() below is one OpenBLAS places).
// The fused frame writes every output at the dense concatenated input index
// (culled inputs get depth key ~0 and leave in the depth sort's first pass),
// so the source index order -- the depth sort's tie order -- needs no
// compaction; the compat entry points (lodge_project, the cost
// table) compact survivors in input order with a decoupled look-back scan.
//
// Restates reference src/raster.py:188-291 (project_scene),
// src/raster.py:176-185 (filter_opacity_factor), src/raster.py:136-173
// (eval_sh), src/scene.py:23-42 (quat_to_matrix), src/raster.py:303-313
// (_tile_ranges) and src/lod.py:216-227 (project_selection, level-major).
#include <type_traits>

#include <algorithm>

#include "internal.cuh"

namespace lodge {

__device__ __constant__ double c_SH_C0 = 0.28209479177387814;
__device__ __constant__ double c_SH_C1 = 0.4886025119029199;
__device__ __constant__ double c_SH_C2[5] = {1.0925484305920792, -1.0925484305920792,
                                            0.31539156525252005, -1.0925484305920792,
                                            0.5462742152960396};
__device__ __constant__ double c_SH_C3[7] = {-0.5900435899266435, 2.890611442640554,
                                            -0.4570457994644658, 0.3731763325901154,
                                            -0.4570457994644658, 1.445305721320277,
                                            -0.5900435899266435};

struct Proj {
  double mx, my, z, ex, ey, op;
  double c00, c01, c10, c11, det;
  bool ok;
};

template <typename GT>
__device__ __forceinline__ void load_geom(const GT *__restrict__ g, double v[12]);

template <>
__device__ __forceinline__ void load_geom<double>(const double *__restrict__ g, double v[12]) {
  const double2 *p = reinterpret_cast<const double2 *>(g);
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    double2 t = __ldg(p + i);
    v[2 * i] = t.x;
    v[2 * i + 1] = t.y;
  }
}

template <>
__device__ __forceinline__ void load_geom<float>(const float *__restrict__ g, double v[12]) {
  const float4 *p = reinterpret_cast<const float4 *>(g);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    float4 t = __ldg(p + i);
    v[4 * i] = t.x;
    v[4 * i + 1] = t.y;
    v[4 * i + 2] = t.z;
    v[4 * i + 3] = t.w;
  }
}

// read_asset's load-time normalisation of the raw asset rotations
// (src/assets.py:275-278): q / np.linalg.norm(q), the norm summed in
// add.reduce's order over the length-4 row.
__device__ __forceinline__ void normalize_rot(double v[12]) {
  const double nn = sqrt(((v[6] * v[6] + v[7] * v[7]) + v[8] * v[8]) + v[9] * v[9]);
  v[6] = v[6] / nn;
  v[7] = v[7] / nn;
  v[8] = v[8] / nn;
  v[9] = v[9] / nn;
}

// Camera rotation patterns (bit 3i+j set: W_ij may be nonzero).  A term
// (W_ij * cw_jk) * W_lk of cov_cam = W cov_world W^T with W_ij = 0 or W_lk = 0
// is an exact zero for finite cov_world, and adding it to the running sum
// leaves the sum unchanged (up to the sign of an all-zero total, which
// compares equal), so the kernels drop those terms at compile time for
// cameras whose rotation has that zero pattern: the identity-orientation
// sweep (config 5) keeps 9 of the 81 terms, yaw-only cameras (config 4) 25.
enum : int { W_FULL = 0x1FF, W_IDENT = 0x111, W_YAW = 0x155 };

__device__ __forceinline__ int camera_wpattern(const lodge_camera &cam) {
  int m = 0;
#pragma unroll
  for (int i = 0; i < 9; ++i) m |= (cam.R[i] != 0.0) ? (1 << i) : 0;
  if ((m & ~W_IDENT) == 0) return W_IDENT;
  if ((m & ~W_YAW) == 0) return W_YAW;
  return W_FULL;
}

__device__ __forceinline__ bool all_finite9(const double c[9]) {
  bool ok = true;
#pragma unroll
  for (int i = 0; i < 9; ++i) ok = ok && isfinite(c[i]);
  return ok;
}

// The camera's clamp limits on x/z, y/z (src/raster.py:230-231), per
// camera: computed once per CTA in the frame kernels (the same fp64
// expression, so the same bits).
struct CamLims {
  double x, y;
};
__host__ __device__ inline CamLims cam_lims(const lodge_camera &cam) {
  return CamLims{1.3 * 0.5 * (double)cam.w / cam.fx, 1.3 * 0.5 * (double)cam.h / cam.fy};
}

// v: [mean3, scale3, rot4 wxyz, opacity, fv]
template <int WM = W_FULL>
__device__ __forceinline__ Proj project_core(const double v[12], const lodge_camera &cam,
                                             const lodge_raster_params &rp, double mod,
                                             bool has_mod, const CamLims &lim) {
  Proj p;
  p.ok = false;
  const double *W = cam.R;
  const double d0 = v[0] - cam.pos[0], d1 = v[1] - cam.pos[1], d2 = v[2] - cam.pos[2];
  const double x = fma(d2, W[2], fma(d1, W[1], d0 * W[0]));
  const double y = fma(d2, W[5], fma(d1, W[4], d0 * W[3]));
  const double z = fma(d2, W[8], fma(d1, W[7], d0 * W[6]));
  p.z = z;
  if (!(z > cam.near_plane)) return p;
  const double fx = cam.fx, fy = cam.fy;
  p.mx = ((fx * x) / z) + cam.cx;
  p.my = ((fy * y) / z) + cam.cy;
  const double qw = v[6], qx = v[7], qy = v[8], qz = v[9];
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
  const double s2[3] = {v[3] * v[3], v[4] * v[4], v[5] * v[5]};
  const double fv = v[11];
  double cw[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < 3; ++j) acc = acc + (r[3 * i + j] * s2[j]) * r[3 * k + j];
      cw[3 * i + k] = acc;
    }
  cw[0] = cw[0] + fv;
  cw[4] = cw[4] + fv;
  cw[8] = cw[8] + fv;
  double cc[9];
  if (WM == W_FULL || !all_finite9(cw)) {  // 0 * inf would be a NaN term: keep them all
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
          for (int k = 0; k < 3; ++k) acc = acc + (W[3 * i + j] * cw[3 * j + k]) * W[3 * l + k];
        cc[3 * i + l] = acc;
      }
  } else {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          if (!((WM >> (3 * i + j)) & 1)) continue;
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            if (!((WM >> (3 * l + k)) & 1)) continue;
            acc = acc + (W[3 * i + j] * cw[3 * j + k]) * W[3 * l + k];
          }
        }
        cc[3 * i + l] = acc;
      }
  }
  const double lim_x = lim.x, lim_y = lim.y;
  double tx = x / z, ty = y / z;
  tx = tx < -lim_x ? -lim_x : (tx > lim_x ? lim_x : tx);
  ty = ty < -lim_y ? -lim_y : (ty > lim_y ? lim_y : ty);
  const double jx = tx * z, jy = ty * z;
  const double inv_z = 1.0 / z;
  const double J00 = fx * inv_z, J02 = ((-fx * jx) * inv_z) * inv_z;
  const double J11 = fy * inv_z, J12 = ((-fy * jy) * inv_z) * inv_z;
  // cov2d = einsum("nij,njk,nlk->nil", J, cc, J); J01 = J10 = 0 terms add
  // exact zeros, so only the (j,k) in {i,2}x{l,2} terms are kept, in order.
  const double Jr[2][3] = {{J00, 0.0, J02}, {0.0, J11, J12}};
  double c2[4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int l = 0; l < 2; ++l) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        if (j != i && j != 2) continue;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          if (k != l && k != 2) continue;
          acc = acc + (Jr[i][j] * cc[3 * j + k]) * Jr[l][k];
        }
      }
      c2[2 * i + l] = acc;
    }
  double det_raw = c2[0] * c2[3] - c2[1] * c2[2];
  det_raw = det_raw > 0.0 ? det_raw : 0.0;
  c2[0] = c2[0] + rp.dilation2d;
  c2[3] = c2[3] + rp.dilation2d;
  const double det = c2[0] * c2[3] - c2[1] * c2[2];
  const double ra = s2[0] / (s2[0] + fv), rb = s2[1] / (s2[1] + fv), rc = s2[2] / (s2[2] + fv);
  double op = v[10] * sqrt((ra * rb) * rc);
  if (rp.dilation2d > 0) op = op * sqrt(det_raw / det);
  if (has_mod) op = op * mod;
  const double e0 = c2[0] > 0.0 ? c2[0] : 0.0, e1 = c2[3] > 0.0 ? c2[3] : 0.0;
  const double ex = 3.0 * sqrt(e0), ey = 3.0 * sqrt(e1);
  bool ok = det > 1e-12;
  ok = ok && (p.mx + ex > 0) && (p.mx - ex < (double)cam.w);
  ok = ok && (p.my + ey > 0) && (p.my - ey < (double)cam.h);
  p.ex = ex;
  p.ey = ey;
  p.op = op;
  p.c00 = c2[0];
  p.c01 = c2[1];
  p.c10 = c2[2];
  p.c11 = c2[3];
  p.det = det;
  p.ok = ok;
  return p;
}

// project_core for the camera's rotation zero pattern (uniform per camera).
__device__ __forceinline__ Proj project_any(const double v[12], const lodge_camera &cam,
                                            const lodge_raster_params &rp, double mod,
                                            bool has_mod, int wpat, const CamLims &lim) {
  if (wpat == W_IDENT) return project_core<W_IDENT>(v, cam, rp, mod, has_mod, lim);
  if (wpat == W_YAW) return project_core<W_YAW>(v, cam, rp, mod, has_mod, lim);
  return project_core<W_FULL>(v, cam, rp, mod, has_mod, lim);
}

// Coefficients of one record, (3, (DEG+1)^2), loaded with 16-byte vector
// loads when the record size allows it (fp32 SH1/SH3, fp64 SH1/SH3).
template <typename ST, int DEG>
__device__ __forceinline__ void load_sh(const ST *__restrict__ k, ST (&co)[3 * (DEG + 1) * (DEG + 1)]) {
  constexpr int N = 3 * (DEG + 1) * (DEG + 1);
  constexpr int PER = 16 / sizeof(ST);
  if constexpr ((N * sizeof(ST)) % 16 == 0) {
    using V = typename std::conditional<sizeof(ST) == 4, float4, double2>::type;
    const V *p = reinterpret_cast<const V *>(k);
#pragma unroll
    for (int i = 0; i < N / PER; ++i) {
      const V t = __ldg(p + i);
      const ST *ts = reinterpret_cast<const ST *>(&t);
#pragma unroll
      for (int e = 0; e < PER; ++e) co[i * PER + e] = ts[e];
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) co[i] = __ldg(k + i);
  }
}

// eval_sh (src/raster.py:136-173) with compile-time degree.
template <typename ST, int DEG>
__device__ __forceinline__ void eval_sh_t(const ST *__restrict__ k, double xs, double ys,
                                          double zs, double rgb[3]) {
  constexpr int T = (DEG + 1) * (DEG + 1);
  ST co[3 * T];
  load_sh<ST, DEG>(k, co);
  double b2[5], b3[7];
  const double c1y = c_SH_C1 * ys, c1z = c_SH_C1 * zs, c1x = c_SH_C1 * xs;
  if (DEG >= 2) {
    const double xx = xs * xs, yy = ys * ys, zz = zs * zs;
    const double xy = xs * ys, yz = ys * zs, xz = xs * zs;
    b2[0] = c_SH_C2[0] * xy;
    b2[1] = c_SH_C2[1] * yz;
    b2[2] = c_SH_C2[2] * (((2 * zz) - xx) - yy);
    b2[3] = c_SH_C2[3] * xz;
    b2[4] = c_SH_C2[4] * (xx - yy);
    if (DEG >= 3) {
      b3[0] = c_SH_C3[0] * (ys * ((3 * xx) - yy));
      b3[1] = c_SH_C3[1] * (xy * zs);
      b3[2] = c_SH_C3[2] * (ys * (((4 * zz) - xx) - yy));
      b3[3] = c_SH_C3[3] * (zs * (((2 * zz) - (3 * xx)) - (3 * yy)));
      b3[4] = c_SH_C3[4] * (xs * (((4 * zz) - xx) - yy));
      b3[5] = c_SH_C3[5] * (zs * (xx - yy));
      b3[6] = c_SH_C3[6] * (xs * (xx - (3 * yy)));
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const ST *kc = co + c * T;
    double out = c_SH_C0 * (double)kc[0];
    if (DEG >= 1) {
      out = out - c1y * (double)kc[1];
      out = out + c1z * (double)kc[2];
      out = out - c1x * (double)kc[3];
      if (DEG >= 2) {
#pragma unroll
        for (int q = 0; q < 5; ++q) out = out + b2[q] * (double)kc[4 + q];
      }
      if (DEG >= 3) {
#pragma unroll
        for (int q = 0; q < 7; ++q) out = out + b3[q] * (double)kc[9 + q];
      }
    }
    out = out + 0.5;
    rgb[c] = (out > 0.0 || out != out) ? out : 0.0;
  }
}

template <typename ST>
__device__ __forceinline__ void eval_sh_dev(const ST *__restrict__ k, int terms, int degree,
                                            const double v[12], const lodge_camera &cam,
                                            double rgb[3]) {
  const double dd0 = v[0] - cam.pos[0], dd1 = v[1] - cam.pos[1], dd2 = v[2] - cam.pos[2];
  const double nrm = sqrt((dd0 * dd0 + dd1 * dd1) + dd2 * dd2);
  const double xs = dd0 / nrm, ys = dd1 / nrm, zs = dd2 / nrm;
  switch (degree) {
    case 0: eval_sh_t<ST, 0>(k, xs, ys, zs, rgb); return;
    case 1: eval_sh_t<ST, 1>(k, xs, ys, zs, rgb); return;
    case 2: eval_sh_t<ST, 2>(k, xs, ys, zs, rgb); return;
    default: eval_sh_t<ST, 3>(k, xs, ys, zs, rgb); return;
  }
}

template <typename ST>
__device__ __forceinline__ void eval_sh_dev_scalar(const ST *__restrict__ k, int terms, int degree,
                                                   const double v[12], const lodge_camera &cam,
                                                   double rgb[3]) {
  const double dd0 = v[0] - cam.pos[0], dd1 = v[1] - cam.pos[1], dd2 = v[2] - cam.pos[2];
  const double nrm = sqrt((dd0 * dd0 + dd1 * dd1) + dd2 * dd2);
  const double xs = dd0 / nrm, ys = dd1 / nrm, zs = dd2 / nrm;
  double b2[5], b3[7];
  const double c1y = c_SH_C1 * ys, c1z = c_SH_C1 * zs, c1x = c_SH_C1 * xs;
  if (degree >= 2) {
    const double xx = xs * xs, yy = ys * ys, zz = zs * zs;
    const double xy = xs * ys, yz = ys * zs, xz = xs * zs;
    b2[0] = c_SH_C2[0] * xy;
    b2[1] = c_SH_C2[1] * yz;
    b2[2] = c_SH_C2[2] * (((2 * zz) - xx) - yy);
    b2[3] = c_SH_C2[3] * xz;
    b2[4] = c_SH_C2[4] * (xx - yy);
    if (degree >= 3) {
      b3[0] = c_SH_C3[0] * (ys * ((3 * xx) - yy));
      b3[1] = c_SH_C3[1] * (xy * zs);
      b3[2] = c_SH_C3[2] * (ys * (((4 * zz) - xx) - yy));
      b3[3] = c_SH_C3[3] * (zs * (((2 * zz) - (3 * xx)) - (3 * yy)));
      b3[4] = c_SH_C3[4] * (xs * (((4 * zz) - xx) - yy));
      b3[5] = c_SH_C3[5] * (zs * (xx - yy));
      b3[6] = c_SH_C3[6] * (xs * (xx - (3 * yy)));
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const ST *kc = k + c * terms;
    double out = c_SH_C0 * (double)__ldg(kc);
    if (degree >= 1) {
      out = out - c1y * (double)__ldg(kc + 1);
      out = out + c1z * (double)__ldg(kc + 2);
      out = out - c1x * (double)__ldg(kc + 3);
      if (degree >= 2)
        for (int q = 0; q < 5; ++q) out = out + b2[q] * (double)__ldg(kc + 4 + q);
      if (degree >= 3)
        for (int q = 0; q < 7; ++q) out = out + b3[q] * (double)__ldg(kc + 9 + q);
    }
    out = out + 0.5;
    rgb[c] = (out > 0.0 || out != out) ? out : 0.0;
  }
}

// Compositing payload from fp64 batch values (shared by K2 and the compat
// import).  q_eff folds both skip tests of src/raster.py:356 into one cut-off
// on q; tol bounds |q_fp32 - q_fp64| near that cut-off; both
// are stored as the scaled guard band [lo, hi] (internal.cuh Payload).
__device__ __forceinline__ void make_payload(double mx, double my, double A, double B, double C,
                                             double o, const double rgb[3], uint32_t src,
                                             double ex, double ey,
                                             const lodge_raster_params &rp, Payload &pl,
                                             Precise &pr) {
  pl.mx = mx;
  pl.my = my;
  pl.As = (float)(KQ * A);
  pl.B2s = (float)(KQ * (2.0 * B));
  pl.Cs = (float)(KQ * C);
  pl.lo2 = (float)log2(o);
  pl.r = (float)rgb[0];
  pl.g = (float)rgb[1];
  pl.b = (float)rgb[2];
  pl.src = src;
  double q_eff;
  if (rp.alpha_min <= 0.0) q_eff = LODGE_SUPPORT_Q;
  else if (!(o >= rp.alpha_min)) q_eff = -INFINITY;  // alpha <= o < alpha_min everywhere
  else q_eff = fmin(LODGE_SUPPORT_Q, 2.0 * log(o / rp.alpha_min));
  const double lmid = 0.5 * (A + C);
  const double rad = sqrt(0.25 * (A - C) * (A - C) + B * B);
  const double lmax = lmid + rad, lmin = lmid - rad;
  double tol;
  if (!(lmin > 0.0) || !(q_eff > -INFINITY)) {
    tol = (q_eff > -INFINITY) ? INFINITY : 0.0;
  } else {
    const double qr = fmax(q_eff, 0.0) + 1.0;
    const double cond = lmax / lmin;
    tol = 5.96e-8 * (48.0 * cond * qr + 96.0 * sqrt(lmax * cond * qr) + 4.0 * qr) + 1e-9 * qr;
  }
  // the scaled coefficients carry one rounding each, like (float)A did, so
  // |qs_fp32 - KQ * q_fp64| <= |KQ| * tol; KQ < 0 flips the band
  pl.hi = __double2float_ru(KQ * (q_eff - tol));
  pl.lo = __double2float_rd(KQ * (q_eff + tol));
  // {q <= Q} lies in |dx| <= sqrt(Q/9) * ex, |dy| <= sqrt(Q/9) * ey (ex = 3 sqrt(cov00));
  // Q = q_eff + tol bounds every pixel the fp64 reference may keep.  Generous
  // relative/absolute margins cover the rounding of cov2d and of the bounds.
  const double Q = fmin(fmax(q_eff, 0.0) + tol, LODGE_SUPPORT_Q * 1.001);
  const double sc = (q_eff > -INFINITY) ? sqrt(Q / 9.0) * 1.0001 : 0.0;
  pl.bx = (q_eff > -INFINITY) ? (float)(sc * ex + 1e-3) : -1.0f;
  pl.by = (q_eff > -INFINITY) ? (float)(sc * ey + 1e-3) : -1.0f;
  pr.A = A;
  pr.B = B;
  pr.C = C;
  pr.o = o;
  pr.r = rgb[0];
  pr.g = rgb[1];
  pr.b = rgb[2];
  pr.pad = 0.0;
}

__device__ __forceinline__ uint64_t tile_rect(double mx, double my, double ex, double ey,
                                              int32_t tiles_x, int32_t tiles_y) {
  // floor((m -/+ e) / 16), clipped (src/raster.py:303-313)
  int64_t x0 = (int64_t)floor((mx - ex) / 16.0), x1 = (int64_t)floor((mx + ex) / 16.0);
  int64_t y0 = (int64_t)floor((my - ey) / 16.0), y1 = (int64_t)floor((my + ey) / 16.0);
  x0 = x0 < 0 ? 0 : (x0 > tiles_x - 1 ? tiles_x - 1 : x0);
  x1 = x1 < 0 ? 0 : (x1 > tiles_x - 1 ? tiles_x - 1 : x1);
  y0 = y0 < 0 ? 0 : (y0 > tiles_y - 1 ? tiles_y - 1 : y0);
  y1 = y1 < 0 ? 0 : (y1 > tiles_y - 1 ? tiles_y - 1 : y1);
  return (uint64_t)x0 | ((uint64_t)x1 << 16) | ((uint64_t)y0 << 32) | ((uint64_t)y1 << 48);
}

// ---------------------------------------------------------------------------
// Frame mode: inputs come from the K1 union (tags), outputs are the internal
// compositing representation.
// ---------------------------------------------------------------------------
struct ProjLevels {
  const void *geom[LODGE_MAX_LEVELS];
  const void *sh[LODGE_MAX_LEVELS];
  int32_t degree[LODGE_MAX_LEVELS];
  int32_t qnorm[LODGE_MAX_LEVELS];  // LODGE_GEOM_QNORM per level
  uint32_t slot_base[LODGE_MAX_LEVELS + 1];
  int32_t L;
  // chunk slabs (lodge_chunks.slab_*_dev), or NULL: the union then holds
  // positions in the owning chunk's set and these tables locate the records
  const void *const *slab_geom;
  const void *const *slab_sh;
  uint32_t n[LODGE_MAX_LEVELS];  // records per level (bounds checks)
  int32_t diff_in_smem;          // k_project_frame: CTA-private difference array
};

// Shared per-CTA frame context of the frame kernels (camera, blend factor,
// chunk pair, per-level concatenated offsets and sizes).
struct FrameCtx {
  lodge_camera cam;
  double t;
  int32_t f, o;
  int32_t wpat;  // camera rotation zero pattern (project_any)
  CamLims lim;   // the camera's x/z, y/z clamp limits
  uint32_t used[LODGE_MAX_LEVELS], cat[LODGE_MAX_LEVELS];
};

__device__ __forceinline__ void stage_frame_ctx(FrameCtx &F, const ProjLevels &lv,
                                                const FrameState *fs,
                                                const lodge_camera *__restrict__ cam_p) {
  if (threadIdx.x == 0) {
    F.cam = *cam_p;
    F.wpat = camera_wpattern(F.cam);
    F.lim = cam_lims(F.cam);
    F.t = fs->stats.t;
    F.f = fs->stats.f;
    F.o = fs->stats.o < 0 ? fs->stats.f : fs->stats.o;
    uint32_t c = 0;
    for (int k = 0; k < lv.L; ++k) {
      F.cat[k] = c;  // concatenated index offset of level k
      F.used[k] = fs->stats.U_level[k];
      c += F.used[k];
    }
  }
  __syncthreads();
}

// The record of union slot `slot` of level l: geometry loaded (rotation
// normalised if the level asks), modulation from the blend tag, SH pointer
// and record index for the colour.  Shared by the projection and the
// payload kernel, so both evaluate the identical fp64 projection (DISPATCH:
// drop the exact-zero camera terms, project_any; the fields are the same).
// (gidx, tag: the slot's union entry.)
template <typename GT, typename ST, bool DISPATCH = true>
__device__ __forceinline__ Proj slot_project_at(const ProjLevels &lv, const FrameCtx &F,
                                                const lodge_raster_params &rp, int l,
                                                uint32_t gidx, uint8_t tag, double v[12],
                                                const ST *&sp) {
  const GT *gp = reinterpret_cast<const GT *>(lv.geom[l]);
  sp = reinterpret_cast<const ST *>(lv.sh[l]);
  const double mod = (tag == 3) ? 1.0 : (tag == 1 ? F.t : 1.0 - F.t);
  if (lv.slab_geom) {  // tag 3 / 1: the primary chunk's slab, 2: the other's
    const int32_t e = ((tag == 2) ? F.o : F.f) * lv.L + l;
    gp = reinterpret_cast<const GT *>(lv.slab_geom[e]);
    sp = reinterpret_cast<const ST *>(lv.slab_sh[e]);
  }
  load_geom<GT>(gp + (size_t)gidx * 12, v);
  if (lv.qnorm[l]) normalize_rot(v);
  return DISPATCH ? project_any(v, F.cam, rp, mod, true, F.wpat, F.lim)
                  : project_core<W_FULL>(v, F.cam, rp, mod, true, F.lim);
}
template <typename GT, typename ST, bool DISPATCH = true>
__device__ __forceinline__ Proj slot_project(const ProjLevels &lv, const Work &w,
                                             const FrameCtx &F, const lodge_raster_params &rp,
                                             int l, uint32_t slot, double v[12],
                                             const ST *&sp, uint32_t &gidx) {
  gidx = w.union_idx[slot];
  return slot_project_at<GT, ST, DISPATCH>(lv, F, rp, l, gidx, w.union_tag[slot], v, sp);
}

// K2, geometry only.  Outputs are written at the dense concatenated input
// index g (level-major union position, the reference's Splat2DBatch.concat
// source index), with no compaction: culled inputs get depth key ~0, so the
// stable depth sort over all U inputs orders the M survivors by (depth, g)
// -- exactly np.lexsort((source_index, depth)) -- and leaves the culled ones
// after them.  Colour and the compositing records are left to k_payload,
// which runs only for the splats a frame composites (a few percent of M on
// the bench sweep: the tiles finish early).
#ifndef PROJ_RUN
#define PROJ_RUN 128  // survivors staged per warp before a flush
#endif
template <typename GT, typename ST>
#ifndef LODGE_PROJ_MINB
#define LODGE_PROJ_MINB 3  // resident CTAs per SM (the persistent grid's size; 80 registers)
#endif
__global__ void __launch_bounds__(256, LODGE_PROJ_MINB) k_project_frame(ProjLevels lv, Work w, FrameState *fs,
                                                       const lodge_camera *__restrict__ cam_p,
                                                       lodge_raster_params rp, int32_t tiles_x,
                                                       int32_t tiles_y) {
  // persistent CTAs (grid-stride over the slots): the camera and the level
  // table are staged once per CTA
  __shared__ FrameCtx F;
  // per_tile_count's 2-D difference array, CTA-private in shared memory when
  // it fits (the host passes its size as the dynamic shared memory), flushed
  // once at the end: the corners of border-clipped splats are shared by most
  // of a frame's splats, and global atomics on them serialised the kernel
  // (0.15 of its 0.27 ms at config 3, profiles/r02_stress.md)
  extern __shared__ int32_t s_diff[];
  const int32_t n_diff = (tiles_x + 1) * (tiles_y + 1);
  const bool priv = lv.diff_in_smem != 0;
  if (priv)
    for (int32_t i = threadIdx.x; i < n_diff; i += blockDim.x) s_diff[i] = 0;
  stage_frame_ctx(F, lv, fs, cam_p);
  // the tile grid is the frame's (host W, H), so the difference-array
  // indices stay in range whatever the device camera holds
  const uint32_t nslots = lv.slot_base[lv.L];
  // survivors leave compacted (32-bit depth key, input index) for the depth
  // sort, staged per warp and flushed in runs (one atomic per run on
  // stats.M, which ends as the survivor count); the order of the runs does
  // not matter: the sort orders by (key, fp64 key, index)
  __shared__ uint32_t s_ck[8][PROJ_RUN], s_cg[8][PROJ_RUN];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t *const ckey = depth_keys_compact(w);
  uint32_t wc = 0;  // staged survivors of this warp
  auto flush = [&]() {
    __syncwarp();
    uint32_t b0 = 0;
    if (lane == 0) b0 = atomicAdd(&fs->stats.M, wc);
    b0 = __shfl_sync(FULL_MASK, b0, 0);
    for (uint32_t i = lane; i < wc; i += 32) {
      if (b0 + i < (uint32_t)w.M_cap) {
        ckey[b0 + i] = s_ck[wid][i];
        w.val_depth[1][b0 + i] = s_cg[wid][i];
      } else {
        raise_fault(fs, FAULT_SCATTER);
      }
    }
    __syncwarp();
    wc = 0;
  };
  for (uint32_t base = blockIdx.x * blockDim.x; base < nslots; base += gridDim.x * blockDim.x) {
    const uint32_t slot = base + threadIdx.x;
    // map slot -> level
    int l = 0;  // the levels' slot ranges are consecutive: count the starts passed
#pragma unroll
    for (int k = 1; k < LODGE_MAX_LEVELS; ++k) l += (k < lv.L && slot >= lv.slot_base[k]) ? 1 : 0;
    const uint32_t pos = slot - lv.slot_base[l];
    const bool valid = slot < nslots && pos < F.used[l];
    const uint32_t g = F.cat[l] + pos;
    Proj p;
    p.ok = false;
    if (valid) {
      double v[12];
      const ST *sp;
      uint32_t gidx;
      p = slot_project<GT, ST>(lv, w, F, rp, l, slot, v, sp, gidx);
    }
    const bool keep = valid && p.ok;
#ifdef LODGE_DEPTH64  // the 64-bit sort reads every input's key by position
    if (valid) {
      w.val_depth[1][g] = g;
      if (!keep) w.key_depth[0][g] = ~0ull;
    }
    if (keep) atomicAdd(&fs->stats.M, 1u);
    const uint32_t kb = 0u;
#else
    const uint32_t kb = __ballot_sync(FULL_MASK, keep);
#endif
    if (wc + __popc(kb) > PROJ_RUN) flush();
    if (keep) {
      const uint32_t at = wc + __popc(kb & ((1u << lane) - 1u));
      s_ck[wid][at] = __float_as_uint(__double2float_rz(p.z));  // depth_key32
      s_cg[wid][at] = g;
    }
    wc += __popc(kb);
    const uint64_t rc = keep ? tile_rect(p.mx, p.my, p.ex, p.ey, tiles_x, tiles_y) : 0ull;
    if (priv) add_tile_diff_shared(s_diff, rc, tiles_x, tiles_y, keep);
    else add_tile_diff(w.tile_diff, rc, tiles_x, keep);
    if (keep) {  // the full key (tie repair) and the rectangle, by input index
      w.key_depth[0][g] = (uint64_t)__double_as_longlong(p.z);
      w.rect[g] = rc;
    }
  }
  if (wc) flush();
  if (priv) {
    __syncthreads();
    for (int32_t i = threadIdx.x; i < n_diff; i += blockDim.x) {
      const int32_t v = s_diff[i];
      if (v) atomicAdd(w.tile_diff + i, v);
    }
  }
}

// Compositing records (payload + fp64 record, colour from the SH) of the
// splats ids[0 .. *n): concatenated indices g of survivors.  The projection
// is re-evaluated from the same record with the same code as K2, so every
// field is bit-identical to an eager evaluation.
#ifndef LODGE_PAYLOAD_MINB
#define LODGE_PAYLOAD_MINB 3  // resident CTAs per SM (register cap)
#endif
template <typename GT, typename ST>
__global__ void __launch_bounds__(256, LODGE_PAYLOAD_MINB) k_payload(ProjLevels lv, Work w, FrameState *fs,
                                                 const lodge_camera *__restrict__ cam_p,
                                                 lodge_raster_params rp, int32_t shade,
                                                 const uint32_t *__restrict__ ids,
                                                 const uint32_t *n_ptr) {
  __shared__ FrameCtx F;
  stage_frame_ctx(F, lv, fs, cam_p);
  const uint32_t n = fs->stats.overflow ? 0u : *n_ptr;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t g = ids[i];
    int l = 0;
    while (l + 1 < lv.L && g >= F.cat[l + 1]) ++l;
    if (g >= F.cat[l] + F.used[l] || g >= (uint32_t)w.M_cap) {  // not an input of this frame
      raise_fault(fs, FAULT_PAYLOAD);
      continue;
    }
    const uint32_t slot = lv.slot_base[l] + (g - F.cat[l]);
    if (!lv.slab_geom && w.union_idx[slot] >= lv.n[l]) {
      raise_fault(fs, FAULT_PAYLOAD);
      continue;
    }
    double v[12];
    const ST *sp;
    uint32_t gidx;
    const Proj p = slot_project<GT, ST, false>(lv, w, F, rp, l, slot, v, sp, gidx);
    double rgb[3] = {0.0, 0.0, 0.0};
    if (shade) {
      const int deg = lv.degree[l];
      const int terms = (deg + 1) * (deg + 1);
      eval_sh_dev<ST>(sp + (size_t)gidx * 3 * terms, terms, deg, v, F.cam, rgb);
    }
    const double inv_det = 1.0 / p.det;
    const double A = p.c11 * inv_det, B = (-p.c01) * inv_det, C = p.c00 * inv_det;
    Payload pl;
    Precise pr;
    make_payload(p.mx, p.my, A, B, C, p.op, rgb, g, p.ex, p.ey, rp, pl, pr);
    w.payload[g] = pl;
    w.precise[g] = pr;
  }
}

// ---------------------------------------------------------------------------
// Compat mode: one level, explicit indices/modulation, exports Splat2DBatch.
// ---------------------------------------------------------------------------
template <typename GT, typename ST>
__global__ void __launch_bounds__(256) k_project_compat(const GT *geom, const ST *sh, int32_t deg,
                                                        const int64_t *idx, int64_t n,
                                                        const double *mod, Work w, FrameState *fs,
                                                        const lodge_camera *__restrict__ cam_p,
                                                        lodge_raster_params rp, int32_t shade,
                                                        lodge_batch out, int32_t qnorm) {
  __shared__ uint32_t s_warp[32];
  __shared__ uint32_t s_base;
  __shared__ lodge_camera cam;
  if (threadIdx.x == 0) cam = *cam_p;
  const uint32_t part = take_ticket(&fs->tickets[TK_COMPACT], &s_base);
  const int64_t e = (int64_t)part * blockDim.x + threadIdx.x;
  Proj p;
  p.ok = false;
  double v[12];
  int64_t g = 0;
  if (e < n) {
    g = idx ? idx[e] : e;
    load_geom<GT>(geom + (size_t)g * 12, v);
    if (qnorm) normalize_rot(v);
    p = project_any(v, cam, rp, mod ? mod[e] : 1.0, mod != nullptr, camera_wpattern(cam),
                    cam_lims(cam));
  }
  const int64_t m = compact_slot(e < n && p.ok, w.status, fs->epoch + TK_COMPACT, part, s_warp,
                                 &s_base);
  if (m < 0) return;
  double rgb[3] = {0.0, 0.0, 0.0};
  if (shade) {
    const int terms = (deg + 1) * (deg + 1);
    eval_sh_dev<ST>(sh + (size_t)g * 3 * terms, terms, deg, v, cam, rgb);
  }
  const double inv_det = 1.0 / p.det;
  out.src_dev[m] = e;
  out.mean2d_dev[2 * m] = p.mx;
  out.mean2d_dev[2 * m + 1] = p.my;
  out.cov2d_dev[4 * m] = p.c00;
  out.cov2d_dev[4 * m + 1] = p.c01;
  out.cov2d_dev[4 * m + 2] = p.c10;
  out.cov2d_dev[4 * m + 3] = p.c11;
  out.conic_dev[3 * m] = p.c11 * inv_det;
  out.conic_dev[3 * m + 1] = (-p.c01) * inv_det;
  out.conic_dev[3 * m + 2] = p.c00 * inv_det;
  out.extent_dev[2 * m] = p.ex;
  out.extent_dev[2 * m + 1] = p.ey;
  out.depth_dev[m] = p.z;
  out.opacity_dev[m] = p.op;
  out.color_dev[3 * m] = rgb[0];
  out.color_dev[3 * m + 1] = rgb[1];
  out.color_dev[3 * m + 2] = rgb[2];
  atomicMax(&fs->stats.M, (uint32_t)(m + 1));
}

// Threshold-search cost table, first half (ThresholdSearcher._table,
// src/thresholds.py:80-90): project_scene(shade=False) of every input, and
// for each survivor, compacted in input order (the batch order), its tile
// cover count (tile_cover_counts, src/raster.py:316-324) and its camera
// distance np.linalg.norm(means[src] - position) = sqrt((dx*dx + dy*dy) +
// dz*dz) as a depth-sort key (IEEE bits of a non-negative double) with the
// count as its value; the stable depth sort then yields argsort(dist, stable).
template <typename GT>
__global__ void __launch_bounds__(256) k_cover_keys(const GT *geom, const int64_t *idx, int64_t n,
                                                    int32_t qnorm, Work w, FrameState *fs,
                                                    const lodge_camera *__restrict__ cam_p,
                                                    lodge_raster_params rp) {
  __shared__ uint32_t s_warp[32];
  __shared__ uint32_t s_base;
  __shared__ lodge_camera cam;
  if (threadIdx.x == 0) cam = *cam_p;
  const uint32_t part = take_ticket(&fs->tickets[TK_COMPACT], &s_base);
  const int64_t e = (int64_t)part * blockDim.x + threadIdx.x;
  Proj p;
  p.ok = false;
  double v[12];
  if (e < n) {
    const int64_t g = idx ? idx[e] : e;
    load_geom<GT>(geom + (size_t)g * 12, v);
    if (qnorm) normalize_rot(v);
    p = project_any(v, cam, rp, 1.0, false, camera_wpattern(cam), cam_lims(cam));
  }
  const int64_t m = compact_slot(e < n && p.ok, w.status, fs->epoch + TK_COMPACT, part, s_warp,
                                 &s_base);
  if (m < 0) return;
  const int32_t tiles_x = (cam.w + 15) / 16, tiles_y = (cam.h + 15) / 16;
  const uint64_t rc = tile_rect(p.mx, p.my, p.ex, p.ey, tiles_x, tiles_y);
  const uint32_t x0 = rc & 0xffff, x1 = (rc >> 16) & 0xffff, y0 = (rc >> 32) & 0xffff,
                 y1 = rc >> 48;
  const double dx = v[0] - cam.pos[0], dy = v[1] - cam.pos[1], dz = v[2] - cam.pos[2];
  const double dist = sqrt((dx * dx + dy * dy) + dz * dz);
  w.key_depth[0][m] = (uint64_t)__double_as_longlong(dist);
  w.val_depth[0][m] = (x1 - x0 + 1) * (y1 - y0 + 1);
  atomicMax(&fs->stats.M, (uint32_t)(m + 1));
}

int launch_cover_keys(const lodge_level &level, const int64_t *idx, int64_t n, const Work &w,
                      FrameState *fs, const lodge_camera *cam_dev, const lodge_raster_params &rp,
                      cudaStream_t s) {
  if (n <= 0) return 0;
  const unsigned grid = (unsigned)((n + 255) / 256);
  const int32_t qn = (level.flags & LODGE_GEOM_QNORM) ? 1 : 0;
  if (level.flags & LODGE_GEOM_FP32)
    k_cover_keys<float><<<grid, 256, 0, s>>>((const float *)level.geom_dev, idx, n, qn, w, fs,
                                             cam_dev, rp);
  else
    k_cover_keys<double><<<grid, 256, 0, s>>>((const double *)level.geom_dev, idx, n, qn, w, fs,
                                              cam_dev, rp);
  return 0;
}

// Compat rasterize: import a host-made Splat2DBatch into the internal form.
__global__ void __launch_bounds__(256) k_import_batch(lodge_batch b, int64_t M, Work w,
                                                      FrameState *fs,
                                                      const lodge_camera *__restrict__ cam_p,
                                                      lodge_raster_params rp) {
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const lodge_camera &cam = *cam_p;
  const int32_t tiles_x = (cam.w + 15) / 16, tiles_y = (cam.h + 15) / 16;
  const bool valid = m < M;
  const uint64_t rc = valid ? tile_rect(b.mean2d_dev[2 * m], b.mean2d_dev[2 * m + 1],
                                        b.extent_dev[2 * m], b.extent_dev[2 * m + 1], tiles_x,
                                        tiles_y)
                            : 0ull;
  add_tile_diff(w.tile_diff, rc, tiles_x, valid);
  if (!valid) return;
  const double mx = b.mean2d_dev[2 * m], my = b.mean2d_dev[2 * m + 1];
  const double rgb[3] = {b.color_dev[3 * m], b.color_dev[3 * m + 1], b.color_dev[3 * m + 2]};
  Payload pl;
  Precise pr;
  make_payload(mx, my, b.conic_dev[3 * m], b.conic_dev[3 * m + 1], b.conic_dev[3 * m + 2],
               b.opacity_dev[m], rgb, (uint32_t)b.src_dev[m], b.extent_dev[2 * m],
               b.extent_dev[2 * m + 1], rp, pl, pr);
  w.payload[m] = pl;
  w.precise[m] = pr;
  w.rect[m] = rc;
  // lexsort((src, depth)): the depth sort is stable, so feed rows in
  // source-index order via the values; the batch's src order is ascending
  // for project_scene outputs, otherwise the host pre-sorts (see raster.py).
  w.key_depth[0][m] = (uint64_t)__double_as_longlong(b.depth_dev[m]);
  w.val_depth[1][m] = (uint32_t)m;  // the depth sort's input values
  if (m == 0) {
    fs->stats.M = (uint32_t)M;
    fs->n_sort = (uint32_t)M;
  }
}

static int sm_count() {
  static PerDevice sms;
  if (!sms()) {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    sms() = n > 0 ? n : 148;
  }
  return (int)sms();
}

// Largest CTA-private difference array of the projection (int32 entries):
// 96 KB, two CTAs per SM -- up to ~2560 x 1440 (4K frames use global atomics).
constexpr int32_t PROJ_DIFF_SMEM_MAX = 96 * 1024;

template <typename GT, typename ST>
static void launch_pf(ProjLevels lv, const Work &w, FrameState *fs,
                      const lodge_camera *cam, const lodge_raster_params &rp, uint32_t nslots,
                      int32_t tiles_x, int32_t tiles_y, cudaStream_t s) {
  const uint32_t per = w.grid_share > 0 ? std::min(w.grid_share, LODGE_PROJ_MINB) : LODGE_PROJ_MINB;
  const uint32_t want = (nslots + 255) / 256, cap = per * (uint32_t)sm_count();
  const int64_t bytes = 4ll * (tiles_x + 1) * (tiles_y + 1);
  lv.diff_in_smem = bytes <= PROJ_DIFF_SMEM_MAX ? 1 : 0;
  const size_t sm = lv.diff_in_smem ? (size_t)bytes : 0;
  static PerDevice attr;
  if (sm > 48 * 1024 && !attr()) {
    cudaFuncSetAttribute(k_project_frame<GT, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         PROJ_DIFF_SMEM_MAX);
    attr() = 1;
  }
  k_project_frame<GT, ST><<<want < cap ? want : cap, 256, sm, s>>>(lv, w, fs, cam, rp, tiles_x,
                                                                    tiles_y);
}

template <typename GT, typename ST>
static void launch_pl(const ProjLevels &lv, const Work &w, FrameState *fs,
                      const lodge_camera *cam, const lodge_raster_params &rp, int32_t shade,
                      const uint32_t *ids, const uint32_t *n_ptr, int64_t n_cap, cudaStream_t s) {
  const int64_t per = w.grid_share > 0 ? std::min(w.grid_share, 4) : 4;  // CTAs per SM
  const int64_t want = (n_cap + 255) / 256, cap = per * (int64_t)sm_count();
  k_payload<GT, ST><<<(unsigned)std::max<int64_t>(1, std::min(want, cap)), 256, 0, s>>>(
      lv, w, fs, cam, rp, shade, ids, n_ptr);
}

static int proj_levels(const lodge_level *levels, const LevelSlots &ls,
                       const void *const *slab_geom, const void *const *slab_sh, ProjLevels &lv,
                       bool &g32, bool &s32) {
  lv.L = ls.n_levels;
  lv.diff_in_smem = 0;
  lv.slab_geom = slab_geom;
  lv.slab_sh = slab_sh;
  const int32_t prec_bits = LODGE_GEOM_FP32 | LODGE_SH_FP32;
  const int32_t fl = levels[0].flags & prec_bits;
  for (int l = 0; l < lv.L; ++l) {
    if ((levels[l].flags & prec_bits) != fl) return -1;  // one storage precision per store
    lv.geom[l] = levels[l].geom_dev;
    lv.sh[l] = levels[l].sh_dev;
    lv.degree[l] = levels[l].sh_degree;
    lv.qnorm[l] = (levels[l].flags & LODGE_GEOM_QNORM) ? 1 : 0;
    lv.n[l] = (uint32_t)levels[l].n;
  }
  for (int l = 0; l <= LODGE_MAX_LEVELS; ++l) lv.slot_base[l] = l <= lv.L ? ls.slot_base[l] : 0;
  g32 = fl & LODGE_GEOM_FP32;
  s32 = fl & LODGE_SH_FP32;
  return 0;
}

int launch_project_frame(const lodge_level *levels, const LevelSlots &ls, const Work &w,
                         FrameState *fs, const lodge_camera *cam_dev,
                         const lodge_raster_params &rp, int32_t W, int32_t H, cudaStream_t s,
                         const void *const *slab_geom, const void *const *slab_sh) {
  const int32_t tx = (W + 15) / 16, ty = (H + 15) / 16;
  ProjLevels lv;
  bool g32, s32;
  if (proj_levels(levels, ls, slab_geom, slab_sh, lv, g32, s32)) return -1;
  const uint32_t nslots = ls.slot_base[lv.L];
  if (nslots == 0) return 0;
  if (g32 && s32) launch_pf<float, float>(lv, w, fs, cam_dev, rp, nslots, tx, ty, s);
  else if (g32) launch_pf<float, double>(lv, w, fs, cam_dev, rp, nslots, tx, ty, s);
  else if (s32) launch_pf<double, float>(lv, w, fs, cam_dev, rp, nslots, tx, ty, s);
  else launch_pf<double, double>(lv, w, fs, cam_dev, rp, nslots, tx, ty, s);
  return 0;
}

int launch_payload(const lodge_level *levels, const LevelSlots &ls, const Work &w,
                   FrameState *fs, const lodge_camera *cam_dev, const lodge_raster_params &rp,
                   int32_t shade, const uint32_t *ids, const uint32_t *n_ptr, int64_t n_cap,
                   cudaStream_t s, const void *const *slab_geom, const void *const *slab_sh) {
  ProjLevels lv;
  bool g32, s32;
  if (proj_levels(levels, ls, slab_geom, slab_sh, lv, g32, s32)) return -1;
  if (n_cap <= 0) return 0;
  if (g32 && s32) launch_pl<float, float>(lv, w, fs, cam_dev, rp, shade, ids, n_ptr, n_cap, s);
  else if (g32) launch_pl<float, double>(lv, w, fs, cam_dev, rp, shade, ids, n_ptr, n_cap, s);
  else if (s32) launch_pl<double, float>(lv, w, fs, cam_dev, rp, shade, ids, n_ptr, n_cap, s);
  else launch_pl<double, double>(lv, w, fs, cam_dev, rp, shade, ids, n_ptr, n_cap, s);
  return 0;
}

int launch_project_compat(const lodge_level &level, const int64_t *idx, int64_t n,
                          const double *mod, const Work &w, FrameState *fs,
                          const lodge_camera *cam_dev, const lodge_raster_params &rp,
                          int32_t shade, const lodge_batch *out, cudaStream_t s) {
  if (n <= 0) return 0;
  const unsigned grid = (unsigned)((n + 255) / 256);
  const bool g32 = level.flags & LODGE_GEOM_FP32, s32 = level.flags & LODGE_SH_FP32;
#define LP(GT, ST)                                                                         \
  k_project_compat<GT, ST><<<grid, 256, 0, s>>>((const GT *)level.geom_dev,                \
                                                (const ST *)level.sh_dev, level.sh_degree, \
                                                idx, n, mod, w, fs, cam_dev, rp, shade, *out, \
                                                (level.flags & LODGE_GEOM_QNORM) ? 1 : 0)
  if (g32 && s32) LP(float, float);
  else if (g32) LP(float, double);
  else if (s32) LP(double, float);
  else LP(double, double);
#undef LP
  return 0;
}

void launch_import_batch(const lodge_batch &b, int64_t M, const Work &w, FrameState *fs,
                         const lodge_camera *cam_dev, const lodge_raster_params &rp, int32_t,
                         cudaStream_t s) {
  if (M <= 0) return;
  k_import_batch<<<(unsigned)((M + 255) / 256), 256, 0, s>>>(b, M, w, fs, cam_dev, rp);
}

}  // namespace lodge
