/*
 * px_oracle.c -- CPU restatement of the PERCH 2.0 parallel-search hot path.
 *
 * TEST INFRASTRUCTURE, NOT PRODUCT.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product (paper_2008_00326_b200 + libpx.so) never links or calls it.
 *
 * It restates, in plain C, the reference's Python/numba algorithm for
 *   render -> occluder mark -> stride cloud -> Lab       raster.py:53-134, 239-280
 *   exact kNN                                            neighbors.py:104-134
 *   k-NN covariances + Jacobi                            registration.py:109-216
 *   GICP linearise / objective / align                   registration.py:233-494
 *   refine apply + 3-DoF re-lift                         search.py:291-301
 *   explanation cost (j_r, explained, j_o)               cost.py:91-152, search.py:189-202
 *   CIELAB / CIEDE2000                                   colorspace.py:29-124
 * (paths relative to /root/reference/pkg/src/rvpose/).
 *
 * Parity pinning: tests/golden/ holds outputs of the reference itself (made by
 * oracle/make_golden.py importing it); tests/test_oracle_golden.py checks this
 * file against every one of them.  Where the reference goes through numpy ->
 * OpenBLAS the fused-multiply-add order observed on the fixture host is
 * restated with explicit fma() (see oracle/README.md, "host BLAS orders");
 * numba kernels contain no contraction, so everything else is compiled with
 * -ffp-contract=off.  Third-party arithmetic that cannot be restated bit for
 * bit (LAPACK dgesv / dgesdd, numpy SIMD pow/cbrt) is restated by its
 * published algorithm: partial-pivot LU, polar projection, libm.
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define ORC_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------------ */
/* small linear algebra in the host-BLAS rounding orders                     */

/* sum_k a[k]*b[k], fused, k = 0,1,2 (numpy matmul mat@mat, (V,3)@R.T, F-view@vec) */
static inline double dot_f012(double a0, double a1, double a2, double b0, double b1, double b2) {
  return fma(a2, b2, fma(a1, b1, a0 * b0));
}
/* k = 1,0,2 (numpy C-contiguous (3,3)@(3,)) */
static inline double dot_f102(double a0, double a1, double a2, double b0, double b1, double b2) {
  return fma(a2, b2, fma(a0, b0, a1 * b1));
}

/* pose = row-major 3x4 [R|t] */
static inline void apply_pose(const double* P, const double* x, double* y) { /* geometry.py:131-134 */
  for (int i = 0; i < 3; ++i)
    y[i] = dot_f012(x[0], x[1], x[2], P[4 * i + 0], P[4 * i + 1], P[4 * i + 2]) + P[4 * i + 3];
}

/* C = A o B with A's rotation laid out C-contiguous (vec_order 0 -> k=1,0,2) or
 * as a transposed view (vec_order 1 -> k=0,1,2); geometry.py:136-141 */
static void compose_pose(const double* A, const double* B, int vec_order, double* C) {
  double out[12];
  for (int i = 0; i < 3; ++i) {
    const double a0 = A[4 * i], a1 = A[4 * i + 1], a2 = A[4 * i + 2];
    for (int j = 0; j < 3; ++j) out[4 * i + j] = dot_f012(a0, a1, a2, B[j], B[4 + j], B[8 + j]);
    double rt = vec_order ? dot_f012(a0, a1, a2, B[3], B[7], B[11]) : dot_f102(a0, a1, a2, B[3], B[7], B[11]);
    out[4 * i + 3] = rt + A[4 * i + 3];
  }
  memcpy(C, out, sizeof out);
}

/* ------------------------------------------------------------------------ */
/* colour                                                                     */

static const double RGB2XYZ[9] = {0.4124564, 0.3575761, 0.1804375, 0.2126729, 0.7151522,
                                  0.0721750, 0.0193339, 0.1191920, 0.9503041};
static const double WHITE[3] = {0.95047, 1.0, 1.08883};

static inline double srgb_encode1(double c) { /* colorspace.py:35-38 */
  if (c < 0.0) c = 0.0;
  if (c > 1.0) c = 1.0;
  return c <= 0.0031308 ? 12.92 * c : 1.055 * pow(c, 1.0 / 2.4) - 0.055;
}
static inline double srgb_decode1(double c) { /* colorspace.py:29-32 */
  return c <= 0.04045 ? c / 12.92 : pow((c + 0.055) / 1.055, 2.4);
}

ORC_API void orc_srgb_to_lab(const double* rgb, int64_t n, double* lab) { /* colorspace.py:41-55 */
  const double d = 6.0 / 29.0;
  const double d3 = pow(d, 3.0), lin_div = 3.0 * d * d, off = 4.0 / 29.0;
  for (int64_t p = 0; p < n; ++p) {
    double l0 = srgb_decode1(rgb[3 * p]), l1 = srgb_decode1(rgb[3 * p + 1]), l2 = srgb_decode1(rgb[3 * p + 2]);
    double f[3];
    for (int i = 0; i < 3; ++i) {
      double xyz = dot_f012(l0, l1, l2, RGB2XYZ[3 * i], RGB2XYZ[3 * i + 1], RGB2XYZ[3 * i + 2]);
      double t = xyz / WHITE[i];
      f[i] = t > d3 ? cbrt(t) : t / lin_div + off;
    }
    lab[3 * p] = 116.0 * f[1] - 16.0;
    lab[3 * p + 1] = 500.0 * (f[0] - f[1]);
    lab[3 * p + 2] = 200.0 * (f[1] - f[2]);
  }
}

static inline double pymod360(double x) { /* numpy float % 360.0 */
  double m = fmod(x, 360.0);
  if (m != 0.0) {
    if (m < 0.0) m += 360.0;
  } else {
    m = copysign(0.0, 360.0);
  }
  return m;
}
#define DEG(x) ((x) * (180.0 / M_PI))
#define RAD(x) ((x) * (M_PI / 180.0))

ORC_API double orc_ciede2000(const double* x, const double* y) { /* colorspace.py:58-124 */
  const double P25_7 = pow(25.0, 7.0);
  double L1 = x[0], a1 = x[1], b1 = x[2], L2 = y[0], a2 = y[1], b2 = y[2];
  double c1 = hypot(a1, b1), c2 = hypot(a2, b2);
  double cb = 0.5 * (c1 + c2);
  double cb7 = pow(cb, 7.0);
  double g = 0.5 * (1.0 - sqrt(cb7 / (cb7 + P25_7)));
  double a1p = (1.0 + g) * a1, a2p = (1.0 + g) * a2;
  double c1p = hypot(a1p, b1), c2p = hypot(a2p, b2);
  double h1 = pymod360(DEG(atan2(b1, a1p))), h2 = pymod360(DEG(atan2(b2, a2p)));
  if (a1p == 0.0 && b1 == 0.0) h1 = 0.0;
  if (a2p == 0.0 && b2 == 0.0) h2 = 0.0;
  double dL = L2 - L1, dC = c2p - c1p;
  int grey = (c1p * c2p) == 0.0;
  double dh = h2 - h1;
  if (dh > 180.0) dh -= 360.0;
  if (dh < -180.0) dh += 360.0;
  if (grey) dh = 0.0;
  double dH = 2.0 * sqrt(c1p * c2p) * sin(RAD(0.5 * dh));
  double Lm = 0.5 * (L1 + L2), Cm = 0.5 * (c1p + c2p);
  double hs = h1 + h2, hd = fabs(h1 - h2);
  double hm = hd <= 180.0 ? 0.5 * hs : (hs < 360.0 ? 0.5 * (hs + 360.0) : 0.5 * (hs - 360.0));
  if (grey) hm = hs;
  double t = 1.0 - 0.17 * cos(RAD(hm - 30.0)) + 0.24 * cos(RAD(2.0 * hm)) +
             0.32 * cos(RAD(3.0 * hm + 6.0)) - 0.20 * cos(RAD(4.0 * hm - 63.0));
  double q = (hm - 275.0) / 25.0;
  double dth = 30.0 * exp(-(q * q));
  double Cm7 = pow(Cm, 7.0);
  double rc = 2.0 * sqrt(Cm7 / (Cm7 + P25_7));
  double lm50 = (Lm - 50.0) * (Lm - 50.0);
  double sl = 1.0 + 0.015 * lm50 / sqrt(20.0 + lm50);
  double sc = 1.0 + 0.045 * Cm;
  double sh = 1.0 + 0.015 * Cm * t;
  double rt = -sin(RAD(2.0 * dth)) * rc;
  double tl = dL / sl, tc = dC / sc, th = dH / sh;
  return sqrt(tl * tl + tc * tc + th * th + rt * tc * th);
}

/* ------------------------------------------------------------------------ */
/* scene / model descriptors                                                  */

typedef struct {
  int32_t H, W, stride, pad_;
  const double* depth;    /* (H,W) */
  const uint8_t* valid;   /* (H,W) */
  const int32_t* labels;  /* (H,W) */
  double fx, fy, cx, cy;
  int64_t n_obs;
  const double* obs_pts;      /* (n_obs,3) */
  const double* obs_lab;      /* (n_obs,3) */
  const int32_t* obs_labels;  /* (n_obs,) */
} orc_scene;

typedef struct {
  int32_t object_id, V, T, pad_;
  const double* verts;    /* (V,3) object frame */
  const double* col_lin;  /* (V,3) linear light (host srgb_decode) */
  const int32_t* tris;    /* (T,3) */
  double cyl_r2, cyl_zmin, cyl_zmax; /* radius**2 as computed by the host */
} orc_model;

/* ------------------------------------------------------------------------ */
/* rasteriser: raster.py:53-134, literal.  `owner` (may be NULL) records the  */
/* winning triangle per pixel.  `box` returns the touched pixel rectangle.    */

#define NEAR_PLANE 1e-4

static void raster_kernel(const double* verts, const int32_t* tris, int T, const double* col, double fx,
                          double fy, double cx, double cy, int W, int H, double* zbuf, double* cbuf,
                          uint8_t* valid, int32_t* owner, int* box) {
  for (int ti = 0; ti < T; ++ti) {
    int ia = tris[3 * ti], ib = tris[3 * ti + 1], ic = tris[3 * ti + 2];
    double za = verts[3 * ia + 2], zb = verts[3 * ib + 2], zc = verts[3 * ic + 2];
    if (za <= NEAR_PLANE || zb <= NEAR_PLANE || zc <= NEAR_PLANE) continue;
    double u0 = fx * verts[3 * ia] / za + cx, v0 = fy * verts[3 * ia + 1] / za + cy;
    double u1 = fx * verts[3 * ib] / zb + cx, v1 = fy * verts[3 * ib + 1] / zb + cy;
    double u2 = fx * verts[3 * ic] / zc + cx, v2 = fy * verts[3 * ic + 1] / zc + cy;
    double z0 = za, z1 = zb, z2 = zc;
    const double *c0 = col + 3 * ia, *c1 = col + 3 * ib, *c2 = col + 3 * ic;
    double area2 = (u1 - u0) * (v2 - v0) - (v1 - v0) * (u2 - u0);
    if (area2 == 0.0) continue;
    if (area2 < 0.0) {
      double t;
      t = u1, u1 = u2, u2 = t;
      t = v1, v1 = v2, v2 = t;
      t = z1, z1 = z2, z2 = t;
      const double* tc = c1;
      c1 = c2, c2 = tc;
      area2 = -area2;
    }
    double umin = fmin(u0, fmin(u1, u2)), umax = fmax(u0, fmax(u1, u2));
    double vmin = fmin(v0, fmin(v1, v2)), vmax = fmax(v0, fmax(v1, v2));
    double lo;
    int px_lo, px_hi, py_lo, py_hi;
    /* int(np.ceil(x)) saturates far outside the image; clamp in double first */
    lo = ceil(umin - 0.5);
    px_lo = lo < 0.0 ? 0 : (lo > (double)W ? W : (int)lo);
    lo = floor(umax - 0.5);
    px_hi = lo > (double)(W - 1) ? W - 1 : (lo < -1.0 ? -1 : (int)lo);
    lo = ceil(vmin - 0.5);
    py_lo = lo < 0.0 ? 0 : (lo > (double)H ? H : (int)lo);
    lo = floor(vmax - 0.5);
    py_hi = lo > (double)(H - 1) ? H - 1 : (lo < -1.0 ? -1 : (int)lo);
    if (px_lo > px_hi || py_lo > py_hi) continue;
    double e0u = u1 - u0, e0v = v1 - v0, e1u = u2 - u1, e1v = v2 - v1, e2u = u0 - u2, e2v = v0 - v2;
    int tl0 = e0v < 0.0 || (e0v == 0.0 && e0u > 0.0);
    int tl1 = e1v < 0.0 || (e1v == 0.0 && e1u > 0.0);
    int tl2 = e2v < 0.0 || (e2v == 0.0 && e2u > 0.0);
    double iz0 = 1.0 / z0, iz1 = 1.0 / z1, iz2 = 1.0 / z2, inv_area = 1.0 / area2;
    if (box) {
      if (px_lo < box[0]) box[0] = px_lo;
      if (py_lo < box[1]) box[1] = py_lo;
      if (px_hi > box[2]) box[2] = px_hi;
      if (py_hi > box[3]) box[3] = py_hi;
    }
    for (int py = py_lo; py <= py_hi; ++py) {
      double sy = py + 0.5;
      for (int px = px_lo; px <= px_hi; ++px) {
        double sx = px + 0.5;
        double w0 = e1u * (sy - v1) - e1v * (sx - u1);
        double w1 = e2u * (sy - v2) - e2v * (sx - u2);
        double w2 = e0u * (sy - v0) - e0v * (sx - u0);
        if (w0 < 0.0 || w1 < 0.0 || w2 < 0.0) continue;
        if ((w0 == 0.0 && !tl1) || (w1 == 0.0 && !tl2) || (w2 == 0.0 && !tl0)) continue;
        double b0 = w0 * inv_area, b1 = w1 * inv_area, b2 = w2 * inv_area;
        double inv_z = b0 * iz0 + b1 * iz1 + b2 * iz2;
        double depth = 1.0 / inv_z;
        size_t o = (size_t)py * W + px;
        if (depth < zbuf[o]) {
          zbuf[o] = depth;
          double s0 = b0 * iz0 * depth, s1 = b1 * iz1 * depth, s2 = b2 * iz2 * depth;
          cbuf[3 * o] = s0 * c0[0] + s1 * c1[0] + s2 * c2[0];
          cbuf[3 * o + 1] = s0 * c0[1] + s1 * c1[1] + s2 * c2[1];
          cbuf[3 * o + 2] = s0 * c0[2] + s1 * c1[2] + s2 * c2[2];
          valid[o] = 1;
          if (owner) owner[o] = ti;
        }
      }
    }
  }
}

/* Full-image single-view raster (raster.py:137-158 minus the sRGB encode):
 * zbuf = +inf / cbuf = linear colour / valid / owner triangle (-1 = none). */
ORC_API void orc_rasterize(const orc_model* m, const double* pose, double fx, double fy, double cx,
                           double cy, int W, int H, double* zbuf, double* cbuf, uint8_t* valid,
                           int32_t* owner) {
  double* vc = (double*)malloc(sizeof(double) * 3 * (size_t)m->V);
  for (int i = 0; i < m->V; ++i) apply_pose(pose, m->verts + 3 * i, vc + 3 * i);
  for (size_t i = 0; i < (size_t)W * H; ++i) {
    zbuf[i] = INFINITY;
    valid[i] = 0;
    owner[i] = -1;
    cbuf[3 * i] = cbuf[3 * i + 1] = cbuf[3 * i + 2] = 0.0;
  }
  raster_kernel(vc, m->tris, m->T, m->col_lin, fx, fy, cx, cy, W, H, zbuf, cbuf, valid, owner, NULL);
  free(vc);
}

/* per-thread scratch: full-size buffers kept clean between candidates (the
 * reference refills the whole image per candidate, raster.py:253-254; only the
 * touched rectangle is reset here, which is equivalent) */
typedef struct {
  int W, H;
  double* zbuf;
  double* cbuf;
  uint8_t* valid;
  double* vc;
  int vcap;
} orc_scratch;

static orc_scratch* scratch_new(int W, int H) {
  orc_scratch* s = (orc_scratch*)calloc(1, sizeof *s);
  s->W = W, s->H = H;
  s->zbuf = (double*)malloc(sizeof(double) * (size_t)W * H);
  s->cbuf = (double*)malloc(sizeof(double) * 3 * (size_t)W * H);
  s->valid = (uint8_t*)calloc((size_t)W * H, 1);
  for (size_t i = 0; i < (size_t)W * H; ++i) s->zbuf[i] = INFINITY;
  return s;
}
static void scratch_free(orc_scratch* s) {
  free(s->zbuf), free(s->cbuf), free(s->valid), free(s->vc), free(s);
}

/* raster.py:239-280: one candidate -> cloud.  Returns n_r, or -1 if cap is too
 * small.  pts/lab (cap,3), src (cap,2). */
static int render_one(const orc_scene* sc, const orc_model* m, const double* pose, int occl,
                      double delta_occ, orc_scratch* s, double* pts, double* lab, int32_t* src,
                      int cap) {
  const int W = sc->W, H = sc->H, st = sc->stride;
  if (s->vcap < m->V) {
    free(s->vc);
    s->vc = (double*)malloc(sizeof(double) * 3 * (size_t)m->V);
    s->vcap = m->V;
  }
  for (int i = 0; i < m->V; ++i) apply_pose(pose, m->verts + 3 * i, s->vc + 3 * i);
  int box[4] = {W, H, -1, -1};
  raster_kernel(s->vc, m->tris, m->T, m->col_lin, sc->fx, sc->fy, sc->cx, sc->cy, W, H, s->zbuf, s->cbuf,
                s->valid, NULL, box);
  int n = 0, overflow = 0;
  if (box[2] >= box[0] && box[3] >= box[1]) {
    if (occl) { /* raster.py:263-270 */
      for (int v = box[1]; v <= box[3]; ++v)
        for (int u = box[0]; u <= box[2]; ++u) {
          size_t o = (size_t)v * W + u;
          if (s->valid[o] && sc->valid[o] && sc->depth[o] < s->zbuf[o] - delta_occ &&
              sc->labels[o] != m->object_id)
            s->valid[o] = 0;
        }
    }
    /* stride sample in row-major order (raster.py:271-279) */
    int v0 = ((box[1] + st - 1) / st) * st, u0 = ((box[0] + st - 1) / st) * st;
    for (int v = v0; v <= box[3]; v += st)
      for (int u = u0; u <= box[2]; u += st) {
        size_t o = (size_t)v * W + u;
        if (!s->valid[o]) continue;
        if (n >= cap) {
          overflow = 1;
          continue;
        }
        double z = s->zbuf[o];
        pts[3 * n] = ((u + 0.5) - sc->cx) * z / sc->fx; /* geometry.py:229-230 */
        pts[3 * n + 1] = ((v + 0.5) - sc->cy) * z / sc->fy;
        pts[3 * n + 2] = z;
        double rgb[3] = {srgb_encode1(s->cbuf[3 * o]), srgb_encode1(s->cbuf[3 * o + 1]),
                         srgb_encode1(s->cbuf[3 * o + 2])};
        orc_srgb_to_lab(rgb, 1, lab + 3 * n);
        src[2 * n] = u, src[2 * n + 1] = v;
        ++n;
      }
    for (int v = box[1]; v <= box[3]; ++v)
      for (int u = box[0]; u <= box[2]; ++u) {
        size_t o = (size_t)v * W + u;
        s->zbuf[o] = INFINITY;
        s->valid[o] = 0;
      }
  }
  return overflow ? -1 : n;
}

ORC_API int orc_render_one(const orc_scene* sc, const orc_model* m, const double* pose, int occl,
                           double delta_occ, double* pts, double* lab, int32_t* src, int cap) {
  orc_scratch* s = scratch_new(sc->W, sc->H);
  int n = render_one(sc, m, pose, occl, delta_occ, s, pts, lab, src, cap);
  scratch_free(s);
  return n;
}

/* ------------------------------------------------------------------------ */
/* exact kNN, neighbors.py:104-134 (bounded sorted insertion, ties -> lowest   */
/* index).  idx (nq,k) int64 filled with -1 / d2 (nq,k) filled with +inf.      */

ORC_API void orc_knn(const double* q, int64_t nq, const double* t, int64_t nt, int k, int64_t* idx,
                     double* d2o) {
  for (int64_t i = 0; i < nq * k; ++i) idx[i] = -1, d2o[i] = INFINITY;
  for (int64_t i = 0; i < nq; ++i) {
    double qx = q[3 * i], qy = q[3 * i + 1], qz = q[3 * i + 2];
    double* od = d2o + i * k;
    int64_t* oi = idx + i * k;
    int cnt = 0;
    for (int64_t j = 0; j < nt; ++j) {
      double dx = t[3 * j] - qx, dy = t[3 * j + 1] - qy, dz = t[3 * j + 2] - qz;
      double d2 = dx * dx + dy * dy + dz * dz;
      int pos;
      if (cnt < k)
        pos = cnt++;
      else if (d2 < od[k - 1])
        pos = k - 1;
      else
        continue;
      while (pos > 0 && od[pos - 1] > d2) od[pos] = od[pos - 1], oi[pos] = oi[pos - 1], --pos;
      od[pos] = d2, oi[pos] = j;
    }
  }
}

/* ------------------------------------------------------------------------ */
/* covariances: registration.py:109-216.  out (n,3,3).  Caller guarantees n>k. */

ORC_API void orc_covariances(const double* pts, int64_t n, int k, double eps, double* out) {
  double* nd = (double*)malloc(sizeof(double) * k);
  int64_t* ni = (int64_t*)malloc(sizeof(int64_t) * k);
  for (int64_t i = 0; i < n; ++i) {
    int cnt = 0;
    for (int64_t j = 0; j < n; ++j) {
      double dx = pts[3 * j] - pts[3 * i], dy = pts[3 * j + 1] - pts[3 * i + 1],
             dz = pts[3 * j + 2] - pts[3 * i + 2];
      double d2 = dx * dx + dy * dy + dz * dz;
      int pos;
      if (cnt < k)
        pos = cnt++;
      else if (d2 < nd[k - 1])
        pos = k - 1;
      else
        continue;
      while (pos > 0 && nd[pos - 1] > d2) nd[pos] = nd[pos - 1], ni[pos] = ni[pos - 1], --pos;
      nd[pos] = d2, ni[pos] = j;
    }
    double mx = 0, my = 0, mz = 0;
    for (int q = 0; q < k; ++q) mx += pts[3 * ni[q]], my += pts[3 * ni[q] + 1], mz += pts[3 * ni[q] + 2];
    mx /= k, my /= k, mz /= k;
    double a[3][3] = {{0}};
    for (int q = 0; q < k; ++q) {
      double dx = pts[3 * ni[q]] - mx, dy = pts[3 * ni[q] + 1] - my, dz = pts[3 * ni[q] + 2] - mz;
      a[0][0] += dx * dx, a[0][1] += dx * dy, a[0][2] += dx * dz;
      a[1][1] += dy * dy, a[1][2] += dy * dz, a[2][2] += dz * dz;
    }
    /* registration.py:158-163: upper entries divided once; the lower ones are
     * read from the (already divided) upper ones and divided again, then
     * overwritten by the symmetric copy */
    for (int u = 0; u < 3; ++u)
      for (int v = u; v < 3; ++v) a[u][v] = a[u][v] / k;
    a[1][0] = a[0][1], a[2][0] = a[0][2], a[2][1] = a[1][2];
    double vm[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
    for (int sweep = 0; sweep < 16; ++sweep) {
      double off = fabs(a[0][1]) + fabs(a[0][2]) + fabs(a[1][2]);
      double scale = fabs(a[0][0]) + fabs(a[1][1]) + fabs(a[2][2]) + 1e-300;
      if (off <= 1e-14 * scale) break;
      for (int p = 0; p < 2; ++p)
        for (int q = p + 1; q < 3; ++q) {
          double apq = a[p][q];
          if (apq == 0.0) continue;
          double theta = (a[q][q] - a[p][p]) / (2.0 * apq), tt;
          if (theta >= 0.0)
            tt = 1.0 / (theta + sqrt(theta * theta + 1.0));
          else
            tt = -1.0 / (-theta + sqrt(theta * theta + 1.0));
          double c = 1.0 / sqrt(tt * tt + 1.0), s = tt * c;
          for (int r = 0; r < 3; ++r) {
            double tmp = a[r][p];
            a[r][p] = c * tmp - s * a[r][q];
            a[r][q] = s * tmp + c * a[r][q];
          }
          for (int r = 0; r < 3; ++r) {
            double tmp = a[p][r];
            a[p][r] = c * tmp - s * a[q][r];
            a[q][r] = s * tmp + c * a[q][r];
          }
          for (int r = 0; r < 3; ++r) {
            double tmp = vm[r][p];
            vm[r][p] = c * tmp - s * vm[r][q];
            vm[r][q] = s * tmp + c * vm[r][q];
          }
        }
    }
    int m = 0;
    if (a[1][1] < a[m][m]) m = 1;
    if (a[2][2] < a[m][m]) m = 2;
    double x = vm[0][m], y = vm[1][m], z = vm[2][m], f = 1.0 - eps;
    double* o = out + 9 * i;
    o[0] = 1.0 - f * x * x, o[1] = -f * x * y, o[2] = -f * x * z;
    o[3] = o[1], o[4] = 1.0 - f * y * y, o[5] = -f * y * z;
    o[6] = o[2], o[7] = o[5], o[8] = 1.0 - f * z * z;
  }
  free(nd), free(ni);
}

/* ------------------------------------------------------------------------ */
/* GICP                                                                       */

/* registration.py:233-338, literal.  r (3,3) row-major, t (3).  h (36), g (6)
 * must be zeroed by the caller.  Returns f0; *n_corr_out = count. */
ORC_API double orc_gicp_linearize(const double* src, int64_t n, const double* tgt, int64_t nt,
                                  const double* ca, const double* cb, const double* r, const double* t,
                                  double gate2, double* h, double* g, int64_t* corr, double* w_buf,
                                  int64_t* n_corr_out) {
  double f0 = 0.0;
  int64_t n_corr = 0;
  for (int64_t i = 0; i < n; ++i) {
    double ax = src[3 * i], ay = src[3 * i + 1], az = src[3 * i + 2];
    double px = r[0] * ax + r[1] * ay + r[2] * az + t[0];
    double py = r[3] * ax + r[4] * ay + r[5] * az + t[1];
    double pz = r[6] * ax + r[7] * ay + r[8] * az + t[2];
    double best = INFINITY;
    int64_t bj = -1;
    for (int64_t j = 0; j < nt; ++j) {
      double dx = tgt[3 * j] - px, dy = tgt[3 * j + 1] - py, dz = tgt[3 * j + 2] - pz;
      double d2 = dx * dx + dy * dy + dz * dz;
      if (d2 < best) best = d2, bj = j;
    }
    if (bj < 0 || best > gate2) {
      corr[i] = -1;
      continue;
    }
    corr[i] = bj;
    ++n_corr;
    double m[3][3], rc[3][3];
    const double* cai = ca + 9 * i;
    const double* cbj = cb + 9 * bj;
    for (int u = 0; u < 3; ++u)
      for (int v = 0; v < 3; ++v) {
        double s = 0.0;
        for (int w = 0; w < 3; ++w) s += r[3 * u + w] * cai[3 * w + v];
        rc[u][v] = s;
      }
    for (int u = 0; u < 3; ++u)
      for (int v = 0; v < 3; ++v) {
        double s = 0.0;
        for (int w = 0; w < 3; ++w) s += rc[u][w] * r[3 * v + w];
        m[u][v] = cbj[3 * u + v] + s;
      }
    double det = (m[0][0] * (m[1][1] * m[2][2] - m[1][2] * m[2][1]) -
                  m[0][1] * (m[1][0] * m[2][2] - m[1][2] * m[2][0]) +
                  m[0][2] * (m[1][0] * m[2][1] - m[1][1] * m[2][0]));
    if (det <= 0.0 || !isfinite(det)) {
      corr[i] = -1;
      --n_corr;
      continue;
    }
    double inv_det = 1.0 / det;
    double* w = w_buf + 9 * i;
    w[0] = (m[1][1] * m[2][2] - m[1][2] * m[2][1]) * inv_det;
    w[1] = (m[0][2] * m[2][1] - m[0][1] * m[2][2]) * inv_det;
    w[2] = (m[0][1] * m[1][2] - m[0][2] * m[1][1]) * inv_det;
    w[3] = (m[1][2] * m[2][0] - m[1][0] * m[2][2]) * inv_det;
    w[4] = (m[0][0] * m[2][2] - m[0][2] * m[2][0]) * inv_det;
    w[5] = (m[0][2] * m[1][0] - m[0][0] * m[1][2]) * inv_det;
    w[6] = (m[1][0] * m[2][1] - m[1][1] * m[2][0]) * inv_det;
    w[7] = (m[0][1] * m[2][0] - m[0][0] * m[2][1]) * inv_det;
    w[8] = (m[0][0] * m[1][1] - m[0][1] * m[1][0]) * inv_det;
    double dx = tgt[3 * bj] - px, dy = tgt[3 * bj + 1] - py, dz = tgt[3 * bj + 2] - pz;
    double J[3][6] = {{0.0, -pz, py, -1.0, 0.0, 0.0}, {pz, 0.0, -px, 0.0, -1.0, 0.0}, {-py, px, 0.0, 0.0, 0.0, -1.0}};
    double wd0 = w[0] * dx + w[1] * dy + w[2] * dz;
    double wd1 = w[3] * dx + w[4] * dy + w[5] * dz;
    double wd2 = w[6] * dx + w[7] * dy + w[8] * dz;
    f0 += dx * wd0 + dy * wd1 + dz * wd2;
    for (int u = 0; u < 6; ++u) g[u] -= J[0][u] * wd0 + J[1][u] * wd1 + J[2][u] * wd2;
    double wj[3][6];
    for (int a = 0; a < 3; ++a)
      for (int u = 0; u < 6; ++u) wj[a][u] = w[3 * a] * J[0][u] + w[3 * a + 1] * J[1][u] + w[3 * a + 2] * J[2][u];
    for (int u = 0; u < 6; ++u)
      for (int v = 0; v < 6; ++v) h[6 * u + v] += J[0][u] * wj[0][v] + J[1][u] * wj[1][v] + J[2][u] * wj[2][v];
  }
  *n_corr_out = n_corr;
  return f0;
}

/* registration.py:387-407 */
static double gicp_objective(const double* src, int64_t n, const double* tgt, const int64_t* corr,
                             const double* w_buf, const double* r, const double* t) {
  double f = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t j = corr[i];
    if (j < 0) continue;
    double ax = src[3 * i], ay = src[3 * i + 1], az = src[3 * i + 2];
    double px = r[0] * ax + r[1] * ay + r[2] * az + t[0];
    double py = r[3] * ax + r[4] * ay + r[5] * az + t[1];
    double pz = r[6] * ax + r[7] * ay + r[8] * az + t[2];
    double dx = tgt[3 * j] - px, dy = tgt[3 * j + 1] - py, dz = tgt[3 * j + 2] - pz;
    const double* w = w_buf + 9 * i;
    double wd0 = w[0] * dx + w[1] * dy + w[2] * dz;
    double wd1 = w[3] * dx + w[4] * dy + w[5] * dz;
    double wd2 = w[6] * dx + w[7] * dy + w[8] * dz;
    f += dx * wd0 + dy * wd1 + dz * wd2;
  }
  return f;
}

/* registration.py:341-361 */
static void so3_exp_fast(double wx, double wy, double wz, double* o) {
  double theta2 = wx * wx + wy * wy + wz * wz, theta = sqrt(theta2), a, b;
  if (theta < 1e-10)
    a = 1.0, b = 0.5;
  else
    a = sin(theta) / theta, b = (1.0 - cos(theta)) / theta2;
  o[0] = 1.0 + b * (-wz * wz - wy * wy);
  o[1] = -a * wz + b * wx * wy;
  o[2] = a * wy + b * wx * wz;
  o[3] = a * wz + b * wx * wy;
  o[4] = 1.0 + b * (-wz * wz - wx * wx);
  o[5] = -a * wx + b * wy * wz;
  o[6] = -a * wy + b * wx * wz;
  o[7] = a * wx + b * wy * wz;
  o[8] = 1.0 + b * (-wy * wy - wx * wx);
}

/* registration.py:364-384 */
static void renorm_rotation(const double* r, double* o) {
  double n0 = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
  double x0 = r[0] / n0, x1 = r[1] / n0, x2 = r[2] / n0;
  double y0 = r[3], y1 = r[4], y2 = r[5];
  double dot = x0 * y0 + x1 * y1 + x2 * y2;
  y0 -= dot * x0, y1 -= dot * x1, y2 -= dot * x2;
  double ny = sqrt(y0 * y0 + y1 * y1 + y2 * y2);
  y0 = y0 / ny, y1 = y1 / ny, y2 = y2 / ny;
  o[0] = x0, o[1] = x1, o[2] = x2, o[3] = y0, o[4] = y1, o[5] = y2;
  o[6] = x1 * y2 - x2 * y1, o[7] = x2 * y0 - x0 * y2, o[8] = x0 * y1 - x1 * y0;
}

/* np.linalg.solve(h, g) (registration.py:487) restated as LAPACK dgesv's
 * published algorithm: LU with partial (row) pivoting, first maximal |a| wins,
 * exact zero pivot = singular.  Returns 0 on success. */
static int solve6(const double* h, const double* g, double* x) {
  double a[6][7];
  for (int i = 0; i < 6; ++i) {
    for (int j = 0; j < 6; ++j) a[i][j] = h[6 * i + j];
    a[i][6] = g[i];
  }
  for (int c = 0; c < 6; ++c) {
    int p = c;
    double best = fabs(a[c][c]);
    for (int i = c + 1; i < 6; ++i)
      if (fabs(a[i][c]) > best) best = fabs(a[i][c]), p = i;
    if (best == 0.0 || isnan(best)) return 1;
    if (p != c)
      for (int j = 0; j < 7; ++j) {
        double tmp = a[c][j];
        a[c][j] = a[p][j], a[p][j] = tmp;
      }
    double inv = 1.0 / a[c][c];
    for (int i = c + 1; i < 6; ++i) {
      double l = a[i][c] * inv;
      a[i][c] = l;
      for (int j = c + 1; j < 7; ++j) a[i][j] = a[i][j] - l * a[c][j];
    }
  }
  for (int i = 5; i >= 0; --i) {
    double s = a[i][6];
    for (int j = i + 1; j < 6; ++j) s = s - a[i][j] * x[j];
    x[i] = s / a[i][i];
  }
  return 0;
}

/* registration.py:479-494 */
static int solve_normal_equations(const double* h, const double* g, double* xi) {
  const double pi2 = M_PI * M_PI;
  for (int damped = 0; damped < 2; ++damped) {
    double hh[36];
    for (int i = 0; i < 36; ++i) hh[i] = h[i] + ((damped && i % 7 == 0) ? 1e-6 : 0.0);
    if (solve6(damped ? hh : h, g, xi)) continue;
    int fin = 1;
    for (int i = 0; i < 6; ++i) fin &= isfinite(xi[i]) != 0;
    if (fin && xi[0] * xi[0] + xi[1] * xi[1] + xi[2] * xi[2] < pi2 &&
        xi[3] * xi[3] + xi[4] * xi[4] + xi[5] * xi[5] < 1.0)
      return 0;
  }
  return 1;
}

/* nearest rotation (geometry.py:82-89 uses LAPACK SVD; restated as the polar
 * factor by Newton iteration X <- (X + X^-T)/2, which converges to the same
 * matrix U V^T; the input is within 1e-12 of a rotation, so 3 steps reach
 * machine precision) */
static void orthonormalize3(const double* r, double* o) {
  double x[9];
  memcpy(x, r, sizeof x);
  for (int it = 0; it < 3; ++it) {
    double c[9] = {x[4] * x[8] - x[5] * x[7], x[5] * x[6] - x[3] * x[8], x[3] * x[7] - x[4] * x[6],
                   x[2] * x[7] - x[1] * x[8], x[0] * x[8] - x[2] * x[6], x[1] * x[6] - x[0] * x[7],
                   x[1] * x[5] - x[2] * x[4], x[2] * x[3] - x[0] * x[5], x[0] * x[4] - x[1] * x[3]};
    double det = x[0] * c[0] + x[1] * c[1] + x[2] * c[2];
    for (int i = 0; i < 9; ++i) x[i] = 0.5 * (x[i] + c[i] / det); /* cofactor/det = X^-T */
  }
  memcpy(o, x, sizeof x);
}

enum { ORC_OK = 0, ORC_TOO_FEW = 1, ORC_DEGENERATE = 2, ORC_SINGULAR = 3, ORC_NO_DECREASE = 4 };

typedef struct {
  int32_t k_cov, max_iter;
  double eps, tol_t, tol_r, gate;
} orc_gicp_cfg;

/* registration.py:410-476 with init = (r0, t0).  out_T = 3x4 [orthonormalize(r)|t].
 * trace (may be NULL): 2*max_iter doubles (f0, f_try) per accepted step.
 * Returns failure code; *iters, *converged set. */
ORC_API int orc_gicp_align(const double* src, int64_t n, const double* tgt, int64_t nt, const double* ca,
                           const double* cb, const double* init, const orc_gicp_cfg* cfg, double* out_T,
                           int32_t* iters, int32_t* converged, double* trace, int32_t* n_trace,
                           double* r_raw) {
  double gate2 = cfg->gate * cfg->gate;
  double r_cur[9], t_cur[3];
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) r_cur[3 * i + j] = init[4 * i + j];
    t_cur[i] = init[4 * i + 3];
  }
  *converged = 0, *iters = 0;
  if (n_trace) *n_trace = 0;
  if (n < 3 || nt < 3) {
    memcpy(out_T, init, 12 * sizeof(double));
    return ORC_DEGENERATE;
  }
  int failure = ORC_OK;
  int64_t* corr = (int64_t*)malloc(sizeof(int64_t) * n);
  double* w_buf = (double*)malloc(sizeof(double) * 9 * n);
  double r_try[9], t_try[3];
  for (int it = 1; it <= cfg->max_iter; ++it) {
    *iters = it;
    double h[36] = {0}, g[6] = {0}, xi[6];
    int64_t n_corr;
    double f0 = orc_gicp_linearize(src, n, tgt, nt, ca, cb, r_cur, t_cur, gate2, h, g, corr, w_buf, &n_corr);
    if (n_corr < 6) {
      failure = ORC_DEGENERATE;
      break;
    }
    if (solve_normal_equations(h, g, xi)) {
      failure = ORC_SINGULAR;
      break;
    }
    int accepted = 0;
    double scale = 1.0, f_try = 0.0;
    for (int tr = 0; tr < 9; ++tr) {
      double rs[9];
      so3_exp_fast(scale * xi[0], scale * xi[1], scale * xi[2], rs);
      for (int i = 0; i < 3; ++i) { /* r_step @ r_cur, r_step @ t_cur + scale*xi[3:] */
        for (int j = 0; j < 3; ++j)
          r_try[3 * i + j] = dot_f012(rs[3 * i], rs[3 * i + 1], rs[3 * i + 2], r_cur[j], r_cur[3 + j], r_cur[6 + j]);
        t_try[i] = dot_f102(rs[3 * i], rs[3 * i + 1], rs[3 * i + 2], t_cur[0], t_cur[1], t_cur[2]) + scale * xi[3 + i];
      }
      f_try = gicp_objective(src, n, tgt, corr, w_buf, r_try, t_try);
      if (isfinite(f_try) && f_try <= f0) {
        accepted = 1;
        break;
      }
      scale *= 0.5;
    }
    if (!accepted) {
      failure = ORC_NO_DECREASE;
      break;
    }
    renorm_rotation(r_try, r_cur);
    memcpy(t_cur, t_try, sizeof t_cur);
    if (trace) trace[2 * (it - 1)] = f0, trace[2 * (it - 1) + 1] = f_try;
    if (n_trace) *n_trace = it;
    double step_t2 = scale * scale * (xi[3] * xi[3] + xi[4] * xi[4] + xi[5] * xi[5]);
    double step_r2 = scale * scale * (xi[0] * xi[0] + xi[1] * xi[1] + xi[2] * xi[2]);
    if (step_t2 < cfg->tol_t * cfg->tol_t && step_r2 < cfg->tol_r * cfg->tol_r) {
      *converged = 1;
      break;
    }
    if (it >= 5 && f0 > 0.0 && (f0 - f_try) <= 1e-4 * f0) break;
  }
  free(corr), free(w_buf);
  double ro[9];
  orthonormalize3(r_cur, ro);
  if (r_raw) memcpy(r_raw, r_cur, sizeof r_cur);
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) out_T[4 * i + j] = ro[3 * i + j];
    out_T[4 * i + 3] = t_cur[i];
  }
  return failure;
}

/* registration.py:59-67 (rms residual at the final transform) */
ORC_API double orc_rms_residual(const double* src, int64_t n, const double* tgt, int64_t nt, const double* T,
                                double gate) {
  double sum = 0.0;
  int64_t cnt = 0;
  /* numpy mean of d2[mask]: pairwise summation is not restated; callers compare
   * to 1e-12 relative */
  for (int64_t i = 0; i < n; ++i) {
    double p[3];
    apply_pose(T, src + 3 * i, p);
    double best = INFINITY;
    for (int64_t j = 0; j < nt; ++j) {
      double dx = tgt[3 * j] - p[0], dy = tgt[3 * j + 1] - p[1], dz = tgt[3 * j + 2] - p[2];
      double d2 = dx * dx + dy * dy + dz * dz;
      if (d2 < best) best = d2;
    }
    if (best <= gate * gate) sum += best, ++cnt;
  }
  return cnt ? sqrt(sum / (double)cnt) : INFINITY;
}

/* search.py:291-301: cam = reg o cam; 3-DoF: world = c2w o cam; planar; cam = w2c o lift.
 * c2w_vec_order / w2c_vec_order: 0 = rotation stored C-contiguous, 1 = transposed view. */
ORC_API void orc_refine_apply(const double* reg_T, const double* cam_in, int mode3dof, const double* c2w,
                              int c2w_vec_order, const double* w2c, int w2c_vec_order, double fixed_z,
                              double* cam_out) {
  double cam[12];
  compose_pose(reg_T, cam_in, 0, cam);
  if (mode3dof) {
    double world[12], lift[12];
    compose_pose(c2w, cam, c2w_vec_order, world);
    double yaw = atan2(world[4], world[0]); /* registration.py:556 */
    double y = fmod(yaw, 2.0 * M_PI);       /* geometry.py:98-105 */
    if (y < 0.0) y += 2.0 * M_PI;
    if (y >= 2.0 * M_PI) y -= 2.0 * M_PI;
    double c = cos(y), s = sin(y);
    double l[12] = {c, -s, 0.0, world[3], s, c, 0.0, world[7], 0.0, 0.0, 1.0, fixed_z};
    memcpy(lift, l, sizeof l);
    compose_pose(w2c, lift, w2c_vec_order, cam);
  }
  memcpy(cam_out, cam, sizeof cam);
}

/* ------------------------------------------------------------------------ */
/* cost: cost.py:91-152                                                       */

/* rendered_cost with the reference's AABB pre-crop.  explained (n_obs) bytes,
 * zeroed here.  `inbox` scratch (n_obs int32).  Returns j_r. */
static int rendered_cost(const double* rp, const double* rlab, int n_r, const double* op,
                         const double* olab, int64_t n_obs, double delta, double tau_c, int use_color,
                         uint8_t* explained, int32_t* inbox, int32_t* touched, int* n_touched) {
  *n_touched = 0;
  if (n_r == 0) return 0;
  if (n_obs == 0) return n_r;
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int i = 0; i < n_r; ++i)
    for (int a = 0; a < 3; ++a) {
      double v = rp[3 * i + a];
      if (v < lo[a]) lo[a] = v;
      if (v > hi[a]) hi[a] = v;
    }
  for (int a = 0; a < 3; ++a) lo[a] = lo[a] - delta, hi[a] = hi[a] + delta;
  int64_t nb = 0;
  for (int64_t j = 0; j < n_obs; ++j) {
    const double* p = op + 3 * j;
    if (p[0] >= lo[0] && p[0] <= hi[0] && p[1] >= lo[1] && p[1] <= hi[1] && p[2] >= lo[2] && p[2] <= hi[2])
      inbox[nb++] = (int32_t)j;
  }
  if (nb == 0) return n_r;
  int within = 0, color_fail = 0;
  double d2max = delta * delta;
  for (int i = 0; i < n_r; ++i) {
    double qx = rp[3 * i], qy = rp[3 * i + 1], qz = rp[3 * i + 2], best = INFINITY;
    int64_t bj = -1;
    for (int64_t c = 0; c < nb; ++c) {
      const double* p = op + 3 * (int64_t)inbox[c];
      double dx = p[0] - qx, dy = p[1] - qy, dz = p[2] - qz;
      double d2 = dx * dx + dy * dy + dz * dz;
      if (d2 < best) best = d2, bj = inbox[c];
    }
    if (bj < 0 || !(best <= d2max)) continue;
    ++within;
    if (use_color && !(orc_ciede2000(rlab + 3 * i, olab + 3 * bj) <= tau_c)) {
      ++color_fail;
      continue;
    }
    if (!explained[bj]) explained[bj] = 1, touched[(*n_touched)++] = (int32_t)bj;
  }
  return n_r - within + color_fail;
}

ORC_API int orc_rendered_cost(const double* rp, const double* rlab, int n_r, const double* op,
                              const double* olab, int64_t n_obs, double delta, double tau_c, int use_color,
                              uint8_t* explained) {
  memset(explained, 0, (size_t)n_obs);
  int32_t* inbox = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_obs + 1));
  int32_t* touched = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_r + 1));
  int nt;
  int jr = rendered_cost(rp, rlab, n_r, op, olab, n_obs, delta, tau_c, use_color, explained, inbox, touched, &nt);
  free(inbox), free(touched);
  return jr;
}

/* cost.py:138-152 cylinder mode: pose^-1 applied to every observed point */
ORC_API int orc_observed_cost_cyl(const double* op, int64_t n_obs, const double* pose, double r2, double zmin,
                                  double zmax, const uint8_t* explained, uint8_t* selected_out) {
  /* inverse(): rt = R^T view; t_inv = (-rt) @ t in F-view order k=0,1,2 (geometry.py:143-145) */
  double ti[3];
  for (int i = 0; i < 3; ++i) ti[i] = dot_f012(-pose[i], -pose[4 + i], -pose[8 + i], pose[3], pose[7], pose[11]);
  int cnt = 0;
  for (int64_t j = 0; j < n_obs; ++j) {
    const double* p = op + 3 * j;
    /* p @ rt.T = p @ R: out[c] = sum_k p[k] R[k][c] */
    double x = dot_f012(p[0], p[1], p[2], pose[0], pose[4], pose[8]) + ti[0];
    double y = dot_f012(p[0], p[1], p[2], pose[1], pose[5], pose[9]) + ti[1];
    double z = dot_f012(p[0], p[1], p[2], pose[2], pose[6], pose[10]) + ti[2];
    int sel = (x * x + y * y <= r2) && z >= zmin && z <= zmax;
    if (selected_out) selected_out[j] = (uint8_t)sel;
    if (sel && !explained[j]) ++cnt;
  }
  return cnt;
}

/* ------------------------------------------------------------------------ */
/* threaded search driver: search.py:217-377 restricted to the per-candidate   */
/* stages (render, refine, re-render, cost).  Proposal generation, target       */
/* cropping and the argmin stay in the Python wrapper.                          */

typedef struct {
  int32_t mode3dof, use_color, occluder_marking, refine;
  double delta, tau_c;
  orc_gicp_cfg gicp;
  double c2w[12], w2c[12];
  int32_t c2w_vec_order, w2c_vec_order;
  double fixed_z;
  int32_t n_threads, cloud_cap;
} orc_search_cfg;

typedef struct {
  const orc_scene* sc;
  const orc_model* models;
  int64_t N;
  const int32_t* model_slot;
  const double* poses;
  int32_t n_targets;
  const int64_t* tgt_off;
  const double* tgt_pts;
  const int32_t* tgt_idx;
  double** tgt_cov; /* per target, NULL if too few points */
  const orc_search_cfg* cfg;
  double* refined;
  double* reg_T;
  int32_t *iters, *flags, *j_o, *j_r, *n_first, *n_final;
  int64_t next;     /* atomic work counter */
  int64_t next_tgt; /* atomic target counter */
  double stage_s[4];
  pthread_mutex_t mu;
} job_t;

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

static void* cov_worker(void* arg) {
  job_t* J = (job_t*)arg;
  for (;;) {
    int64_t t = __atomic_fetch_add(&J->next_tgt, 1, __ATOMIC_RELAXED);
    if (t >= J->n_targets) break;
    int64_t n = J->tgt_off[t + 1] - J->tgt_off[t];
    if (n <= J->cfg->gicp.k_cov) {
      J->tgt_cov[t] = NULL;
      continue;
    }
    J->tgt_cov[t] = (double*)malloc(sizeof(double) * 9 * n);
    orc_covariances(J->tgt_pts + 3 * J->tgt_off[t], n, J->cfg->gicp.k_cov, J->cfg->gicp.eps, J->tgt_cov[t]);
  }
  return NULL;
}

static void* cand_worker(void* arg) {
  job_t* J = (job_t*)arg;
  const orc_search_cfg* cfg = J->cfg;
  const orc_scene* sc = J->sc;
  const int cap = cfg->cloud_cap;
  orc_scratch* s = scratch_new(sc->W, sc->H);
  double* pts = (double*)malloc(sizeof(double) * 3 * cap);
  double* lab = (double*)malloc(sizeof(double) * 3 * cap);
  int32_t* src = (int32_t*)malloc(sizeof(int32_t) * 2 * cap);
  double* cov = (double*)malloc(sizeof(double) * 9 * cap);
  uint8_t* explained = (uint8_t*)calloc((size_t)sc->n_obs + 1, 1);
  int32_t* inbox = (int32_t*)malloc(sizeof(int32_t) * ((size_t)sc->n_obs + 1));
  int32_t* touched = (int32_t*)malloc(sizeof(int32_t) * (cap + 1));
  double st[4] = {0, 0, 0, 0};
  const int64_t CH = 4;
  for (;;) {
    int64_t c0 = __atomic_fetch_add(&J->next, CH, __ATOMIC_RELAXED);
    if (c0 >= J->N) break;
    int64_t c1 = c0 + CH < J->N ? c0 + CH : J->N;
    for (int64_t c = c0; c < c1; ++c) {
      const orc_model* m = J->models + J->model_slot[c];
      const double* pose_in = J->poses + 12 * c;
      double pose[12];
      memcpy(pose, pose_in, sizeof pose);
      double t0 = now_s();
      int n = render_one(sc, m, pose, cfg->occluder_marking, cfg->delta, s, pts, lab, src, cap);
      double t1 = now_s();
      st[0] += t1 - t0;
      J->n_first[c] = n;
      J->iters[c] = 0, J->flags[c] = 0;
      static const double I12[12] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0};
      memcpy(J->reg_T + 12 * c, I12, sizeof I12);
      if (n < 0) {
        J->flags[c] = -1; /* capacity overflow: reported, never silent */
        n = 0;
      }
      if (cfg->refine) {
        int fail;
        int32_t it = 0, conv = 0;
        double T[12];
        memcpy(T, I12, sizeof T);
        int ti = J->tgt_idx[c];
        if (n <= cfg->gicp.k_cov || J->tgt_cov[ti] == NULL) {
          fail = ORC_TOO_FEW; /* registration.py:504-510 */
        } else {
          orc_covariances(pts, n, cfg->gicp.k_cov, cfg->gicp.eps, cov);
          int64_t nt = J->tgt_off[ti + 1] - J->tgt_off[ti];
          fail = orc_gicp_align(pts, n, J->tgt_pts + 3 * J->tgt_off[ti], nt, cov, J->tgt_cov[ti], I12,
                                &cfg->gicp, T, &it, &conv, NULL, NULL, NULL);
        }
        J->iters[c] = it;
        J->flags[c] = fail | (conv ? 0x100 : 0);
        if (!(fail == ORC_TOO_FEW && it == 0)) { /* search.py:292-301 */
          memcpy(J->reg_T + 12 * c, T, sizeof T);
          orc_refine_apply(T, pose_in, cfg->mode3dof, cfg->c2w, cfg->c2w_vec_order, cfg->w2c,
                           cfg->w2c_vec_order, cfg->fixed_z, pose);
        }
        double t2 = now_s();
        st[1] += t2 - t1;
        n = render_one(sc, m, pose, cfg->occluder_marking, cfg->delta, s, pts, lab, src, cap);
        if (n < 0) J->flags[c] = -1, n = 0;
        t1 = now_s();
        st[2] += t1 - t2;
      }
      memcpy(J->refined + 12 * c, pose, sizeof pose);
      J->n_final[c] = n;
      int nt_;
      int jr = rendered_cost(pts, lab, n, sc->obs_pts, sc->obs_lab, sc->n_obs, cfg->delta, cfg->tau_c,
                             cfg->use_color, explained, inbox, touched, &nt_);
      int jo = 0;
      if (cfg->mode3dof) {
        jo = orc_observed_cost_cyl(sc->obs_pts, sc->n_obs, pose, m->cyl_r2, m->cyl_zmin, m->cyl_zmax, explained,
                                   NULL);
      } else { /* search.py:197-199 */
        for (int64_t j = 0; j < sc->n_obs; ++j)
          if (sc->obs_labels[j] == m->object_id && !explained[j]) ++jo;
      }
      for (int q = 0; q < nt_; ++q) explained[touched[q]] = 0;
      J->j_r[c] = jr, J->j_o[c] = jo;
      st[3] += now_s() - t1;
    }
  }
  pthread_mutex_lock(&J->mu);
  for (int i = 0; i < 4; ++i) J->stage_s[i] += st[i];
  pthread_mutex_unlock(&J->mu);
  scratch_free(s);
  free(pts), free(lab), free(src), free(cov), free(explained), free(inbox), free(touched);
  return NULL;
}

ORC_API int orc_search(const orc_scene* sc, const orc_model* models, int64_t N, const int32_t* model_slot,
                       const double* poses, int32_t n_targets, const int64_t* tgt_off, const double* tgt_pts,
                       const int32_t* tgt_idx, const orc_search_cfg* cfg, double* refined, double* reg_T,
                       int32_t* iters, int32_t* flags, int32_t* j_o, int32_t* j_r, int32_t* n_first,
                       int32_t* n_final, double* stage_seconds /* [5]: render, refine, rerender, cost (thread-summed), target covs (wall) */) {
  job_t J;
  memset(&J, 0, sizeof J);
  J.sc = sc, J.models = models, J.N = N, J.model_slot = model_slot, J.poses = poses;
  J.n_targets = n_targets, J.tgt_off = tgt_off, J.tgt_pts = tgt_pts, J.tgt_idx = tgt_idx, J.cfg = cfg;
  J.refined = refined, J.reg_T = reg_T, J.iters = iters, J.flags = flags, J.j_o = j_o, J.j_r = j_r;
  J.n_first = n_first, J.n_final = n_final;
  pthread_mutex_init(&J.mu, NULL);
  int nth = cfg->n_threads > 0 ? cfg->n_threads : 1;
  if (nth > 256) nth = 256;
  pthread_t th[256];
  double t0 = now_s();
  J.tgt_cov = (double**)calloc((size_t)(n_targets > 0 ? n_targets : 1), sizeof(double*));
  if (cfg->refine && n_targets > 0) {
    for (int i = 0; i < nth; ++i) pthread_create(&th[i], NULL, cov_worker, &J);
    for (int i = 0; i < nth; ++i) pthread_join(th[i], NULL);
  }
  double t1 = now_s();
  for (int i = 0; i < nth; ++i) pthread_create(&th[i], NULL, cand_worker, &J);
  for (int i = 0; i < nth; ++i) pthread_join(th[i], NULL);
  for (int i = 0; i < n_targets; ++i) free(J.tgt_cov[i]);
  free(J.tgt_cov);
  if (stage_seconds) {
    for (int i = 0; i < 4; ++i) stage_seconds[i] = J.stage_s[i];
    stage_seconds[4] = t1 - t0;
  }
  pthread_mutex_destroy(&J.mu);
  return 0;
}
