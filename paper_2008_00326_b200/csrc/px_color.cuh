// px_color.cuh -- per-point colour maths on the device.
// Reference: pkg/src/rvpose/colorspace.py:29-124.  The transcendental calls
// (pow, cbrt, hypot, atan2, sin, cos, exp) are CUDA libdevice's; the reference
// uses numpy's SIMD/libm versions, which differ in the last ulp, so Lab and
// dE agree to ~1e-12 relative, not bit for bit.  They only feed the
// `dE <= tau_c` gate (cost.py:127-129).
#pragma once
#include "px_common.cuh"

namespace px {

__device__ __forceinline__ double srgb_encode1(double c) {  // colorspace.py:35-38
  c = c < 0.0 ? 0.0 : (c > 1.0 ? 1.0 : c);
  return c <= 0.0031308 ? 12.92 * c : 1.055 * pow(c, 1.0 / 2.4) - 0.055;
}
__device__ __forceinline__ double srgb_decode1(double c) {  // colorspace.py:29-32
  return c <= 0.04045 ? c / 12.92 : pow((c + 0.055) / 1.055, 2.4);
}

// sRGB in [0,1] -> CIELAB (D65), colorspace.py:41-55
__device__ __forceinline__ void srgb_to_lab(double r, double g, double b, double& L, double& A, double& B) {
  const double l0 = srgb_decode1(r), l1 = srgb_decode1(g), l2 = srgb_decode1(b);
  const double d = 6.0 / 29.0;
  const double d3 = d * d * d, lin_div = 3.0 * d * d, off = 4.0 / 29.0;
  const double x = dot_f012(l0, l1, l2, 0.4124564, 0.3575761, 0.1804375) / 0.95047;
  const double y = dot_f012(l0, l1, l2, 0.2126729, 0.7151522, 0.0721750) / 1.0;
  const double z = dot_f012(l0, l1, l2, 0.0193339, 0.1191920, 0.9503041) / 1.08883;
  const double f0 = x > d3 ? cbrt(x) : x / lin_div + off;
  const double f1 = y > d3 ? cbrt(y) : y / lin_div + off;
  const double f2 = z > d3 ? cbrt(z) : z / lin_div + off;
  L = 116.0 * f1 - 16.0;
  A = 500.0 * (f0 - f1);
  B = 200.0 * (f1 - f2);
}

__device__ __forceinline__ double pymod360(double x) {  // numpy `% 360.0`
  double m = fmod(x, 360.0);
  if (m != 0.0) {
    if (m < 0.0) m += 360.0;
  } else {
    m = 0.0;
  }
  return m;
}

// CIEDE2000 with k_L = k_C = k_H = 1, colorspace.py:58-124
__device__ __forceinline__ double ciede2000(double L1, double a1, double b1, double L2, double a2, double b2) {
  const double P25_7 = 6103515625.0;  // 25**7
  const double R2D = 180.0 / CUDART_PI, D2R = CUDART_PI / 180.0;
  const double c1 = hypot(a1, b1), c2 = hypot(a2, b2);
  const double cb = 0.5 * (c1 + c2);
  const double cb7 = pow(cb, 7.0);
  const double g = 0.5 * (1.0 - sqrt(cb7 / (cb7 + P25_7)));
  const double a1p = (1.0 + g) * a1, a2p = (1.0 + g) * a2;
  const double c1p = hypot(a1p, b1), c2p = hypot(a2p, b2);
  double h1 = pymod360(atan2(b1, a1p) * R2D), h2 = pymod360(atan2(b2, a2p) * R2D);
  if (a1p == 0.0 && b1 == 0.0) h1 = 0.0;
  if (a2p == 0.0 && b2 == 0.0) h2 = 0.0;
  const double dL = L2 - L1, dC = c2p - c1p;
  const bool grey = (c1p * c2p) == 0.0;
  double dh = h2 - h1;
  // |h2 - h1| > 180 decides two branches (colorspace.py:91-92, :97-99).  For (near-)antipodal hues the rounded angles
  // sit on that threshold and the last bit of atan2 (libdevice here, libm / SVML in numpy) would pick the branch --
  // e.g. published pair 14, (50, -0.001, 2.49) vs (50, 0.001, -2.49), whose hue difference is exactly 180.  Within
  // 1e-9 degrees of the threshold the decision is therefore taken on the exact sign of the cross product of the two
  // chroma vectors: |dh| > 180 iff the turn from h1 to h2 overshoots the half circle.
  bool over = fabs(dh) > 180.0;
  if (fabs(fabs(dh) - 180.0) < 1e-9) {
    const double p = a1p * b2, q = a2p * b1;
    const double cross = (p - q) + (fma(a1p, b2, -p) - fma(a2p, b1, -q));  // error-free products: exact sign
    over = cross != 0.0 && ((cross < 0.0) == (dh > 0.0));
  }
  if (over) dh += dh > 0.0 ? -360.0 : 360.0;
  if (grey) dh = 0.0;
  const double dH = 2.0 * sqrt(c1p * c2p) * sin((0.5 * dh) * D2R);
  const double Lm = 0.5 * (L1 + L2), Cm = 0.5 * (c1p + c2p);
  const double hs = h1 + h2;
  double hm = !over ? 0.5 * hs : (hs < 360.0 ? 0.5 * (hs + 360.0) : 0.5 * (hs - 360.0));
  if (grey) hm = hs;
  const double t = 1.0 - 0.17 * cos((hm - 30.0) * D2R) + 0.24 * cos((2.0 * hm) * D2R) +
                   0.32 * cos((3.0 * hm + 6.0) * D2R) - 0.20 * cos((4.0 * hm - 63.0) * D2R);
  const double q = (hm - 275.0) / 25.0;
  const double dth = 30.0 * exp(-(q * q));
  const double Cm7 = pow(Cm, 7.0);
  const double rc = 2.0 * sqrt(Cm7 / (Cm7 + P25_7));
  const double lm50 = (Lm - 50.0) * (Lm - 50.0);
  const double sl = 1.0 + 0.015 * lm50 / sqrt(20.0 + lm50);
  const double sc = 1.0 + 0.045 * Cm;
  const double sh = 1.0 + 0.015 * Cm * t;
  const double rt = -sin((2.0 * dth) * D2R) * rc;
  const double tl = dL / sl, tc = dC / sc, th = dH / sh;
  return sqrt(tl * tl + tc * tc + th * th + rt * tc * th);
}

}  // namespace px
