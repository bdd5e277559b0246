// px_common.cuh -- shared device helpers for libpx (sm_100a).
//
// All arithmetic on this path is IEEE binary64.  The translation units are
// compiled with -fmad=false so that `a*b+c` is two roundings, exactly like the
// reference's numba kernels (which contain no contraction);
// where the reference goes through numpy matmul the fused order observed on the
// host BLAS is written out with __fma_rn (dot_f012 / dot_f102 below).
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#define PX_NEAR_PLANE 1e-4
#define PX_WARP 32

namespace px {

// sum_k a_k*b_k fused in the order k = 0,1,2: numpy (V,3)@R.T, mat@mat,
// transposed-view @ vec (geometry.py:131-141 evaluated by OpenBLAS)
__device__ __forceinline__ double dot_f012(double a0, double a1, double a2, double b0, double b1, double b2) {
  return __fma_rn(a2, b2, __fma_rn(a1, b1, __dmul_rn(a0, b0)));
}
// order k = 1,0,2: numpy C-contiguous (3,3) @ (3,)
__device__ __forceinline__ double dot_f102(double a0, double a1, double a2, double b0, double b1, double b2) {
  return __fma_rn(a2, b2, __fma_rn(a0, b0, __dmul_rn(a1, b1)));
}

// y = R x + t for a row-major 3x4 pose, numpy `p @ R.T + t` rounding
__device__ __forceinline__ void apply_pose(const double* __restrict__ P, double x0, double x1, double x2,
                                           double& y0, double& y1, double& y2) {
  y0 = dot_f012(x0, x1, x2, P[0], P[1], P[2]) + P[3];
  y1 = dot_f012(x0, x1, x2, P[4], P[5], P[6]) + P[7];
  y2 = dot_f012(x0, x1, x2, P[8], P[9], P[10]) + P[11];
}

// C = A o B (geometry.py:136-141).  vec_order 0: A's rotation is C-contiguous on
// the host (matvec k = 1,0,2); 1: transposed view (k = 0,1,2).
__device__ __forceinline__ void compose_pose(const double* A, const double* B, int vec_order, double* C) {
  double out[12];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double a0 = A[4 * i], a1 = A[4 * i + 1], a2 = A[4 * i + 2];
#pragma unroll
    for (int j = 0; j < 3; ++j) out[4 * i + j] = dot_f012(a0, a1, a2, B[j], B[4 + j], B[8 + j]);
    double rt = vec_order ? dot_f012(a0, a1, a2, B[3], B[7], B[11]) : dot_f102(a0, a1, a2, B[3], B[7], B[11]);
    out[4 * i + 3] = rt + A[4 * i + 3];
  }
#pragma unroll
  for (int i = 0; i < 12; ++i) C[i] = out[i];
}

__device__ __forceinline__ unsigned long long dbits(double x) { return (unsigned long long)__double_as_longlong(x); }
__device__ __forceinline__ double bits_d(unsigned long long b) { return __longlong_as_double((long long)b); }

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

struct Camera {
  double fx, fy, cx, cy;
  int W, H, stride, GW, GH;  // GW/GH: stride-grid dimensions ceil(W/stride), ceil(H/stride)
  double ray_k;              // stride / (max(fx,fy) * sqrt(max over the image of 1+a^2+b^2)) * (1 - 1e-9)
};

}  // namespace px
