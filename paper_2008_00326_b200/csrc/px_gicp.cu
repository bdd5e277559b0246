// px_gicp.cu -- k-NN covariances and batched many-to-many GICP refinement.
//
// Replaces registration._covariance_kernel / _gicp_linearize / _gicp_objective /
// gicp_align / _m2m_task (reference pkg/src/rvpose/registration.py:109-511) and
// the refine-apply + 3-DoF re-lift of search.py:291-301 for a whole batch.
//
// One warp per candidate.  Everything that is order-sensitive in the reference
// is evaluated in the reference's order:
//   * nearest neighbour = lexicographic min of (d2, index) (strict `<` scan);
//   * the 36 H / 6 g / f0 accumulators are sums over the source index in
//     ascending order: per-point terms are computed lane-parallel, staged
//     through shared memory (transposed, padded), and 43 lanes then add their
//     entry serially in index order -- bit-identical to the scalar loop;
//   * the fixed-association objective is summed in index order via shuffles.
// numpy products in gicp_align (r_step @ r_cur, r_step @ t_cur) use the host
// BLAS fused orders (px_common.cuh); np.linalg.solve is LAPACK dgesv's
// algorithm (partial-pivot LU); orthonormalize is the polar projection.
// Compiled with -fmad=false.
#include <algorithm>
#include <cstdio>
#include <cstring>

#include "px_kernels.h"

#ifdef PX_NO_STREAM_HINTS  // experiment: default cache policy for the per-iteration scratch (L2-blocked chunks)
#define PX_LDCS(p) (*(p))
#define PX_STCS(p, v) (*(p) = (v))
#else
#define PX_LDCS(p) __ldcs(p)
#define PX_STCS(p, v) __stcs(p, v)
#endif

namespace px {

enum { F_OK = 0, F_TOO_FEW = 1, F_DEGENERATE = 2, F_SINGULAR = 3, F_NO_DECREASE = 4 };

// registration.py:206-216: C = I - (1 - eps) v0 v0^T, written entry by entry.  The matrix is a pure function
// of (v0, eps), so the GICP scratch and the target planes keep the 3 doubles of v0 instead of the 6 distinct
// entries and the linearise kernel re-evaluates these very expressions (same bits, a third less traffic).
__device__ __forceinline__ void cov_from_normal(double x, double y, double z, double f, double* __restrict__ out) {
  out[0] = 1.0 - f * x * x, out[1] = -f * x * y, out[2] = -f * x * z;
  out[3] = out[1], out[4] = 1.0 - f * y * y, out[5] = -f * y * z;
  out[6] = out[2], out[7] = out[5], out[8] = 1.0 - f * z * z;
}

// registration.py:117-216 for point i of a cloud of n points (n > k); out = covariance (9) + v0 (3)
__device__ void cov_point(const double* __restrict__ pts, int n, int i, int k, double eps, double* __restrict__ out) {
  double nd[PX_KCOV_MAX];
  int ni[PX_KCOV_MAX];
  const double xi = pts[3 * i], yi = pts[3 * i + 1], zi = pts[3 * i + 2];
  int cnt = 0;
  double worst = CUDART_INF;
  for (int j = 0; j < n; ++j) {
    const double dx = pts[3 * j] - xi, dy = pts[3 * j + 1] - yi, dz = pts[3 * j + 2] - zi;
    const double d2 = dx * dx + dy * dy + dz * dz;
    int pos;
    if (cnt < k)
      pos = cnt++;
    else if (d2 < worst)
      pos = k - 1;
    else
      continue;
    while (pos > 0 && nd[pos - 1] > d2) nd[pos] = nd[pos - 1], ni[pos] = ni[pos - 1], --pos;
    nd[pos] = d2, ni[pos] = j;
    if (cnt == k) worst = nd[k - 1];
  }
  double mx = 0.0, my = 0.0, mz = 0.0;
  for (int q = 0; q < k; ++q) mx += pts[3 * ni[q]], my += pts[3 * ni[q] + 1], mz += pts[3 * ni[q] + 2];
  const double kd = (double)k;
  mx /= kd, my /= kd, mz /= kd;
  double a00 = 0, a01 = 0, a02 = 0, a11 = 0, a12 = 0, a22 = 0;
  for (int q = 0; q < k; ++q) {
    const double dx = pts[3 * ni[q]] - mx, dy = pts[3 * ni[q] + 1] - my, dz = pts[3 * ni[q] + 2] - mz;
    a00 += dx * dx, a01 += dx * dy, a02 += dx * dz, a11 += dy * dy, a12 += dy * dz, a22 += dz * dz;
  }
  double a[3][3], vm[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  a[0][0] = a00 / kd, a[0][1] = a01 / kd, a[0][2] = a02 / kd;
  a[1][1] = a11 / kd, a[1][2] = a12 / kd, a[2][2] = a22 / kd;
  a[1][0] = a[0][1], a[2][0] = a[0][2], a[2][1] = a[1][2];
  for (int sweep = 0; sweep < 16; ++sweep) {
    const double off = fabs(a[0][1]) + fabs(a[0][2]) + fabs(a[1][2]);
    const double scale = fabs(a[0][0]) + fabs(a[1][1]) + fabs(a[2][2]) + 1e-300;
    if (off <= 1e-14 * scale) break;
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
      for (int q = p + 1; q < 3; ++q) {
        const double apq = a[p][q];
        if (apq == 0.0) continue;
        const double theta = (a[q][q] - a[p][p]) / (2.0 * apq);
        double tt;
        if (theta >= 0.0)
          tt = 1.0 / (theta + sqrt(theta * theta + 1.0));
        else
          tt = -1.0 / (-theta + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(tt * tt + 1.0), s = tt * c;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          const double tmp = a[r][p];
          a[r][p] = c * tmp - s * a[r][q];
          a[r][q] = s * tmp + c * a[r][q];
        }
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          const double tmp = a[p][r];
          a[p][r] = c * tmp - s * a[q][r];
          a[q][r] = s * tmp + c * a[q][r];
        }
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          const double tmp = vm[r][p];
          vm[r][p] = c * tmp - s * vm[r][q];
          vm[r][q] = s * tmp + c * vm[r][q];
        }
      }
  }
  double dmin = a[0][0], x = vm[0][0], y = vm[1][0], z = vm[2][0];
  if (a[1][1] < dmin) dmin = a[1][1], x = vm[0][1], y = vm[1][1], z = vm[2][1];
  if (a[2][2] < dmin) dmin = a[2][2], x = vm[0][2], y = vm[1][2], z = vm[2][2];
  cov_from_normal(x, y, z, 1.0 - eps, out);
  out[9] = x, out[10] = y, out[11] = z;
}

// ---------------------------------------------------------------------------
// Organised views.  Rendered clouds and GICP targets are subsets of a pixel grid
// (stride-grid pixels of the candidate's screen box / of the observed frame), so
// neighbourhoods can be enumerated by pixel rings.  Everything below is EXACT:
// a ring search stops only when the distance already found is strictly smaller
// than a lower bound on the distance to every pixel not yet visited.
//
// Bound: p = z (a, b, 1) in normalised image coordinates; a point on the ray of a
// pixel whose normalised offset from p is (da, db) is at least
// z * sqrt(da^2 + db^2) / sqrt(1 + a_j^2 + b_j^2) away.  Camera::ray_k folds the
// stride, max(fx, fy), the image-wide bound on 1 + a^2 + b^2 and a 1e-9 safety
// factor: a pixel >= m grid steps away (Chebyshev) is >= z * m * ray_k distant.

// The same bound restricted to a window of the stride grid [gx0, gx0+w) x [gy0, gy0+h): every point of an organised
// cloud that lives inside that window sits on the ray of one of ITS pixel centres, so 1 + a_j^2 + b_j^2 only has to
// be bounded over the window, not over the whole image (1.52 at the corners of a 60-degree camera, ~1.0-1.2 for an
// object near the principal point): rings end sooner, ~20 % fewer cells are visited.  Same safety factor.
__device__ __forceinline__ double window_ray_k(const Camera& cam, int gx0, int gy0, int w, int h) {
  const double u0 = (double)(gx0 * cam.stride) + 0.5, u1 = (double)((gx0 + w - 1) * cam.stride) + 0.5;
  const double v0 = (double)(gy0 * cam.stride) + 0.5, v1 = (double)((gy0 + h - 1) * cam.stride) + 0.5;
  const double am = fmax(fabs(u0 - cam.cx), fabs(u1 - cam.cx)) / cam.fx, bm = fmax(fabs(v0 - cam.cy), fabs(v1 - cam.cy)) / cam.fy;
  return (double)cam.stride / (fmax(cam.fx, cam.fy) * sqrt(1.0 + am * am + bm * bm)) * (1.0 - 1e-9);
}

struct OrgView {
  const double* pts;   // (n,3) points in local-index order (row-major pixel order)
  const int32_t* map;  // (h,w) local index or -1
  int w, h;
};

// k nearest (d2, index)-lexicographic neighbours of point i sitting at map cell
// (cx, cy); identical to the reference's brute-force insertion scan
// (registration.py:117-142).  nd/ni come back sorted ascending.
// S = element stride of the nd / ni lists (1: thread-local arrays; 32: one column per lane of a
// warp-shared staging area, which keeps the lists out of the small L1).
template <int S>
__device__ __forceinline__ void knn_ring(const OrgView& V, int i, int cx, int cy, int k, double ray_k, double* nd, int* ni) {
  const double xi = V.pts[3 * i], yi = V.pts[3 * i + 1], zi = V.pts[3 * i + 2];
  int cnt = 0;
  double worst = CUDART_INF;
  int worst_j = 0x7fffffff;
  const int wmax = max(max(cx, V.w - 1 - cx), max(cy, V.h - 1 - cy));
  for (int w = 0; w <= wmax; ++w) {
    const int y0 = cy - w, y1 = cy + w, x0 = cx - w, x1 = cx + w;
    for (int y = max(y0, 0); y <= min(y1, V.h - 1); ++y) {
      const bool edge_row = (y == y0 || y == y1);
      const int step = edge_row ? 1 : max(2 * w, 1);
      for (int x = x0; x <= x1; x += step) {
        if (x < 0 || x >= V.w) continue;
        const int j = V.map[y * V.w + x];
        if (j < 0) continue;
        const double dx = V.pts[3 * j] - xi, dy = V.pts[3 * j + 1] - yi, dz = V.pts[3 * j + 2] - zi;
        const double d2 = dx * dx + dy * dy + dz * dz;
        int pos;
        if (cnt < k)
          pos = cnt++;
        else if (d2 < worst || (d2 == worst && j < worst_j))
          pos = k - 1;
        else
          continue;
        while (pos > 0 && (nd[(pos - 1) * S] > d2 || (nd[(pos - 1) * S] == d2 && ni[(pos - 1) * S] > j)))
          nd[pos * S] = nd[(pos - 1) * S], ni[pos * S] = ni[(pos - 1) * S], --pos;
        nd[pos * S] = d2, ni[pos * S] = j;
        if (cnt == k) worst = nd[(k - 1) * S], worst_j = ni[(k - 1) * S];
      }
    }
    if (cnt == k) {
      const double D = zi * (double)(w + 1) * ray_k;
      if (worst < D * D) break;
    }
  }
}

// Same search over a DENSE copy of an organised cloud: three planes of w*h doubles (NaN where the map is
// empty) instead of map -> compact index -> point.  The distance comes straight from the cell (one
// dependent load less per visited cell, NaN fails every comparison); the compact index is only
// fetched for the cells that enter the list.
template <int S, typename IdxT = int>
__device__ __forceinline__ void knn_ring_dense(const double* __restrict__ G, long long plane, const int32_t* __restrict__ map,
                                               int W, int H, double xi, double yi, double zi, int cx, int cy, int k,
                                               double ray_k, double* nd, IdxT* ni) {
  int cnt = 0;
  double worst = CUDART_INF;
  int worst_j = 0x7fffffff;
  const int wmax = max(max(cx, W - 1 - cx), max(cy, H - 1 - cy));
  for (int w = 0; w <= wmax; ++w) {
    const int y0 = cy - w, y1 = cy + w, x0 = cx - w, x1 = cx + w;
    for (int y = max(y0, 0); y <= min(y1, H - 1); ++y) {
      const bool edge_row = (y == y0 || y == y1);
      const int step = edge_row ? 1 : max(2 * w, 1);
      for (int x = x0; x <= x1; x += step) {
        if (x < 0 || x >= W) continue;
        const int cell = y * W + x;
        const double dx = G[cell] - xi, dy = G[plane + cell] - yi, dz = G[2 * plane + cell] - zi;
        const double d2 = dx * dx + dy * dy + dz * dz;
        if (cnt < k ? !(d2 == d2) : !(d2 <= worst)) continue;  // empty cell, or farther than the k-th
        const int j = map[cell];
        int pos;
        if (cnt < k)
          pos = cnt++;
        else if (d2 < worst || j < worst_j)
          pos = k - 1;
        else
          continue;
        while (pos > 0 && (nd[(pos - 1) * S] > d2 || (nd[(pos - 1) * S] == d2 && (int)ni[(pos - 1) * S] > j)))
          nd[pos * S] = nd[(pos - 1) * S], ni[pos * S] = ni[(pos - 1) * S], --pos;
        nd[pos * S] = d2, ni[pos * S] = (IdxT)j;
        if (cnt == k) worst = nd[(k - 1) * S], worst_j = (int)ni[(k - 1) * S];
      }
    }
    if (cnt == k) {
      const double D = zi * (double)(w + 1) * ray_k;
      if (worst < D * D) break;
    }
  }
}

// mean / covariance / Jacobi / regularised output for a sorted neighbour list
// (registration.py:143-216)
template <int S, typename IdxT = int>
__device__ __forceinline__ void cov_from_neighbours(const double* __restrict__ pts, const IdxT* ni, int k, double eps,
                                                    double* __restrict__ out) {
  double mx = 0.0, my = 0.0, mz = 0.0;
  for (int q = 0; q < k; ++q) mx += pts[3 * ni[q * S]], my += pts[3 * ni[q * S] + 1], mz += pts[3 * ni[q * S] + 2];
  const double kd = (double)k;
  mx /= kd, my /= kd, mz /= kd;
  double a00 = 0, a01 = 0, a02 = 0, a11 = 0, a12 = 0, a22 = 0;
  for (int q = 0; q < k; ++q) {
    const double dx = pts[3 * ni[q * S]] - mx, dy = pts[3 * ni[q * S] + 1] - my, dz = pts[3 * ni[q * S] + 2] - mz;
    a00 += dx * dx, a01 += dx * dy, a02 += dx * dz, a11 += dy * dy, a12 += dy * dz, a22 += dz * dz;
  }
  double a[3][3], vm[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  a[0][0] = a00 / kd, a[0][1] = a01 / kd, a[0][2] = a02 / kd;
  a[1][1] = a11 / kd, a[1][2] = a12 / kd, a[2][2] = a22 / kd;
  a[1][0] = a[0][1], a[2][0] = a[0][2], a[2][1] = a[1][2];
  for (int sweep = 0; sweep < 16; ++sweep) {
    const double off = fabs(a[0][1]) + fabs(a[0][2]) + fabs(a[1][2]);
    const double scale = fabs(a[0][0]) + fabs(a[1][1]) + fabs(a[2][2]) + 1e-300;
    if (off <= 1e-14 * scale) break;
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
      for (int q = p + 1; q < 3; ++q) {
        const double apq = a[p][q];
        if (apq == 0.0) continue;
        const double theta = (a[q][q] - a[p][p]) / (2.0 * apq);
        double tt;
        if (theta >= 0.0)
          tt = 1.0 / (theta + sqrt(theta * theta + 1.0));
        else
          tt = -1.0 / (-theta + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(tt * tt + 1.0), s = tt * c;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          const double tmp = a[r][p];
          a[r][p] = c * tmp - s * a[r][q];
          a[r][q] = s * tmp + c * a[r][q];
        }
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          const double tmp = a[p][r];
          a[p][r] = c * tmp - s * a[q][r];
          a[q][r] = s * tmp + c * a[q][r];
        }
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          const double tmp = vm[r][p];
          vm[r][p] = c * tmp - s * vm[r][q];
          vm[r][q] = s * tmp + c * vm[r][q];
        }
      }
  }
  double dmin = a[0][0], x = vm[0][0], y = vm[1][0], z = vm[2][0];
  if (a[1][1] < dmin) dmin = a[1][1], x = vm[0][1], y = vm[1][1], z = vm[2][1];
  if (a[2][2] < dmin) dmin = a[2][2], x = vm[0][2], y = vm[1][2], z = vm[2][2];
  cov_from_normal(x, y, z, 1.0 - eps, out);
  out[9] = x, out[10] = y, out[11] = z;
}

__device__ void cov_point_org(const OrgView& V, int i, int cx, int cy, int k, double eps, double ray_k, double* __restrict__ out) {
  double nd[PX_KCOV_MAX];
  int ni[PX_KCOV_MAX];
  knn_ring<1>(V, i, cx, cy, k, ray_k, nd, ni);
  cov_from_neighbours<1>(V.pts, ni, k, eps, out);
}
// same, with the neighbour lists in a warp-shared area (column `lane`, stride 32)
__device__ void cov_point_org_sm(const OrgView& V, int i, int cx, int cy, int k, double eps, double ray_k,
                                 double* __restrict__ out, double* nd, int* ni) {
  knn_ring<32>(V, i, cx, cy, k, ray_k, nd, ni);
  cov_from_neighbours<32>(V.pts, ni, k, eps, out);
}

__device__ __forceinline__ void store_cov(const CovArgs& a, long long i, const double* cv) {
#pragma unroll
  for (int q = 0; q < 9; ++q) a.cov[9 * i + q] = cv[q];
  if (a.v0) a.v0[3 * i] = cv[9], a.v0[3 * i + 1] = cv[10], a.v0[3 * i + 2] = cv[11];
}

// one CTA per target cloud, threads over its points
#ifndef PX_COV_MINB
#define PX_COV_MINB 4
#endif
__global__ void __launch_bounds__(128, PX_COV_MINB) cov_kernel(CovArgs a) {
  const int c = blockIdx.x;
  const long long off = a.offset[c];
  const int n = a.count ? a.count[c] : (int)(a.offset[c + 1] - off);
  if (n <= a.k) return;
  const bool org = a.org != nullptr && a.org[c].w > 0;
  if (org) {
    const TgtOrg o = a.org[c];
    OrgView V{a.points + 3 * off, a.tmap + o.map_off, o.w, o.h};
    const double ray_k = a.cam.stride > 0 ? window_ray_k(a.cam, o.gx0, o.gy0, o.w, o.h) : a.ray_k;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int cell = a.tpix[off + i];
      double cv[12];
      cov_point_org(V, i, cell % o.w, cell / o.w, a.k, a.eps, ray_k, cv);
      store_cov(a, off + i, cv);
    }
  } else {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      double cv[12];
      cov_point(a.points + 3 * off, n, i, a.k, a.eps, cv);
      store_cov(a, off + i, cv);
    }
  }
}

cudaError_t launch_cov(const CovArgs& a, long long, cudaStream_t st) {
  if (a.n_clouds == 0) return cudaSuccess;
  cov_kernel<<<a.n_clouds, 128, 0, st>>>(a);
  return cudaGetLastError();
}

__global__ void soa_kernel(const double* __restrict__ pts, const double* __restrict__ v0, double* __restrict__ soa, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  soa[i] = pts[3 * i], soa[n + i] = pts[3 * i + 1], soa[2 * n + i] = pts[3 * i + 2];
  soa[3 * n + i] = v0[3 * i], soa[4 * n + i] = v0[3 * i + 1], soa[5 * n + i] = v0[3 * i + 2];
}

cudaError_t launch_soa(const double* pts, const double* v0, double* soa, long long n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  soa_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(pts, v0, soa, n);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Exact nearest neighbour over an organised target with a two-level box
// hierarchy in image space: blocks of PX_BLK x PX_BLK map cells and super-blocks
// of PX_BLK x PX_BLK blocks, each with the 3-D bounding box of its points.  A
// node is opened only if the squared distance from the query to its box is <=
// the current cut-off; that box distance, evaluated with the same operation
// order as the point distance, can never exceed the point distance of any
// member (floating-point subtraction, multiplication and addition are
// monotone), so no candidate is ever skipped.

#ifdef PX_NN_STATS
__device__ unsigned long long g_nn_stats[8];
__device__ unsigned long long g_nn_rhist[8];
__device__ double g_nn_rayk;
__device__ float* g_nn_prevq;
__device__ unsigned long long g_nn_mhist[8];  // queries, with-prev, sb tests, blk tests, leaf pts, found, leaves opened
__device__ unsigned long long g_nn_lhist[32];  // leaves opened per query: [seeded?][found?][bucket 0,1,2,3-4,5-8,9-16,17-32,33+]
#define NN_STAT(i, v) atomicAdd(&g_nn_stats[i], (unsigned long long)(v))
#else
#define NN_STAT(i, v)
#endif

__device__ __forceinline__ double box_dist2(const double* __restrict__ b, double qx, double qy, double qz) {
  // b = {xlo, ylo, zlo, xhi, yhi, zhi}; empty boxes hold +inf / -inf and give +inf
  const double dx = fmax(fmax(b[0] - qx, qx - b[3]), 0.0);
  const double dy = fmax(fmax(b[1] - qy, qy - b[4]), 0.0);
  const double dz = fmax(fmax(b[2] - qz, qz - b[5]), 0.0);
  return dx * dx + dy * dy + dz * dz;
}

// fp32 squared distance from a point to a box stored as {lo xyz, hi xyz}; lo was rounded down and hi up when the
// box was converted, so the fp32 box contains the exact one and this never exceeds the exact squared distance to
// any member point by more than the threshold slack.
__device__ __forceinline__ float box_dist2f(const float* __restrict__ b, float qx, float qy, float qz) {
  const float2 b0 = __ldg(reinterpret_cast<const float2*>(b)), b1 = __ldg(reinterpret_cast<const float2*>(b) + 1),
               b2 = __ldg(reinterpret_cast<const float2*>(b) + 2);
  const float gx = fmaxf(fmaxf(b0.x - qx, qx - b1.y), 0.f);
  const float gy = fmaxf(fmaxf(b0.y - qy, qy - b2.x), 0.f);
  const float gz = fmaxf(fmaxf(b1.x - qz, qz - b2.y), 0.f);
  return fmaf(gz, gz, fmaf(gy, gy, gx * gx));
}

// Blackwell's two-wide fp32 arithmetic (FADD2 / FMUL2 / FFMA2: one issue slot for two IEEE-rounded results) on
// register pairs; the pruning tests below run on pairs of boxes / pairs of leaf points.
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk2(float lo, float hi) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void upk2(f32x2 v, float& lo, float& hi) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }
__device__ __forceinline__ f32x2 sub2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
  f32x2 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
// squared distances of a query to two boxes {lo, hi} (per axis: max(lo - q, q - hi, 0)), two-wide
__device__ __forceinline__ f32x2 box_pair_dist2(f32x2 lx, f32x2 ly, f32x2 lz, f32x2 hx, f32x2 hy, f32x2 hz, f32x2 qx,
                                                f32x2 qy, f32x2 qz) {
  float a0, a1, b0, b1;
  upk2(sub2(lx, qx), a0, a1), upk2(sub2(qx, hx), b0, b1);
  const f32x2 gx = pk2(fmaxf(fmaxf(a0, b0), 0.f), fmaxf(fmaxf(a1, b1), 0.f));
  upk2(sub2(ly, qy), a0, a1), upk2(sub2(qy, hy), b0, b1);
  const f32x2 gy = pk2(fmaxf(fmaxf(a0, b0), 0.f), fmaxf(fmaxf(a1, b1), 0.f));
  upk2(sub2(lz, qz), a0, a1), upk2(sub2(qz, hz), b0, b1);
  const f32x2 gz = pk2(fmaxf(fmaxf(a0, b0), 0.f), fmaxf(fmaxf(a1, b1), 0.f));
  return fma2(gz, gz, fma2(gy, gy, mul2(gx, gx)));
}
// squared distances of a query to two points, two-wide
__device__ __forceinline__ f32x2 pt_pair_dist2(f32x2 x, f32x2 y, f32x2 z, f32x2 qx, f32x2 qy, f32x2 qz) {
  const f32x2 tx = sub2(x, qx), ty = sub2(y, qy), tz = sub2(z, qz);
  return fma2(tz, tz, fma2(ty, ty, mul2(tx, tx)));
}

// Lexicographic minimum of (d2, index) over the target points with d2 <= gate2,
// identical to the reference's brute-force scan (registration.py:251-260)
// whenever that scan's winner passes the gate; bj = -1 if no point is within the
// gate.  `prev` (last iteration's correspondence, or -1) seeds the cut-off.
//
// Pruning runs in fp32 on conservatively rounded copies (boxes as {lo, hi} rounded
// outwards, points as fixed 16-cell leaf records of fp32 planes), two boxes / two
// points per instruction (FADD2 / FMUL2 / FFMA2): with e = T.org.err bounding every
// rounding involved, a node or point whose fp32 squared distance exceeds
//     thr = roundup_f32((sqrt(best) + 2e)^2 * (1 + 2^-20))
// is provably farther than `best` in exact arithmetic, so it can neither beat nor
// tie the current winner; everything else is evaluated in fp64 with the
// reference's operation order on the original coordinates.  Results are therefore
// bit-identical to the linear scan (tests: organised == generic).
// Upper bound on sqrt(x): the hardware approximation (MUFU, relative error <= 2^-23 -- PTX ISA, sqrt.approx.f32)
// times (1 + 2^-22), rounded up.  An IEEE square root with directed rounding is a ~15-instruction software routine,
// and the thresholds below are recomputed for every leaf that improves the search.
__device__ __forceinline__ float sqrt_upper(float x) {
  float s;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(s) : "f"(x));
  return __fmul_ru(s, 1.0000002384185791015625f);
}
// e2 = 2 err rounded up (once per query)
__device__ __forceinline__ float nn_threshold(double best, float e2) {
  // every step rounds towards +inf (or over-estimates), so the fp32 result is >= (sqrt(best) + 2 err)^2 (1 + 2^-20) in
  // exact arithmetic: a looser threshold only lets a few more nodes through to the exact fp64 evaluation
  const float s = __fadd_ru(sqrt_upper(__double2float_ru(best)), e2);
  return __fmul_ru(__fmul_ru(s, s), 1.00000095367431640625f);
}

// The converse bound: a point whose fp32 squared distance is mm lies at most sqrt(U), U = (sqrt(mm) + 2e)^2 (1 + 2^-20),
// away in exact arithmetic (the same two-sided rounding bound e), so once such a point is known nothing farther than
// U can win, and every point within U has an fp32 squared distance <= nn_threshold(U) <= the value returned here:
// sqrt(U) + 2e <= (sqrt(mm) + 4e)(1 + 2^-21), rounded up throughout.
__device__ __forceinline__ float nn_threshold_f32(float mm, float e2) {
  const float s = __fmul_ru(__fadd_ru(__fadd_ru(sqrt_upper(mm), e2), e2), 1.0000019073486328125f);
  return __fmul_ru(__fmul_ru(s, s), 1.00000095367431640625f);
}

__device__ __forceinline__ void nn_target(const TargetsDev& T, int ti, long long toff, int nt, double qx, double qy,
                                          double qz, int prev, double gate2, double& best, int& bj) {
  const double* P = T.points + 3 * toff;
  const TgtOrg o = T.org ? T.org[ti] : TgtOrg{0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0.0};
  if (o.w > 0) {
    // search state: (best, bj) = lexicographically smallest (d2, index) seen with d2 <= gate2
    best = gate2, bj = 0x7fffffff;
    NN_STAT(0, 1);
    if (prev >= 0) {
      NN_STAT(1, 1);
      const double dx = P[3 * prev] - qx, dy = P[3 * prev + 1] - qy, dz = P[3 * prev + 2] - qz;
      const double d2 = dx * dx + dy * dy + dz * dz;
      if (d2 <= best) best = d2, bj = prev;
    }
    const float e2 = __double2float_ru(2.0 * o.err);
    float thr = nn_threshold(best, e2);
#ifdef PX_NN_STATS
    int n_leaves_ = 0, n_improved_ = 0;
#endif
    // the query in the frame of the fp32 structures (TargetsDev::rot; the exact evaluations below stay in the original frame)
    const float qxf = (float)(T.rot[0] * qx + T.rot[1] * qy + T.rot[2] * qz);
    const float qyf = (float)(T.rot[3] * qx + T.rot[4] * qy + T.rot[5] * qz);
    const float qzf = (float)(T.rot[6] * qx + T.rot[7] * qy + T.rot[8] * qz);
    const int32_t* map = T.tmap + o.map_off;
    // boxes: per super-block six planes {lox,loy,loz,hix,hiy,hiz} x 16 block slots, then the super-blocks' {lo, hi};
    // leaves: one fixed record per block slot, three planes {x, y, z} x 16 map cells of the block (row-major;
    // cells without a point hold a far-away sentinel), so a leaf is 12 vector loads and 8 two-wide distance
    // evaluations without loop control; the local index of a survivor comes from the pixel map
    const float* bb = T.boxes32 + 6 * o.box_off;
    const float* sb = bb + 96 * (long long)o.sw * o.sh;
    const ulonglong2* leaves = reinterpret_cast<const ulonglong2*>(T.leaf32) + 12 * o.box_off;
    const f32x2 QX = pk2(qxf, qxf), QY = pk2(qyf, qyf), QZ = pk2(qzf, qzf);
    for (int sy = 0; sy < o.sh; ++sy)
      for (int sx = 0; sx < o.sw; ++sx) {
        NN_STAT(2, 1);
        const int sbi = sy * o.sw + sx;
        if (box_dist2f(sb + 6 * sbi, qxf, qyf, qzf) > thr) continue;
        // phase 1: test the 16 block slots of this super-block back to back -- vector loads, independent
        // arithmetic, no control flow (slots outside the map hold empty boxes) -- survivors into a bit mask
        const ulonglong2* pl = reinterpret_cast<const ulonglong2*>(bb + 96 * sbi);
        unsigned bmask = 0;
#ifndef PX_NN_NO_NEAREST_FIRST
        unsigned kmin = 0xffffffffu;  // (box distance bits, low 4 bits = slot) of the nearest block: non-negative floats order like their bits
#define PX_KMIN(d, slot) kmin = min(kmin, (__float_as_uint(d) & ~15u) | (unsigned)(slot))
#else
#define PX_KMIN(d, slot) (void)0
#endif
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const ulonglong2 lx = __ldg(pl + g), ly = __ldg(pl + 4 + g), lz = __ldg(pl + 8 + g);
          const ulonglong2 hx = __ldg(pl + 12 + g), hy = __ldg(pl + 16 + g), hz = __ldg(pl + 20 + g);
          float d0, d1, d2_, d3;
          upk2(box_pair_dist2(lx.x, ly.x, lz.x, hx.x, hy.x, hz.x, QX, QY, QZ), d0, d1);
          upk2(box_pair_dist2(lx.y, ly.y, lz.y, hx.y, hy.y, hz.y, QX, QY, QZ), d2_, d3);
          if (!(d0 > thr)) bmask |= 1u << (4 * g);
          if (!(d1 > thr)) bmask |= 2u << (4 * g);
          if (!(d2_ > thr)) bmask |= 4u << (4 * g);
          if (!(d3 > thr)) bmask |= 8u << (4 * g);
          PX_KMIN(d0, 4 * g), PX_KMIN(d1, 4 * g + 1), PX_KMIN(d2_, 4 * g + 2), PX_KMIN(d3, 4 * g + 3);
        }
#undef PX_KMIN
        NN_STAT(3, PX_BLK * PX_BLK);
#ifndef PX_NN_NO_NEAREST_FIRST
        // The NEAREST block is opened first -- its leaf usually holds the winner, and the threshold tightened there
        // closes most of the other blocks that passed the test above: each of those is re-tested (six scalar loads)
        // against the current threshold before its 192-byte leaf is fetched.  The warp waits for the lane that opens
        // the most leaves, so this is worth more than the leaves it saves on average.
        const float thr_blk = thr;  // the threshold the mask was built with
        bool first = true;
#endif
        while (bmask) {
#ifndef PX_NN_NO_NEAREST_FIRST
          int q;
          if (first) {
            q = (int)(kmin & 15u), first = false;  // its bit is set: the mask is not empty and it is the minimum
          } else {
            q = __ffs(bmask) - 1;
          }
          bmask &= ~(1u << q);
          if (thr < thr_blk) {
            const float* bf = bb + 96 * sbi + q;
            const float gx = fmaxf(fmaxf(__ldg(bf) - qxf, qxf - __ldg(bf + 48)), 0.f);
            const float gy = fmaxf(fmaxf(__ldg(bf + 16) - qyf, qyf - __ldg(bf + 64)), 0.f);
            const float gz = fmaxf(fmaxf(__ldg(bf + 32) - qzf, qzf - __ldg(bf + 80)), 0.f);
            if (fmaf(gz, gz, fmaf(gy, gy, gx * gx)) > thr) continue;
          }
#else
          const int q = __ffs(bmask) - 1;
          bmask &= bmask - 1;
#endif
          NN_STAT(4, 16);
          NN_STAT(6, 1);
          // phase 1 over the leaf record (16 cells): fp32 squared distances two at a time, survivors into a mask
          const ulonglong2* lr = leaves + 12 * (16 * sbi + q);
          unsigned pmask = 0;
#ifndef PX_NN_NO_LEAFMIN
          {
            float d[16];
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              const ulonglong2 X = __ldg(lr + g), Y = __ldg(lr + 4 + g), Z = __ldg(lr + 8 + g);
              upk2(pt_pair_dist2(X.x, Y.x, Z.x, QX, QY, QZ), d[4 * g], d[4 * g + 1]);
              upk2(pt_pair_dist2(X.y, Y.y, Z.y, QX, QY, QZ), d[4 * g + 2], d[4 * g + 3]);
            }
            const float m0 = fminf(fminf(d[0], d[1]), d[2]), m1 = fminf(fminf(d[3], d[4]), d[5]), m2 = fminf(fminf(d[6], d[7]), d[8]);
            const float m3 = fminf(fminf(d[9], d[10]), d[11]), m4 = fminf(fminf(d[12], d[13]), d[14]);
            const float mm = fminf(fminf(fminf(m0, m1), m2), fminf(fminf(m3, m4), d[15]));
            if (mm > thr) continue;  // most opened leaves hold no point within the threshold
            // the leaf's fp32-closest point is at most U = (sqrt(mm) + 2e)^2 (1 + 2^-20) away in exact arithmetic, so
            // nothing farther than U can win: tighten the threshold BEFORE the exact evaluations (typically one
            // survivor -- that point -- instead of every point closer than the seed)
            thr = fminf(thr, nn_threshold_f32(mm, e2));
#pragma unroll
            for (int k = 0; k < 16; ++k)
              if (!(d[k] > thr)) pmask |= 1u << k;
          }
#else
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const ulonglong2 X = __ldg(lr + g), Y = __ldg(lr + 4 + g), Z = __ldg(lr + 8 + g);
            float d0, d1, d2_, d3;
            upk2(pt_pair_dist2(X.x, Y.x, Z.x, QX, QY, QZ), d0, d1);
            upk2(pt_pair_dist2(X.y, Y.y, Z.y, QX, QY, QZ), d2_, d3);
            if (!(d0 > thr)) pmask |= 1u << (4 * g);
            if (!(d1 > thr)) pmask |= 2u << (4 * g);
            if (!(d2_ > thr)) pmask |= 4u << (4 * g);
            if (!(d3 > thr)) pmask |= 8u << (4 * g);
          }
#endif
          // phase 2: exact fp64 evaluation of the few survivors, reference operation order
          if (pmask) {
            const int cell0 = ((sy * PX_BLK + (q >> 2)) * PX_BLK) * o.w + (sx * PX_BLK + (q & 3)) * PX_BLK;
            bool improved = false;
            do {
              const int k = __ffs(pmask) - 1;
              pmask &= pmask - 1;
              const int j = __ldg(map + cell0 + (k >> 2) * o.w + (k & 3));
              if (j < 0) continue;  // cannot happen while thr is finite (gate <= PX_GATE_MAX): an absent cell is infinitely far
              const double dx = P[3 * j] - qx, dy = P[3 * j + 1] - qy, dz = P[3 * j + 2] - qz;
              const double d2 = dx * dx + dy * dy + dz * dz;
              if (d2 < best || (d2 == best && j < bj)) best = d2, bj = j, improved = true;
            } while (pmask);
            if (improved) thr = fminf(thr, nn_threshold(best, e2));
#ifdef PX_NN_STATS
            n_improved_ += improved;
#endif
          }
#ifdef PX_NN_STATS
          ++n_leaves_;
#endif
        }
      }
    if (bj == 0x7fffffff) best = CUDART_INF, bj = -1;
    NN_STAT(5, bj >= 0);
#ifdef PX_NN_STATS
    NN_STAT(7, n_improved_);
    {
      const int L = n_leaves_;
      const int b_ = L == 0 ? 0 : L == 1 ? 1 : L == 2 ? 2 : L <= 4 ? 3 : L <= 8 ? 4 : L <= 16 ? 5 : L <= 32 ? 6 : 7;
      atomicAdd(&g_nn_lhist[(prev >= 0 ? 16 : 0) + (bj >= 0 ? 8 : 0) + b_], 1ull);
    }
    {
      int b_ = 7;
      if (bj >= 0) {
        const double R = sqrt(best) / (qz * g_nn_rayk);
        b_ = R < 0.5 ? 0 : R < 1.5 ? 1 : R < 2.5 ? 2 : R < 3.5 ? 3 : R < 5.5 ? 4 : R < 8.5 ? 5 : 6;
      }
      atomicAdd(&g_nn_rhist[b_], 1ull);
    }
#endif
    return;
  }
  // generic clouds: the reference's linear scan
  best = CUDART_INF, bj = -1;
  for (int j = 0; j < nt; ++j) {
    const double dx = P[3 * j] - qx, dy = P[3 * j + 1] - qy, dz = P[3 * j + 2] - qz;
    const double d2 = dx * dx + dy * dy + dz * dz;
    if (d2 < best) best = d2, bj = j;
  }
}

#define STAGE_LD 33
#define WARP_SM_DOUBLES (43 * STAGE_LD + 43 + 8)

// LAPACK dgesv restated: partial-pivot LU, first maximal |a| wins, zero pivot = singular.
// Fully unrolled with compile-time indices so the 6x7 augmented matrix lives in registers
// (a dynamically indexed copy sat in local memory and cost a fifth of the linearise kernel);
// the row exchange is a chain of predicated swaps.  Same operations, same order.
__device__ __forceinline__ int solve6(const double* h, double diag_add, const double* g, double* x) {
  double a[6][7];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
#pragma unroll
    for (int j = 0; j < 6; ++j) a[i][j] = h[6 * i + j] + (i == j ? diag_add : 0.0);
    a[i][6] = g[i];
  }
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    int p = c;
    double best = fabs(a[c][c]);
#pragma unroll
    for (int i = c + 1; i < 6; ++i)
      if (fabs(a[i][c]) > best) best = fabs(a[i][c]), p = i;
    if (best == 0.0 || isnan(best)) return 1;
#pragma unroll
    for (int i = c + 1; i < 6; ++i) {
      // masked XOR exchange on the bit patterns: a select chain gets turned back into a dynamically
      // indexed (local-memory) array by the compiler
      const long long sw = -(long long)(p == i);
#pragma unroll
      for (int j = c; j < 7; ++j) {  // columns left of c hold multipliers that are never read again
        const long long u = __double_as_longlong(a[c][j]), v = __double_as_longlong(a[i][j]);
        const long long d = (u ^ v) & sw;
        a[c][j] = __longlong_as_double(u ^ d), a[i][j] = __longlong_as_double(v ^ d);
      }
    }
    const double inv = 1.0 / a[c][c];
#pragma unroll
    for (int i = c + 1; i < 6; ++i) {
      const double l = a[i][c] * inv;
#pragma unroll
      for (int j = c + 1; j < 7; ++j) a[i][j] = a[i][j] - l * a[c][j];
    }
  }
#pragma unroll
  for (int i = 5; i >= 0; --i) {
    double s_ = a[i][6];
#pragma unroll
    for (int j = i + 1; j < 6; ++j) s_ = s_ - a[i][j] * x[j];
    x[i] = s_ / a[i][i];
  }
  return 0;
}

// registration.py:479-494
__device__ int solve_normal_equations(const double* h, const double* g, double* xi) {
  const double pi2 = CUDART_PI * CUDART_PI;
  for (int damped = 0; damped < 2; ++damped) {
    if (solve6(h, damped ? 1e-6 : 0.0, g, xi)) continue;
    bool fin = true;
    for (int i = 0; i < 6; ++i) fin = fin && isfinite(xi[i]);
    if (fin && xi[0] * xi[0] + xi[1] * xi[1] + xi[2] * xi[2] < pi2 &&
        xi[3] * xi[3] + xi[4] * xi[4] + xi[5] * xi[5] < 1.0)
      return 0;
  }
  return 1;
}

// registration.py:341-361
__device__ __forceinline__ void so3_exp_fast(double wx, double wy, double wz, double* o) {
  const double theta2 = wx * wx + wy * wy + wz * wz, theta = sqrt(theta2);
  double a, b;
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

// registration.py:364-384
__device__ __forceinline__ void renorm_rotation(const double* r, double* o) {
  const double n0 = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
  const double x0 = r[0] / n0, x1 = r[1] / n0, x2 = r[2] / n0;
  double y0 = r[3], y1 = r[4], y2 = r[5];
  const double dot = x0 * y0 + x1 * y1 + x2 * y2;
  y0 -= dot * x0, y1 -= dot * x1, y2 -= dot * x2;
  const double ny = sqrt(y0 * y0 + y1 * y1 + y2 * y2);
  y0 = y0 / ny, y1 = y1 / ny, y2 = y2 / ny;
  o[0] = x0, o[1] = x1, o[2] = x2, o[3] = y0, o[4] = y1, o[5] = y2;
  o[6] = x1 * y2 - x2 * y1, o[7] = x2 * y0 - x0 * y2, o[8] = x0 * y1 - x1 * y0;
}

// nearest rotation (geometry.py:82-89): polar factor by Newton iteration
__device__ __forceinline__ void orthonormalize3(const double* r, double* x) {
#pragma unroll
  for (int i = 0; i < 9; ++i) x[i] = r[i];
  for (int it = 0; it < 3; ++it) {
    const double c[9] = {x[4] * x[8] - x[5] * x[7], x[5] * x[6] - x[3] * x[8], x[3] * x[7] - x[4] * x[6],
                         x[2] * x[7] - x[1] * x[8], x[0] * x[8] - x[2] * x[6], x[1] * x[6] - x[0] * x[7],
                         x[1] * x[5] - x[2] * x[4], x[2] * x[3] - x[0] * x[5], x[0] * x[4] - x[1] * x[3]};
    const double det = x[0] * c[0] + x[1] * c[1] + x[2] * c[2];
#pragma unroll
    for (int i = 0; i < 9; ++i) x[i] = 0.5 * (x[i] + c[i] / det);
  }
}

__device__ __forceinline__ double shfl_d(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }

// ---------------------------------------------------------------------------
// The batched refinement runs iteration-synchronously over all candidates:
//
//   gicp_init_kernel   once   per-candidate state, source covariances
//   gicp_nn_kernel     / it   exact nearest neighbours of every source point (no shared
//                             memory, 64 registers: the whole 228 KB is L1 for the target
//                             data and twice as many warps hide the dependent loads)
//   gicp_step_kernel   / it   linearise with those neighbours, ordered sums, solve, step
//                             halving, state update (128 registers, staging shared memory)
//   gicp_finish_kernel once   result transform, residual, refine-apply + 3-DoF re-lift
//
// One warp per candidate in every kernel; a candidate that has finished (converged,
// failed, stagnated) makes its warp exit immediately.  The arithmetic and its order are
// exactly those of the reference loop (registration.py:410-476) -- only the place
// where the loop counter lives changed.

// per-candidate integer state (RefineArgs::st_i, 8 ints each)
enum { ST_FAIL = 0, ST_DONE = 1, ST_ITERS = 2, ST_CONV = 3, ST_NTRACE = 4, ST_NCORR = 5, ST_NCOMPACT = 6, ST_LASTTR = 7 };
#define ST_POSE_LD 20  // per-candidate double state: R (9), t (3), xi (6), f0, pad
#ifndef PX_HALVE_MINB
#define PX_HALVE_MINB 6
#endif

struct CandView {
  int n, nt, ti;
  long long off, toff;
};
__device__ __forceinline__ CandView cand_view(const RefineArgs& a, int c) {
  CandView v;
  v.n = a.src.count[c];
  v.off = a.src.offset[c];
  v.ti = a.target_idx[c];
  v.toff = a.tgt.offset[v.ti];
  v.nt = (int)(a.tgt.offset[v.ti + 1] - v.toff);
  return v;
}

// the covariance is bit-symmetric (registration.py:211-216 writes v0 v0^T entry by entry with commuting products)
__device__ __forceinline__ void store_src_soa(double* soa, long long plane, int i, const double* src, const double* cv) {
  soa[i] = src[3 * i], soa[plane + i] = src[3 * i + 1], soa[2 * plane + i] = src[3 * i + 2];
  soa[3 * plane + i] = cv[9], soa[4 * plane + i] = cv[10], soa[5 * plane + i] = cv[11];
}

// `split` (1, 2 or 4) warps of a CTA share a candidate: small batches do not fill the GPU with one warp each.
#ifndef PX_INIT_U16_MAX
#define PX_INIT_U16_MAX 0x10000  // clouds up to this many points keep their neighbour indices in 16 bits (0: never, test builds)
#endif
#ifndef PX_INIT_WARPS
#define PX_INIT_WARPS 4  // warps per CTA of gicp_init_kernel (the warps that share a small batch's candidate sit in one CTA)
#endif
#ifndef PX_INIT_MINB
#define PX_INIT_MINB 7  // resident CTAs per SM asked of ptxas: 72 registers; shared memory allows 7 at k = 20 (swept 4..8: 16.3 / 14.3 / 13.2 / 12.7 / 13.5 ms)
#endif
__global__ void __launch_bounds__(32 * PX_INIT_WARPS, PX_INIT_MINB) gicp_init_kernel(RefineArgs a, int split) {
  extern __shared__ __align__(16) double sm[];  // per warp: [k][32] doubles + [k][32] 16-bit indices of neighbour lists
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = (blockIdx.x * PX_INIT_WARPS + wid) / split, slice = wid % split;
  const bool live = c < a.src.n;
  const GicpCfgDev cfg = a.cfg;
  CandView v{};
  bool too_few = true;
  if (live) {
    v = cand_view(a, c);
    too_few = v.n <= cfg.k_cov || v.nt <= cfg.k_cov;  // registration.py:504-510
    if (slice == 0) {
      int* st = a.st_i + 8 * (size_t)c;
      double* pose = a.st_pose + ST_POSE_LD * (size_t)c;
      if (lane < 12) {
        double val = (lane == 0 || lane == 4 || lane == 8) ? 1.0 : 0.0;  // [R | t] as 9 + 3
        if (a.init_T) {
          const double* T0 = a.init_T + 12 * (size_t)c;
          val = lane < 9 ? T0[4 * (lane / 3) + lane % 3] : T0[4 * (lane - 9) + 3];
        }
        pose[lane] = val;
      }
      if (lane < 8) st[lane] = lane == ST_FAIL ? (too_few ? F_TOO_FEW : F_OK) : (lane == ST_DONE ? (too_few || cfg.max_iter < 1) : 0);
    }
  }
  const bool work = live && !too_few;
  const double* src = a.src.points + 3 * v.off;
  double* soa = a.src_soa + v.off;  // planes x, y, z, v0x, v0y, v0z
  const long long plane = a.plane;
  if (a.src.slot_map) {
    int4 bb = make_int4(0, 0, 0, 0);
    double* G = a.w_buf + v.off;  // dense copy of the cloud over its screen box, in the (still unused) match scratch
    if (work) {
      bb = a.src.bbox[c];
      const int32_t* map = a.src.slot_map + v.off;
      for (int cell = slice * 32 + lane; cell < bb.z * bb.w; cell += 32 * split) {
        const int j = map[cell];
        G[cell] = j >= 0 ? src[3 * j] : CUDART_NAN, G[plane + cell] = j >= 0 ? src[3 * j + 1] : CUDART_NAN;
        G[2 * plane + cell] = j >= 0 ? src[3 * j + 2] : CUDART_NAN;
      }
    }
    __syncthreads();  // the warps of a candidate read each other's part of the grid (uniform: no early exits above)
    if (!work) return;
    const int32_t* map = a.src.slot_map + v.off;
    const int32_t* spx = a.src.src_px + 2 * v.off;
    const int stp = a.cam.stride;
#ifdef PX_GLOBAL_RAYK
    const double ray_k = a.cam.ray_k;
#else
    const double ray_k = window_ray_k(a.cam, bb.x, bb.y, bb.z, bb.w);  // the candidate's screen box
#endif
    double* nd = sm + (size_t)wid * (cfg.k_cov * 40) + lane;
    unsigned short* ni = reinterpret_cast<unsigned short*>(sm + (size_t)wid * (cfg.k_cov * 40) + cfg.k_cov * 32) + lane;
#ifndef PX_INIT_NO_CLASSES
    // Visiting order: a warp waits for its slowest lane, and a point on the silhouette -- half or three quarters of its
    // rings empty -- searches two to three times as many cells as an interior one.  The points are therefore visited
    // class by class (5x5 neighbourhood inside the silhouette / at least 15 of its cells / fewer), so that the 32
    // searches of a step are of one kind.  Results are written by point index: any order gives the same planes.
    // (With several warps per candidate every warp builds the same spans and the same permutation -- identical
    // stores, no cross-warp dependence.)  The permutation lives in the nn[] plane, unused before the first NN launch.
    int32_t* perm = a.nn + v.off;
    {
      int2* span = reinterpret_cast<int2*>(G + 3 * plane);  // fourth scratch plane: first / last non-empty cell per grid row
      for (int y = lane; y < bb.w; y += 32) {
        int lo = bb.z, hi = -1;
        for (int x = 0; x < bb.z; ++x)
          if (map[y * bb.z + x] >= 0) lo = min(lo, x), hi = x;
        span[y] = make_int2(lo, hi);
      }
      __syncwarp();
      auto classify = [&](int i) {
        const int cx = spx[2 * i] / stp - bb.x, cy = spx[2 * i + 1] / stp - bb.y;
        int covered = 0;
#pragma unroll
        for (int dy = -2; dy <= 2; ++dy) {
          const int y = cy + dy;
          if (y < 0 || y >= bb.w) continue;
          const int2 sp = span[y];
          covered += max(0, min(cx + 2, sp.y) - max(cx - 2, sp.x) + 1);
        }
        return covered >= 24 ? 0 : (covered >= 15 ? 1 : 2);
      };
      int n0 = 0, n1 = 0;
      for (int base = 0; base < v.n; base += 32) {
        const int i = base + lane;
        const int cls = i < v.n ? classify(i) : 3;
        n0 += __popc(__ballot_sync(0xffffffffu, cls == 0)), n1 += __popc(__ballot_sync(0xffffffffu, cls == 1));
      }
      int o0 = 0, o1 = n0, o2 = n0 + n1;
      for (int base = 0; base < v.n; base += 32) {
        const int i = base + lane;
        const int cls = i < v.n ? classify(i) : 3;
        const unsigned m0 = __ballot_sync(0xffffffffu, cls == 0), m1 = __ballot_sync(0xffffffffu, cls == 1),
                       m2 = __ballot_sync(0xffffffffu, cls == 2), below = (1u << lane) - 1u;
        if (cls == 0) perm[o0 + __popc(m0 & below)] = i;
        if (cls == 1) perm[o1 + __popc(m1 & below)] = i;
        if (cls == 2) perm[o2 + __popc(m2 & below)] = i;
        o0 += __popc(m0), o1 += __popc(m1), o2 += __popc(m2);
      }
      __syncwarp();
    }
    for (int s_ = slice * 32 + lane; s_ < v.n; s_ += 32 * split) {
      const int i = perm[s_];
#else
    for (int i = slice * 32 + lane; i < v.n; i += 32 * split) {
#endif
      double cv[12];
      if (v.n <= PX_INIT_U16_MAX) {  // neighbour indices fit 16 bits: 80 instead of 96 bytes of list per neighbour slot and lane
        knn_ring_dense<32, unsigned short>(G, plane, map, bb.z, bb.w, src[3 * i], src[3 * i + 1], src[3 * i + 2],
                                           spx[2 * i] / stp - bb.x, spx[2 * i + 1] / stp - bb.y, cfg.k_cov, ray_k, nd, ni);
        cov_from_neighbours<32, unsigned short>(src, ni, cfg.k_cov, cfg.eps, cv);
      } else {  // a cloud of more than 65,536 points (most of a full-resolution frame): thread-local lists
        double nd_l[PX_KCOV_MAX];
        int ni_l[PX_KCOV_MAX];
        knn_ring_dense<1, int>(G, plane, map, bb.z, bb.w, src[3 * i], src[3 * i + 1], src[3 * i + 2], spx[2 * i] / stp - bb.x,
                               spx[2 * i + 1] / stp - bb.y, cfg.k_cov, ray_k, nd_l, ni_l);
        cov_from_neighbours<1, int>(src, ni_l, cfg.k_cov, cfg.eps, cv);
      }
      store_src_soa(soa, plane, i, src, cv);
    }
  } else {
    if (!work) return;
    for (int i = slice * 32 + lane; i < v.n; i += 32 * split) {
      double cv[12];
      cov_point(src, v.n, i, cfg.k_cov, cfg.eps, cv);
      store_src_soa(soa, plane, i, src, cv);
    }
  }
}

#ifndef PX_NN_MINB
#define PX_NN_MINB 8
#endif
// `split` warps share a candidate (its queries dealt round-robin in chunks of 32): small batches do not fill
// the GPU with one warp per candidate, and the queries are independent.
#ifndef PX_NN_WARPS
#define PX_NN_WARPS 4  // warps (candidates) per CTA; a CTA's slot is held until its slowest warp is done
#endif
__global__ void __launch_bounds__(32 * PX_NN_WARPS, PX_NN_MINB * 4 / PX_NN_WARPS) gicp_nn_kernel(RefineArgs a, int it, int split) {
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = blockIdx.x * PX_NN_WARPS + wid;
  const int c = gw / split, slice = gw - c * split;
  if (c >= a.src.n) return;
  if (a.st_i[8 * (size_t)c + ST_DONE]) return;
  const CandView v = cand_view(a, c);
  const double* soa = a.src_soa + v.off;
  const long long plane = a.plane;
  int32_t* nn = a.nn + v.off;
  double r[9], t[3];
#pragma unroll
  for (int q = 0; q < 9; ++q) r[q] = a.st_pose[ST_POSE_LD * (size_t)c + q];
#pragma unroll
  for (int q = 0; q < 3; ++q) t[q] = a.st_pose[ST_POSE_LD * (size_t)c + 9 + q];
  const double gate2 = a.cfg.gate2;
  for (int i = slice * 32 + lane; i < v.n; i += 32 * split) {
    // streamed once per iteration: keep them from displacing the boxes and leaf records in the L1
    const double ax = PX_LDCS(soa + i), ay = PX_LDCS(soa + plane + i), az = PX_LDCS(soa + 2 * plane + i);
    const int seed = it == 1 ? -1 : PX_LDCS(nn + i);
    const double px = r[0] * ax + r[1] * ay + r[2] * az + t[0];
    const double py = r[3] * ax + r[4] * ay + r[5] * az + t[1];
    const double pz = r[6] * ax + r[7] * ay + r[8] * az + t[2];
    double best;
    int bj;
    // seed: this point's gated neighbour of the previous iteration (read before it is overwritten)
    nn_target(a.tgt, v.ti, v.toff, v.nt, px, py, pz, seed, gate2, best, bj);
    PX_STCS(nn + i, (bj >= 0 && !(best > gate2)) ? bj : -1);  // registration.py:261
#ifdef PX_NN_STATS
    {
      float* pq = g_nn_prevq + 3 * (v.off + i);
      if (it > 1) {
        const double mx = px - pq[0], my = py - pq[1], mz = pz - pq[2];
        const double m = sqrt(mx * mx + my * my + mz * mz) * 1e3;  // mm
        const int b_ = m < 0.03 ? 0 : m < 0.1 ? 1 : m < 0.3 ? 2 : m < 1.0 ? 3 : m < 3.0 ? 4 : m < 10.0 ? 5 : 6;
        atomicAdd(&g_nn_mhist[b_], 1ull);
      }
      pq[0] = (float)px, pq[1] = (float)py, pq[2] = (float)pz;
    }
#endif
  }
}

// Linearisation (registration.py:233-338) for iteration `it`: per-point terms lane-parallel, staged
// through shared memory and summed in source-index order by 43 lanes; then the 6x6 solve.
// Matched points are compacted (in index order) into 15 planes {W (9), source point (3), target
// point (3)} for the step-halving kernel, whose objective visits exactly the matched points in
// ascending index order (registration.py:387-407).
__global__ void __launch_bounds__(PX_GICP_WARPS * 32, PX_GICP_MINB) gicp_lin_kernel(RefineArgs a, int it) {
  extern __shared__ __align__(16) double sm[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * PX_GICP_WARPS + wid;
  if (c >= a.src.n) return;
  int* st = a.st_i + 8 * (size_t)c;
  if (st[ST_DONE]) return;
  double* stage = sm + (size_t)wid * WARP_SM_DOUBLES;  // [43][STAGE_LD]
  double* hg = stage + 43 * STAGE_LD;                  // [43]: H (36), g (6), f0
  const CandView v = cand_view(a, c);
  const int n = v.n;
  const double* soa = a.src_soa + v.off;  // planes x, y, z, v0x, v0y, v0z
  const long long plane = a.plane;
  double* wb = a.w_buf + v.off;           // 10 compact planes
  const int32_t* nn = a.nn + v.off;
  const double* tsoa = a.tgt.soa + v.toff;  // same six planes of the target
  const double f_src = 1.0 - a.cfg.eps, f_tgt = a.tgt.f;
  const long long tplane = a.tgt.plane;
  double* pose = a.st_pose + ST_POSE_LD * (size_t)c;
  double r[9], t[3];
#pragma unroll
  for (int q = 0; q < 9; ++q) r[q] = pose[q];
#pragma unroll
  for (int q = 0; q < 3; ++q) t[q] = pose[9 + q];

  double acc0 = 0.0, acc1 = 0.0;
  // the running match count lives in shared memory: as a register it gets spilled, and the local-memory reload
  // queues behind the compaction stores (20 % of this kernel's stall samples)
  volatile int* n_corr_sm = reinterpret_cast<volatile int*>(hg + 43);
  if (lane == 0) *n_corr_sm = 0;
  __syncwarp();
  // software pipeline: a chunk's operands (source point + covariance, gathered target point +
  // covariance) are requested before the ordered sums of the previous chunk, its neighbour
  // indices one chunk earlier still
  int bj_cur = lane < n ? nn[lane] : -1;
  int bj_next = lane + 32 < n ? nn[lane + 32] : -1;
  double in[12];  // ax ay az | source v0 | tx ty tz | target v0
#pragma unroll
  for (int q = 0; q < 12; ++q) in[q] = 0.0;
  if (bj_cur >= 0) {
#pragma unroll
    for (int q = 0; q < 6; ++q) in[q] = PX_LDCS(soa + q * plane + lane);
#pragma unroll
    for (int q = 0; q < 6; ++q) in[6 + q] = __ldg(tsoa + q * tplane + bj_cur);
  }
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    const int bj = bj_cur;
    bool on = false;
    // absent points keep all-zero inputs: every staged term is then an exact (+-)0, which leaves the
    // never-negative-zero accumulators unchanged -- and all lanes run one uniform staging pass
    double w[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    double px = 0, py = 0, pz = 0, dx = 0, dy = 0, dz = 0;
    const double ax = in[0], ay = in[1], az = in[2], tx = in[6], ty = in[7], tz = in[8];
    if (bj >= 0) {
      double cai[9], cbj[9];
      cov_from_normal(in[3], in[4], in[5], f_src, cai);
      cov_from_normal(in[9], in[10], in[11], f_tgt, cbj);
      double rc[9], m[9];
#pragma unroll
      for (int u = 0; u < 3; ++u)
#pragma unroll
        for (int w_ = 0; w_ < 3; ++w_) {
          double s_ = 0.0;
#pragma unroll
          for (int q = 0; q < 3; ++q) s_ += r[3 * u + q] * cai[3 * q + w_];
          rc[3 * u + w_] = s_;
        }
#pragma unroll
      for (int u = 0; u < 3; ++u)
#pragma unroll
        for (int w_ = 0; w_ < 3; ++w_) {
          double s_ = 0.0;
#pragma unroll
          for (int q = 0; q < 3; ++q) s_ += rc[3 * u + q] * r[3 * w_ + q];
          m[3 * u + w_] = cbj[3 * u + w_] + s_;
        }
      const double det = (m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
                          m[2] * (m[3] * m[7] - m[4] * m[6]));
      if (!(det <= 0.0) && isfinite(det)) {
        on = true;
        const double inv_det = 1.0 / det;
        w[0] = (m[4] * m[8] - m[5] * m[7]) * inv_det;
        w[1] = (m[2] * m[7] - m[1] * m[8]) * inv_det;
        w[2] = (m[1] * m[5] - m[2] * m[4]) * inv_det;
        w[3] = (m[5] * m[6] - m[3] * m[8]) * inv_det;
        w[4] = (m[0] * m[8] - m[2] * m[6]) * inv_det;
        w[5] = (m[2] * m[3] - m[0] * m[5]) * inv_det;
        w[6] = (m[3] * m[7] - m[4] * m[6]) * inv_det;
        w[7] = (m[1] * m[6] - m[0] * m[7]) * inv_det;
        w[8] = (m[0] * m[4] - m[1] * m[3]) * inv_det;
        px = r[0] * ax + r[1] * ay + r[2] * az + t[0];
        py = r[3] * ax + r[4] * ay + r[5] * az + t[1];
        pz = r[6] * ax + r[7] * ay + r[8] * az + t[2];
        dx = tx - px, dy = ty - py, dz = tz - pz;
      }
    }
    {
      // J = [ [p]x | -I ] (registration.py:296-309).  The products with J's exact
      // zeros and -1s are dropped / turned into negations below: x*0 = +-0 and
      // a + (+-0) = a never change a non-zero value, (-1)*x = -x and a + (-b) = a - b
      // are exact, and the sign of an all-zero term cannot survive the +0-initialised
      // accumulators -- so every staged term has the reference's bits.
      const double wd0 = w[0] * dx + w[1] * dy + w[2] * dz;
      const double wd1 = w[3] * dx + w[4] * dy + w[5] * dz;
      const double wd2 = w[6] * dx + w[7] * dy + w[8] * dz;
      stage[42 * STAGE_LD + lane] = dx * wd0 + dy * wd1 + dz * wd2;
      // g[u] -= J[0][u]*wd0 + J[1][u]*wd1 + J[2][u]*wd2  (staged negated)
      stage[36 * STAGE_LD + lane] = -(pz * wd1 - py * wd2);
      stage[37 * STAGE_LD + lane] = -(px * wd2 - pz * wd0);
      stage[38 * STAGE_LD + lane] = -(py * wd0 - px * wd1);
      stage[39 * STAGE_LD + lane] = wd0;
      stage[40 * STAGE_LD + lane] = wd1;
      stage[41 * STAGE_LD + lane] = wd2;
      // wj[q][u] = w[q][0]*J[0][u] + w[q][1]*J[1][u] + w[q][2]*J[2][u]
      double wj[3][6];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        wj[q][0] = w[3 * q + 1] * pz - w[3 * q + 2] * py;
        wj[q][1] = w[3 * q + 2] * px - w[3 * q] * pz;
        wj[q][2] = w[3 * q] * py - w[3 * q + 1] * px;
        wj[q][3] = -w[3 * q], wj[q][4] = -w[3 * q + 1], wj[q][5] = -w[3 * q + 2];
      }
      // h[u][v] += J[0][u]*wj[0][v] + J[1][u]*wj[1][v] + J[2][u]*wj[2][v]
#pragma unroll
      for (int u = 0; u < 6; ++u) {
        stage[(0 + u) * STAGE_LD + lane] = pz * wj[1][u] - py * wj[2][u];
        stage[(6 + u) * STAGE_LD + lane] = px * wj[2][u] - pz * wj[0][u];
        stage[(12 + u) * STAGE_LD + lane] = py * wj[0][u] - px * wj[1][u];
        stage[(18 + u) * STAGE_LD + lane] = -wj[0][u];
        stage[(24 + u) * STAGE_LD + lane] = -wj[1][u];
        stage[(30 + u) * STAGE_LD + lane] = -wj[2][u];
      }
    }
    const unsigned onm = __ballot_sync(0xffffffffu, on);
    if (on) {  // ordered compaction for the halving kernel
      double* o = wb + *n_corr_sm + __popc(onm & ((1u << lane) - 1u));
#pragma unroll
      for (int q = 0; q < 9; ++q) PX_STCS(o + q * plane, w[q]);  // streamed: read once, by the halving kernel
      // tenth plane: (source index, target index) -- the halving kernel fetches the two points itself
      PX_STCS(reinterpret_cast<long long*>(o + 9 * plane), (long long)(unsigned)i | ((long long)bj << 32));
    }
    __syncwarp();
    if (lane == 0) *n_corr_sm += __popc(onm);
    __syncwarp();  // stage writes visible to the summing lanes
    // next chunk's operands: requested last, so that nothing between here and the end of the ordered
    // sums has to wait on a long-latency scoreboard they share
    bj_cur = bj_next;
    bj_next = i + 64 < n ? nn[i + 64] : -1;
    if (bj_cur >= 0) {
#pragma unroll
      for (int q = 0; q < 6; ++q) in[q] = PX_LDCS(soa + q * plane + i + 32);  // streamed once per iteration
#pragma unroll
      for (int q = 0; q < 6; ++q) in[6 + q] = __ldg(tsoa + q * tplane + bj_cur);
    }
    {
      const double* row0 = stage + lane * STAGE_LD;
      const double* row1 = stage + (lane + 32) * STAGE_LD;
      const bool second = lane < 11;  // quantities 32..42
#pragma unroll 8
      for (int j = 0; j < 32; ++j) {
        acc0 += row0[j];
        if (second) acc1 += row1[j];  // predicated, not a branch
      }
    }
    __syncwarp();
  }
  // H (36), g (6), f0 go to global memory: the 6x6 solve runs in its own kernel, one THREAD per candidate
  // (as a one-lane tail of this kernel it held the warp, its 128 registers per lane and its staging memory
  // for ~1,000 serial instructions per candidate)
  double* out_hg = a.st_hg + 44 * (size_t)c;
  out_hg[lane] = acc0;
  if (lane < 11) out_hg[32 + lane] = acc1;
  if (lane == 0) {
    const int n_corr = *n_corr_sm;
    st[ST_ITERS] = it;
    st[ST_NCORR] += n_corr;
    st[ST_NCOMPACT] = n_corr;
  }
}

// registration.py:434-437 + :479-494 for iteration `it`: degenerate / singular exits, else the step xi.
__global__ void __launch_bounds__(128) gicp_solve_kernel(RefineArgs a) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= a.src.n) return;
  int* st = a.st_i + 8 * (size_t)c;
  if (st[ST_DONE]) return;
  const double* hg = a.st_hg + 44 * (size_t)c;
  double h[36], g[6], xi0[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
  for (int q = 0; q < 36; ++q) h[q] = hg[q];
#pragma unroll
  for (int q = 0; q < 6; ++q) g[q] = hg[36 + q];
  int failure = F_OK;
  if (st[ST_NCOMPACT] < 6)
    failure = F_DEGENERATE;
  else if (solve_normal_equations(h, g, xi0))
    failure = F_SINGULAR;
  double* pose = a.st_pose + ST_POSE_LD * (size_t)c;
#pragma unroll
  for (int q = 0; q < 6; ++q) pose[12 + q] = xi0[q];
  pose[18] = hg[42];
  if (failure != F_OK) st[ST_FAIL] = failure, st[ST_DONE] = 1;
}

// Step halving, state update and termination tests (registration.py:443-471) for iteration `it`.
//
// The reference tries scales 1, 1/2, ... one after the other and keeps the first with f_try <= f0.
// Here PX_HALVE_NT consecutive trials are evaluated in ONE pass over the matched points (their
// poses sit in shared memory, the point's 15 operands are loaded once, and the NT ordered sums
// run side by side in different lanes), and the first acceptable one in trial order is kept --
// the same decision from the same f values.  Measured trial histogram on C3: 54 / 11 / 23 / 11 /
// 0.3 % -- two trials per pass settle 65 % of the steps in one pass and 99.7 % in two (tuned by sweep).
// The kernel is bound by the re-reads of the 120-byte match records, so a candidate whose previous step
// needed trial >= 2 opens with four trials in its first pass (how the trials are batched does not
// change which one is accepted).
#ifndef PX_HALVE_NT
#define PX_HALVE_NT 2
#endif
#define PX_HALVE_NTMAX 4
__global__ void __launch_bounds__(128, PX_HALVE_MINB) gicp_halve_kernel(RefineArgs a, int it) {
  constexpr int NTMAX = PX_HALVE_NTMAX;
  __shared__ __align__(16) double sm_pose[4][NTMAX][12];
  __shared__ __align__(16) double sm_term[4][NTMAX][34];  // rows padded: the trials' rows start in different banks
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * 4 + wid;
  if (c >= a.src.n) return;
  int* st = a.st_i + 8 * (size_t)c;
  if (st[ST_DONE]) return;
  const GicpCfgDev cfg = a.cfg;
  const long long plane = a.plane;
  const double* wb = a.w_buf + a.src.offset[c];  // 10 compact planes: W (9), (source index, target index)
  const double* soa = a.src_soa + a.src.offset[c];
  const double* tsoa = a.tgt.soa + a.tgt.offset[a.target_idx[c]];
  const long long tplane = a.tgt.plane;
  const int nc = st[ST_NCOMPACT];
  double* pose = a.st_pose + ST_POSE_LD * (size_t)c;
  double xi[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) xi[q] = pose[12 + q];
  const double f0 = pose[18];
  int acc_s = -1, acc_tr = 0;
  double f_acc = 0.0;
  int NT = st[ST_LASTTR] >= PX_HALVE_NT ? NTMAX : PX_HALVE_NT;  // trials in the first pass (a power of two)
  for (int tr0 = 0; tr0 < 9 && acc_s < 0; tr0 += NT, NT = PX_HALVE_NT) {
    const int my = lane & (NT - 1);  // the trial of the pass whose pose this lane builds and whose sum it carries
    {
      double r[9], t[3], rs[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) r[q] = pose[q];
#pragma unroll
      for (int q = 0; q < 3; ++q) t[q] = pose[9 + q];
      const double scale = 1.0 / (double)(1 << (tr0 + my));  // exact power of two, as `scale *= 0.5` yields
      so3_exp_fast(scale * xi[0], scale * xi[1], scale * xi[2], rs);
      __syncwarp();
      if (lane < NT) {
        double* o = sm_pose[wid][lane];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
#pragma unroll
          for (int j = 0; j < 3; ++j)
            o[3 * i + j] = dot_f012(rs[3 * i], rs[3 * i + 1], rs[3 * i + 2], r[j], r[3 + j], r[6 + j]);
          o[9 + i] = dot_f102(rs[3 * i], rs[3 * i + 1], rs[3 * i + 2], t[0], t[1], t[2]) + scale * xi[3 + i];
        }
      }
      __syncwarp();
    }
    // ---- fixed-association objective (registration.py:387-407) of the NT trial poses ----
    double f = 0.0;
    double cur[15];  // W (9) | source point (3) | target point (3)
    // software pipeline: the (source, target) index pair of a chunk is fetched one chunk ahead of its operands
    long long ij_cur = lane < nc ? PX_LDCS(reinterpret_cast<const long long*>(wb + 9 * plane) + lane) : 0;
    long long ij_next = lane + 32 < nc ? PX_LDCS(reinterpret_cast<const long long*>(wb + 9 * plane) + lane + 32) : 0;
    if (lane < nc) {
      const int si = (int)(unsigned)ij_cur, tj = (int)(ij_cur >> 32);
#pragma unroll
      for (int q = 0; q < 9; ++q) cur[q] = PX_LDCS(wb + q * plane + lane);
#pragma unroll
      for (int q = 0; q < 3; ++q) cur[9 + q] = soa[q * plane + si], cur[12 + q] = __ldg(tsoa + q * tplane + tj);
    }
    for (int base = 0; base < nc; base += 32) {
      const int k = base + lane;
      const bool have = k < nc;
#pragma unroll
      for (int s_ = 0; s_ < NTMAX; ++s_) {
        if (s_ >= NT) break;
        double term = 0.0;
        if (have) {
          const double* P = sm_pose[wid][s_];
          const double px = P[0] * cur[9] + P[1] * cur[10] + P[2] * cur[11] + P[9];
          const double py = P[3] * cur[9] + P[4] * cur[10] + P[5] * cur[11] + P[10];
          const double pz = P[6] * cur[9] + P[7] * cur[10] + P[8] * cur[11] + P[11];
          const double dx = cur[12] - px, dy = cur[13] - py, dz = cur[14] - pz;
          const double wd0 = cur[0] * dx + cur[1] * dy + cur[2] * dz;
          const double wd1 = cur[3] * dx + cur[4] * dy + cur[5] * dz;
          const double wd2 = cur[6] * dx + cur[7] * dy + cur[8] * dz;
          term = dx * wd0 + dy * wd1 + dz * wd2;
        }
        sm_term[wid][s_][lane] = term;
      }
      __syncwarp();
      ij_cur = ij_next;
      ij_next = k + 64 < nc ? PX_LDCS(reinterpret_cast<const long long*>(wb + 9 * plane) + k + 64) : 0;
      if (k + 32 < nc) {  // next chunk's operands are in flight during the ordered sums
        const int si = (int)(unsigned)ij_cur, tj = (int)(ij_cur >> 32);
#pragma unroll
        for (int q = 0; q < 9; ++q) cur[q] = PX_LDCS(wb + q * plane + k + 32);
#pragma unroll
        for (int q = 0; q < 3; ++q) cur[9 + q] = soa[q * plane + si], cur[12 + q] = __ldg(tsoa + q * tplane + tj);
      }
      if (lane < NT) {  // the ordered sum of trial `lane`; only these lanes' sums are read below
        const double2* s2 = reinterpret_cast<const double2*>(sm_term[wid][lane]);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const double2 v = s2[j];
          f += v.x;
          f += v.y;
        }
      }
      __syncwarp();
    }
#pragma unroll
    for (int s_ = NTMAX - 1; s_ >= 0; --s_) {  // first acceptable trial in trial order
      const double fs = shfl_d(f, s_);
      if (s_ < NT && tr0 + s_ < 9 && isfinite(fs) && fs <= f0) acc_s = s_, acc_tr = tr0 + s_, f_acc = fs;
    }
  }
  int failure = F_OK, conv = 0;
  bool done = false;
  if (acc_s < 0) {
    failure = F_NO_DECREASE, done = true;
  } else {
    const double* P = sm_pose[wid][acc_s];
    double r_try[9], r[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) r_try[q] = P[q];
    renorm_rotation(r_try, r);
    const double scale = 1.0 / (double)(1 << acc_tr), f_try = f_acc;
    if (a.out_trace && lane == 0) {
      double* trace = a.out_trace + 2 * (size_t)cfg.max_iter * c;
      trace[2 * (it - 1)] = f0, trace[2 * (it - 1) + 1] = f_try;
    }
    const double step_t2 = scale * scale * (xi[3] * xi[3] + xi[4] * xi[4] + xi[5] * xi[5]);
    const double step_r2 = scale * scale * (xi[0] * xi[0] + xi[1] * xi[1] + xi[2] * xi[2]);
    if (step_t2 < cfg.tol_t2 && step_r2 < cfg.tol_r2)
      conv = 1, done = true;
    else if (it >= 5 && f0 > 0.0 && (f0 - f_try) <= 1e-4 * f0)
      done = true;
    if (lane < 9) pose[lane] = r[lane];
    if (lane < 3) pose[9 + lane] = P[9 + lane];
  }
  if (lane == 0) {
    if (failure != F_OK) st[ST_FAIL] = failure;
    if (failure == F_OK) st[ST_NTRACE] = it, st[ST_LASTTR] = acc_tr;  // an accepted step was recorded
    if (conv) st[ST_CONV] = 1;
    if (done || it >= cfg.max_iter) st[ST_DONE] = 1;
  }
}

// solve6 / solve_normal_equations with the six rows of the augmented system [H + diag | g] in lanes 0..5 (row i in
// lane i): pivot search, row exchange, elimination and back-substitution perform exactly the operations of the scalar
// routine (same operands, same order per element), so the result has the same bits; every lane returns x.
__device__ __forceinline__ int warp_solve6(const double* __restrict__ h, double diag_add, const double* __restrict__ g,
                                           double* __restrict__ x, int lane) {
  const int row_id = lane < 6 ? lane : 5;
  double row[7];
#pragma unroll
  for (int j = 0; j < 6; ++j) row[j] = h[6 * row_id + j] + (row_id == j ? diag_add : 0.0);
  row[6] = g[row_id];
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    const double mine = fabs(row[c]);
    int p = c;
    double best = shfl_d(mine, c);
#pragma unroll
    for (int i = c + 1; i < 6; ++i) {
      const double v = shfl_d(mine, i);
      if (v > best) best = v, p = i;
    }
    if (best == 0.0 || isnan(best)) return 1;
#pragma unroll
    for (int j = c; j < 7; ++j) {  // exchange rows c and p (columns left of c are never read again)
      const double vc = shfl_d(row[j], c), vp = shfl_d(row[j], p);
      if (p != c) {
        if (lane == c) row[j] = vp;
        else if (lane == p) row[j] = vc;
      }
    }
    const double inv = 1.0 / shfl_d(row[c], c);
    const double l = row[c] * inv;
#pragma unroll
    for (int j = c + 1; j < 7; ++j) {
      const double pv = shfl_d(row[j], c);
      if (lane > c && lane < 6) row[j] = row[j] - l * pv;
    }
  }
#pragma unroll
  for (int i = 5; i >= 0; --i) {
    double s_ = row[6];
#pragma unroll
    for (int j = i + 1; j < 6; ++j) s_ = s_ - row[j] * x[j];
    x[i] = shfl_d(s_ / row[i], i);
  }
  return 0;
}

// registration.py:479-494 (see solve_normal_equations)
__device__ __forceinline__ int warp_solve_normal_equations(const double* h, const double* g, double* xi, int lane) {
  const double pi2 = CUDART_PI * CUDART_PI;
  for (int damped = 0; damped < 2; ++damped) {
    if (warp_solve6(h, damped ? 1e-6 : 0.0, g, xi, lane)) continue;
    bool fin = true;
    for (int i = 0; i < 6; ++i) fin = fin && isfinite(xi[i]);
    if (fin && xi[0] * xi[0] + xi[1] * xi[1] + xi[2] * xi[2] < pi2 &&
        xi[3] * xi[3] + xi[4] * xi[4] + xi[5] * xi[5] < 1.0)
      return 0;
  }
  return 1;
}

// Fused iteration step: linearise (gicp_lin_kernel's body) -> 6x6 solve -> step halving (gicp_halve_kernel's body) by the
// same warp.  The 80-byte match records {W, index pair} the halving reads are the ones this warp wrote a moment ago:
// they are still in L2 (cache-global stores / loads) instead of making a round trip through DRAM between two kernels
// (round 1: 105 GB of the step's 129 GB of DRAM traffic).  Arithmetic and its order are those of the split kernels.
__global__ void __launch_bounds__(PX_GICP_WARPS * 32, PX_GICP_MINB) gicp_step_kernel(RefineArgs a, int it) {
  extern __shared__ __align__(16) double sm[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * PX_GICP_WARPS + wid;
  if (c >= a.src.n) return;
  int* st = a.st_i + 8 * (size_t)c;
  if (st[ST_DONE]) return;
  double* stage = sm + (size_t)wid * WARP_SM_DOUBLES;  // [43][STAGE_LD]
  double* hg = stage + 43 * STAGE_LD;                  // [43]: H (36), g (6), f0
  const CandView v = cand_view(a, c);
  const int n = v.n;
  const double* soa = a.src_soa + v.off;  // planes x, y, z, v0x, v0y, v0z
  const long long plane = a.plane;
  double* wb = a.w_buf + v.off;           // 10 compact planes
  const int32_t* nn = a.nn + v.off;
  const double* tsoa = a.tgt.soa + v.toff;  // same six planes of the target
  const double f_src = 1.0 - a.cfg.eps, f_tgt = a.tgt.f;
  const long long tplane = a.tgt.plane;
  double* pose = a.st_pose + ST_POSE_LD * (size_t)c;
  double r[9], t[3];
#pragma unroll
  for (int q = 0; q < 9; ++q) r[q] = pose[q];
#pragma unroll
  for (int q = 0; q < 3; ++q) t[q] = pose[9 + q];

  double acc0 = 0.0, acc1 = 0.0;
  // the running match count lives in shared memory: as a register it gets spilled, and the local-memory reload
  // queues behind the compaction stores (20 % of this kernel's stall samples)
  volatile int* n_corr_sm = reinterpret_cast<volatile int*>(hg + 43);
  if (lane == 0) *n_corr_sm = 0;
  __syncwarp();
  // software pipeline: a chunk's operands (source point + covariance, gathered target point +
  // covariance) are requested before the ordered sums of the previous chunk, its neighbour
  // indices one chunk earlier still
  int bj_cur = lane < n ? nn[lane] : -1;
  int bj_next = lane + 32 < n ? nn[lane + 32] : -1;
  double in[12];  // ax ay az | source v0 | tx ty tz | target v0
#pragma unroll
  for (int q = 0; q < 12; ++q) in[q] = 0.0;
  if (bj_cur >= 0) {
#pragma unroll
    for (int q = 0; q < 6; ++q) in[q] = PX_LDCS(soa + q * plane + lane);
#pragma unroll
    for (int q = 0; q < 6; ++q) in[6 + q] = __ldg(tsoa + q * tplane + bj_cur);
  }
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    const int bj = bj_cur;
    bool on = false;
    // absent points keep all-zero inputs: every staged term is then an exact (+-)0, which leaves the
    // never-negative-zero accumulators unchanged -- and all lanes run one uniform staging pass
    double w[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    double px = 0, py = 0, pz = 0, dx = 0, dy = 0, dz = 0;
    const double ax = in[0], ay = in[1], az = in[2], tx = in[6], ty = in[7], tz = in[8];
    if (bj >= 0) {
      double cai[9], cbj[9];
      cov_from_normal(in[3], in[4], in[5], f_src, cai);
      cov_from_normal(in[9], in[10], in[11], f_tgt, cbj);
      double rc[9], m[9];
#pragma unroll
      for (int u = 0; u < 3; ++u)
#pragma unroll
        for (int w_ = 0; w_ < 3; ++w_) {
          double s_ = 0.0;
#pragma unroll
          for (int q = 0; q < 3; ++q) s_ += r[3 * u + q] * cai[3 * q + w_];
          rc[3 * u + w_] = s_;
        }
#pragma unroll
      for (int u = 0; u < 3; ++u)
#pragma unroll
        for (int w_ = 0; w_ < 3; ++w_) {
          double s_ = 0.0;
#pragma unroll
          for (int q = 0; q < 3; ++q) s_ += rc[3 * u + q] * r[3 * w_ + q];
          m[3 * u + w_] = cbj[3 * u + w_] + s_;
        }
      const double det = (m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
                          m[2] * (m[3] * m[7] - m[4] * m[6]));
      if (!(det <= 0.0) && isfinite(det)) {
        on = true;
        const double inv_det = 1.0 / det;
        w[0] = (m[4] * m[8] - m[5] * m[7]) * inv_det;
        w[1] = (m[2] * m[7] - m[1] * m[8]) * inv_det;
        w[2] = (m[1] * m[5] - m[2] * m[4]) * inv_det;
        w[3] = (m[5] * m[6] - m[3] * m[8]) * inv_det;
        w[4] = (m[0] * m[8] - m[2] * m[6]) * inv_det;
        w[5] = (m[2] * m[3] - m[0] * m[5]) * inv_det;
        w[6] = (m[3] * m[7] - m[4] * m[6]) * inv_det;
        w[7] = (m[1] * m[6] - m[0] * m[7]) * inv_det;
        w[8] = (m[0] * m[4] - m[1] * m[3]) * inv_det;
        px = r[0] * ax + r[1] * ay + r[2] * az + t[0];
        py = r[3] * ax + r[4] * ay + r[5] * az + t[1];
        pz = r[6] * ax + r[7] * ay + r[8] * az + t[2];
        dx = tx - px, dy = ty - py, dz = tz - pz;
      }
    }
    {
      // J = [ [p]x | -I ] (registration.py:296-309).  The products with J's exact
      // zeros and -1s are dropped / turned into negations below: x*0 = +-0 and
      // a + (+-0) = a never change a non-zero value, (-1)*x = -x and a + (-b) = a - b
      // are exact, and the sign of an all-zero term cannot survive the +0-initialised
      // accumulators -- so every staged term has the reference's bits.
      const double wd0 = w[0] * dx + w[1] * dy + w[2] * dz;
      const double wd1 = w[3] * dx + w[4] * dy + w[5] * dz;
      const double wd2 = w[6] * dx + w[7] * dy + w[8] * dz;
      stage[42 * STAGE_LD + lane] = dx * wd0 + dy * wd1 + dz * wd2;
      // g[u] -= J[0][u]*wd0 + J[1][u]*wd1 + J[2][u]*wd2  (staged negated)
      stage[36 * STAGE_LD + lane] = -(pz * wd1 - py * wd2);
      stage[37 * STAGE_LD + lane] = -(px * wd2 - pz * wd0);
      stage[38 * STAGE_LD + lane] = -(py * wd0 - px * wd1);
      stage[39 * STAGE_LD + lane] = wd0;
      stage[40 * STAGE_LD + lane] = wd1;
      stage[41 * STAGE_LD + lane] = wd2;
      // wj[q][u] = w[q][0]*J[0][u] + w[q][1]*J[1][u] + w[q][2]*J[2][u]
      double wj[3][6];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        wj[q][0] = w[3 * q + 1] * pz - w[3 * q + 2] * py;
        wj[q][1] = w[3 * q + 2] * px - w[3 * q] * pz;
        wj[q][2] = w[3 * q] * py - w[3 * q + 1] * px;
        wj[q][3] = -w[3 * q], wj[q][4] = -w[3 * q + 1], wj[q][5] = -w[3 * q + 2];
      }
      // h[u][v] += J[0][u]*wj[0][v] + J[1][u]*wj[1][v] + J[2][u]*wj[2][v]
#pragma unroll
      for (int u = 0; u < 6; ++u) {
        stage[(0 + u) * STAGE_LD + lane] = pz * wj[1][u] - py * wj[2][u];
        stage[(6 + u) * STAGE_LD + lane] = px * wj[2][u] - pz * wj[0][u];
        stage[(12 + u) * STAGE_LD + lane] = py * wj[0][u] - px * wj[1][u];
        stage[(18 + u) * STAGE_LD + lane] = -wj[0][u];
        stage[(24 + u) * STAGE_LD + lane] = -wj[1][u];
        stage[(30 + u) * STAGE_LD + lane] = -wj[2][u];
      }
    }
    const unsigned onm = __ballot_sync(0xffffffffu, on);
    if (on) {  // ordered compaction for the halving kernel
      double* o = wb + *n_corr_sm + __popc(onm & ((1u << lane) - 1u));
#pragma unroll
      for (int q = 0; q < 9; ++q) __stcg(o + q * plane, w[q]);  // L2-resident: re-read below by this very warp
      // tenth plane: (source index, target index) -- the halving kernel fetches the two points itself
      __stcg(reinterpret_cast<long long*>(o + 9 * plane), (long long)(unsigned)i | ((long long)bj << 32));
    }
    __syncwarp();
    if (lane == 0) *n_corr_sm += __popc(onm);
    __syncwarp();  // stage writes visible to the summing lanes
    // next chunk's operands: requested last, so that nothing between here and the end of the ordered
    // sums has to wait on a long-latency scoreboard they share
    bj_cur = bj_next;
    bj_next = i + 64 < n ? nn[i + 64] : -1;
    if (bj_cur >= 0) {
#pragma unroll
      for (int q = 0; q < 6; ++q) in[q] = PX_LDCS(soa + q * plane + i + 32);  // streamed once per iteration
#pragma unroll
      for (int q = 0; q < 6; ++q) in[6 + q] = __ldg(tsoa + q * tplane + bj_cur);
    }
    {
      const double* row0 = stage + lane * STAGE_LD;
      const double* row1 = stage + (lane + 32) * STAGE_LD;
      const bool second = lane < 11;  // quantities 32..42
#pragma unroll 8
      for (int j = 0; j < 32; ++j) {
        acc0 += row0[j];
        if (second) acc1 += row1[j];  // predicated, not a branch
      }
    }
    __syncwarp();
  }
  // ---- the sums are complete: H (36), g (6), f0 into this warp's shared memory ----
  hg[lane] = acc0;
  if (lane < 11) hg[32 + lane] = acc1;
  __syncwarp();
  const int nc = *n_corr_sm;
  if (lane == 0) {
    st[ST_ITERS] = it;
    st[ST_NCORR] += nc;
    st[ST_NCOMPACT] = nc;
  }
  // ---- registration.py:434-437 + :479-494: degenerate / singular exits, else the step xi (rows of the augmented
  // system in lanes 0..5: the same partial-pivot LU as solve6, operation for operation) ----
  double xi[6] = {0, 0, 0, 0, 0, 0};
  int failure0 = F_OK;
  if (nc < 6)
    failure0 = F_DEGENERATE;
  else if (warp_solve_normal_equations(hg, hg + 36, xi, lane))
    failure0 = F_SINGULAR;
  if (failure0 != F_OK) {
    if (lane == 0) st[ST_FAIL] = failure0, st[ST_DONE] = 1;
    return;
  }
  const double f0 = hg[42];
  const GicpCfgDev cfg = a.cfg;
  // ---- step halving over the match records this warp has just written (L2 hits) ----
  constexpr int NTMAX = PX_HALVE_NTMAX;
  __syncwarp();  // hg has been read by every lane; the staging rows are free
  double(*sm_pose)[12] = reinterpret_cast<double(*)[12]>(stage);              // [NTMAX][12]
  double(*sm_term)[34] = reinterpret_cast<double(*)[34]>(stage + NTMAX * 12);  // [NTMAX][32 + 2]: rows in different banks
  int acc_s = -1, acc_tr = 0;
  double f_acc = 0.0;
  int NT = st[ST_LASTTR] >= PX_HALVE_NT ? NTMAX : PX_HALVE_NT;  // trials in the first pass (a power of two)
  for (int tr0 = 0; tr0 < 9 && acc_s < 0; tr0 += NT, NT = PX_HALVE_NT) {
    const int my = lane & (NT - 1);  // the trial of the pass whose pose this lane builds and whose sum it carries
    {
      double r[9], t[3], rs[9];
#pragma unroll
      for (int q = 0; q < 9; ++q) r[q] = pose[q];
#pragma unroll
      for (int q = 0; q < 3; ++q) t[q] = pose[9 + q];
      const double scale = 1.0 / (double)(1 << (tr0 + my));  // exact power of two, as `scale *= 0.5` yields
      so3_exp_fast(scale * xi[0], scale * xi[1], scale * xi[2], rs);
      __syncwarp();
      if (lane < NT) {
        double* o = sm_pose[lane];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
#pragma unroll
          for (int j = 0; j < 3; ++j)
            o[3 * i + j] = dot_f012(rs[3 * i], rs[3 * i + 1], rs[3 * i + 2], r[j], r[3 + j], r[6 + j]);
          o[9 + i] = dot_f102(rs[3 * i], rs[3 * i + 1], rs[3 * i + 2], t[0], t[1], t[2]) + scale * xi[3 + i];
        }
      }
      __syncwarp();
    }
    // ---- fixed-association objective (registration.py:387-407) of the NT trial poses ----
    double f = 0.0;
    double cur[15];  // W (9) | source point (3) | target point (3)
    // software pipeline: the (source, target) index pair of a chunk is fetched one chunk ahead of its operands
    long long ij_cur = lane < nc ? __ldcg(reinterpret_cast<const long long*>(wb + 9 * plane) + lane) : 0;
    long long ij_next = lane + 32 < nc ? __ldcg(reinterpret_cast<const long long*>(wb + 9 * plane) + lane + 32) : 0;
    if (lane < nc) {
      const int si = (int)(unsigned)ij_cur, tj = (int)(ij_cur >> 32);
#pragma unroll
      for (int q = 0; q < 9; ++q) cur[q] = __ldcg(wb + q * plane + lane);
#pragma unroll
      for (int q = 0; q < 3; ++q) cur[9 + q] = soa[q * plane + si], cur[12 + q] = __ldg(tsoa + q * tplane + tj);
    }
    for (int base = 0; base < nc; base += 32) {
      const int k = base + lane;
      const bool have = k < nc;
#pragma unroll
      for (int s_ = 0; s_ < NTMAX; ++s_) {
        if (s_ >= NT) break;
        double term = 0.0;
        if (have) {
          const double* P = sm_pose[s_];
          const double px = P[0] * cur[9] + P[1] * cur[10] + P[2] * cur[11] + P[9];
          const double py = P[3] * cur[9] + P[4] * cur[10] + P[5] * cur[11] + P[10];
          const double pz = P[6] * cur[9] + P[7] * cur[10] + P[8] * cur[11] + P[11];
          const double dx = cur[12] - px, dy = cur[13] - py, dz = cur[14] - pz;
          const double wd0 = cur[0] * dx + cur[1] * dy + cur[2] * dz;
          const double wd1 = cur[3] * dx + cur[4] * dy + cur[5] * dz;
          const double wd2 = cur[6] * dx + cur[7] * dy + cur[8] * dz;
          term = dx * wd0 + dy * wd1 + dz * wd2;
        }
        sm_term[s_][lane] = term;
      }
      __syncwarp();
      ij_cur = ij_next;
      ij_next = k + 64 < nc ? __ldcg(reinterpret_cast<const long long*>(wb + 9 * plane) + k + 64) : 0;
      if (k + 32 < nc) {  // next chunk's operands are in flight during the ordered sums
        const int si = (int)(unsigned)ij_cur, tj = (int)(ij_cur >> 32);
#pragma unroll
        for (int q = 0; q < 9; ++q) cur[q] = __ldcg(wb + q * plane + k + 32);
#pragma unroll
        for (int q = 0; q < 3; ++q) cur[9 + q] = soa[q * plane + si], cur[12 + q] = __ldg(tsoa + q * tplane + tj);
      }
      if (lane < NT) {  // the ordered sum of trial `lane`; only these lanes' sums are read below (one wavefront per load)
        const double2* s2 = reinterpret_cast<const double2*>(sm_term[lane]);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const double2 v = s2[j];
          f += v.x;
          f += v.y;
        }
      }
      __syncwarp();
    }
#pragma unroll
    for (int s_ = NTMAX - 1; s_ >= 0; --s_) {  // first acceptable trial in trial order
      const double fs = shfl_d(f, s_);
      if (s_ < NT && tr0 + s_ < 9 && isfinite(fs) && fs <= f0) acc_s = s_, acc_tr = tr0 + s_, f_acc = fs;
    }
  }
  int failure = F_OK, conv = 0;
  bool done = false;
  if (acc_s < 0) {
    failure = F_NO_DECREASE, done = true;
  } else {
    const double* P = sm_pose[acc_s];
    double r_try[9], r[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) r_try[q] = P[q];
    renorm_rotation(r_try, r);
    const double scale = 1.0 / (double)(1 << acc_tr), f_try = f_acc;
    if (a.out_trace && lane == 0) {
      double* trace = a.out_trace + 2 * (size_t)cfg.max_iter * c;
      trace[2 * (it - 1)] = f0, trace[2 * (it - 1) + 1] = f_try;
    }
    const double step_t2 = scale * scale * (xi[3] * xi[3] + xi[4] * xi[4] + xi[5] * xi[5]);
    const double step_r2 = scale * scale * (xi[0] * xi[0] + xi[1] * xi[1] + xi[2] * xi[2]);
    if (step_t2 < cfg.tol_t2 && step_r2 < cfg.tol_r2)
      conv = 1, done = true;
    else if (it >= 5 && f0 > 0.0 && (f0 - f_try) <= 1e-4 * f0)
      done = true;
    if (lane < 9) pose[lane] = r[lane];
    if (lane < 3) pose[9 + lane] = P[9 + lane];
  }
  if (lane == 0) {
    if (failure != F_OK) st[ST_FAIL] = failure;
    if (failure == F_OK) st[ST_NTRACE] = it, st[ST_LASTTR] = acc_tr;  // an accepted step was recorded
    if (conv) st[ST_CONV] = 1;
    if (done || it >= cfg.max_iter) st[ST_DONE] = 1;
  }
}

__global__ void __launch_bounds__(128) gicp_finish_kernel(RefineArgs a) {
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * 4 + wid;
  if (c >= a.src.n) return;
  const int* st = a.st_i + 8 * (size_t)c;
  const int failure = st[ST_FAIL], iters = st[ST_ITERS], conv = st[ST_CONV];
  const CandView v = cand_view(a, c);
  const double* pose = a.st_pose + ST_POSE_LD * (size_t)c;
  double r[9], t[3];
#pragma unroll
  for (int q = 0; q < 9; ++q) r[q] = pose[q];
#pragma unroll
  for (int q = 0; q < 3; ++q) t[q] = pose[9 + q];
  // ---- result transform (registration.py:473) ----
  double T[12];
  {
    double ro[9];
    orthonormalize3(r, ro);
    if (failure == F_TOO_FEW) {
#pragma unroll
      for (int i = 0; i < 9; ++i) ro[i] = r[i];  // init returned untouched
    }
    for (int i = 0; i < 3; ++i) {
      for (int j = 0; j < 3; ++j) T[4 * i + j] = ro[3 * i + j];
      T[4 * i + 3] = t[i];
    }
  }
  if (a.out_resid) {  // registration.py:59-67 (not used by the search path)
    const double* src = a.src.points + 3 * v.off;
    const double* tgt = a.tgt.points + 3 * v.toff;
    double sum = 0.0;
    int cnt = 0;
    if (failure != F_TOO_FEW) {
      for (int i = lane; i < v.n; i += 32) {
        double x, y, z;
        apply_pose(T, src[3 * i], src[3 * i + 1], src[3 * i + 2], x, y, z);
        double best = CUDART_INF;
        for (int j = 0; j < v.nt; ++j) {
          const double dx = tgt[3 * j] - x, dy = tgt[3 * j + 1] - y, dz = tgt[3 * j + 2] - z;
          const double d2 = dx * dx + dy * dy + dz * dz;
          if (d2 < best) best = d2;
        }
        if (best <= a.cfg.gate2) sum += best, ++cnt;
      }
      for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o), cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    }
    if (lane == 0) a.out_resid[c] = cnt ? sqrt(sum / (double)cnt) : CUDART_INF;
  }
  if (lane == 0) {
    for (int i = 0; i < 12; ++i) a.out_T[12 * (size_t)c + i] = T[i];
    a.out_iters[c] = iters;
    a.out_flags[c] = failure | (conv ? 0x100 : 0);
    if (a.out_ntrace) a.out_ntrace[c] = st[ST_NTRACE];
    if (a.out_ncorr_sum) a.out_ncorr_sum[c] = st[ST_NCORR];
    if (a.poses_in) {  // search.py:291-301
      const double* pin = a.poses_in + 12 * (size_t)c;
      double cam[12];
      if (failure == F_TOO_FEW && iters == 0) {
        for (int i = 0; i < 12; ++i) cam[i] = pin[i];
      } else {
        compose_pose(T, pin, 0, cam);
        if (a.mode3dof) {
          double world[12];
          compose_pose(a.c2w, cam, a.c2w_vec_order, world);
          const double yaw = atan2(world[4], world[0]);  // registration.py:556
          double y = fmod(yaw, 2.0 * CUDART_PI);         // geometry.py:98-105
          if (y < 0.0) y += 2.0 * CUDART_PI;
          if (y >= 2.0 * CUDART_PI) y -= 2.0 * CUDART_PI;
          const double cy = cos(y), sy = sin(y);
          const double lift[12] = {cy, -sy, 0.0, world[3], sy, cy, 0.0, world[7], 0.0, 0.0, 1.0, a.fixed_z};
          compose_pose(a.w2c, lift, a.w2c_vec_order, cam);
        }
      }
      for (int i = 0; i < 12; ++i) a.poses_out[12 * (size_t)c + i] = cam[i];
    }
  }
}

#ifdef PX_NN_STATS
void dump_nn_stats() {
  unsigned long long h[8];
  cudaMemcpyFromSymbol(h, g_nn_stats, sizeof h);
  if (h[0])
    fprintf(stderr, "[nn stats] queries %llu, with prev %.3f, found %.3f; per query: sb tests %.2f, blk tests %.2f, leaves %.2f (improving %.2f), leaf pts %.2f\n",
            h[0], (double)h[1] / h[0], (double)h[5] / h[0], (double)h[2] / h[0], (double)h[3] / h[0], (double)h[6] / h[0], (double)h[7] / h[0], (double)h[4] / h[0]);
  cudaMemcpyFromSymbol(h, g_nn_rhist, sizeof h);
  fprintf(stderr, "[nn R hist] <0.5 %llu <1.5 %llu <2.5 %llu <3.5 %llu <5.5 %llu <8.5 %llu >=8.5 %llu notfound %llu\n", h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
  {
    unsigned long long l[32];
    cudaMemcpyFromSymbol(l, g_nn_lhist, sizeof l);
    for (int g = 0; g < 4; ++g)
      fprintf(stderr, "[nn leaves/query seeded=%d found=%d] 0:%llu 1:%llu 2:%llu 3-4:%llu 5-8:%llu 9-16:%llu 17-32:%llu 33+:%llu\n", g >> 1, g & 1,
              l[8 * g], l[8 * g + 1], l[8 * g + 2], l[8 * g + 3], l[8 * g + 4], l[8 * g + 5], l[8 * g + 6], l[8 * g + 7]);
    memset(l, 0, sizeof l);
    cudaMemcpyToSymbol(g_nn_lhist, l, sizeof l);
  }
  cudaMemcpyFromSymbol(h, g_nn_mhist, sizeof h);
  fprintf(stderr, "[nn motion mm] <.03 %llu <.1 %llu <.3 %llu <1 %llu <3 %llu <10 %llu >=10 %llu\n", h[0], h[1], h[2], h[3], h[4], h[5], h[6]);
  memset(h, 0, sizeof h);
  cudaMemcpyToSymbol(g_nn_mhist, h, sizeof h);
  cudaMemcpyToSymbol(g_nn_stats, h, sizeof h);
  cudaMemcpyToSymbol(g_nn_rhist, h, sizeof h);
}
#endif

cudaError_t launch_linearize_once(const RefineArgs& a, cudaStream_t st) {
  if (a.src.n == 0) return cudaSuccess;
  cudaError_t e;
  const size_t smem_init = sizeof(double) * 40 * (size_t)a.cfg.k_cov * PX_INIT_WARPS;
  if ((e = cudaFuncSetAttribute(gicp_init_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_init)) != cudaSuccess) return e;
  gicp_init_kernel<<<(unsigned)((a.src.n + PX_INIT_WARPS - 1) / PX_INIT_WARPS), 32 * PX_INIT_WARPS, smem_init, st>>>(a, 1);
  const size_t smem = sizeof(double) * WARP_SM_DOUBLES * PX_GICP_WARPS;
  if ((e = cudaFuncSetAttribute(gicp_lin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess) return e;
  gicp_nn_kernel<<<(unsigned)((a.src.n + PX_NN_WARPS - 1) / PX_NN_WARPS), 32 * PX_NN_WARPS, 0, st>>>(a, 1, 1);
  gicp_lin_kernel<<<(a.src.n + PX_GICP_WARPS - 1) / PX_GICP_WARPS, PX_GICP_WARPS * 32, smem, st>>>(a, 1);
  return cudaGetLastError();
}

// Returns the number of kernels launched through *launches.
cudaError_t launch_refine(const RefineArgs& a, cudaStream_t st, int* launches, cudaEvent_t* marks) {
  int mk = 0;
#define PX_MARK() do { if (marks) cudaEventRecord(marks[mk++], st); } while (0)
  if (launches) *launches = 0;
  if (a.src.n == 0) return cudaSuccess;
  cudaError_t e;
#ifdef PX_NN_STATS
  cudaMemcpyToSymbol(g_nn_rayk, &a.cam.ray_k, sizeof(double));
  {
    static float* buf = nullptr;
    static long long cap = 0;
    if (cap < a.plane) {
      if (buf) cudaFree(buf);
      cudaMalloc(&buf, sizeof(float) * 3 * a.plane), cap = a.plane;
      cudaMemcpyToSymbol(g_nn_prevq, &buf, sizeof(buf));
    }
  }
#endif
  const int b4 = (a.src.n + 3) / 4;
  const size_t smem_init = sizeof(double) * 40 * (size_t)a.cfg.k_cov * PX_INIT_WARPS;
  if ((e = cudaFuncSetAttribute(gicp_init_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_init)) != cudaSuccess) return e;
  PX_MARK();
  // 1, 2 or 4 warps per candidate: about two waves of 148 SMs x 24 warps when the batch is small
#ifndef PX_INIT_SPLIT_N
#define PX_INIT_SPLIT_N 3552
#endif
  const int init_split = std::min(PX_INIT_WARPS, a.src.n >= 2 * PX_INIT_SPLIT_N ? 1 : (a.src.n >= PX_INIT_SPLIT_N ? 2 : 4));
  gicp_init_kernel<<<(unsigned)(((long long)a.src.n * init_split + PX_INIT_WARPS - 1) / PX_INIT_WARPS), 32 * PX_INIT_WARPS, smem_init, st>>>(a, init_split);
  const size_t smem = sizeof(double) * WARP_SM_DOUBLES * PX_GICP_WARPS;
  if ((e = cudaFuncSetAttribute(gicp_lin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess) return e;
  if ((e = cudaFuncSetAttribute(gicp_step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess) return e;
  cudaFuncSetAttribute(gicp_nn_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 0);  // all of it as L1
  const int blocks = (a.src.n + PX_GICP_WARPS - 1) / PX_GICP_WARPS;
  // enough NN warps for ~one full wave (148 SMs x 32 warps) when the batch is small
#ifndef PX_NN_FILL
#define PX_NN_FILL 4
#endif
#ifndef PX_NN_SPLIT_MAX
#define PX_NN_SPLIT_MAX 8
#endif
  const int nn_split = (int)std::min<long long>(PX_NN_SPLIT_MAX, std::max<long long>(1, (148LL * 32 * PX_NN_FILL + a.src.n - 1) / a.src.n));
  for (int it = 1; it <= a.cfg.max_iter; ++it) {
    PX_MARK();
    gicp_nn_kernel<<<(unsigned)(((long long)a.src.n * nn_split + PX_NN_WARPS - 1) / PX_NN_WARPS), 32 * PX_NN_WARPS, 0, st>>>(a, it, nn_split);
    PX_MARK();
#ifdef PX_GICP_SPLIT
    gicp_lin_kernel<<<blocks, PX_GICP_WARPS * 32, smem, st>>>(a, it);
    gicp_solve_kernel<<<(a.src.n + 127) / 128, 128, 0, st>>>(a);  // timed together with the linearisation
    PX_MARK();
    gicp_halve_kernel<<<b4, 128, 0, st>>>(a, it);
#else
    gicp_step_kernel<<<blocks, PX_GICP_WARPS * 32, smem, st>>>(a, it);  // linearise + solve + halving, one warp per candidate
    PX_MARK();
#endif
  }
  PX_MARK();
  gicp_finish_kernel<<<b4, 128, 0, st>>>(a);
  PX_MARK();
#undef PX_MARK
#ifdef PX_GICP_SPLIT
  if (launches) *launches = 2 + 4 * std::max(a.cfg.max_iter, 0);
#else
  if (launches) *launches = 2 + 2 * std::max(a.cfg.max_iter, 0);
#endif
#ifdef PX_NN_STATS
  cudaStreamSynchronize(st);
  dump_nn_stats();
#endif
  return cudaGetLastError();
}

}  // namespace px
