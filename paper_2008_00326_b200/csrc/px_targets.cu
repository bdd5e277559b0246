// px_targets.cu -- GICP target clouds built on the device.
//
// Replaces search._build_targets / _capsule_crop (reference pkg/src/rvpose/search.py:393-426,
// :205-214): a target is the sub-cloud of the observed cloud inside a capsule around a 3-DoF grid
// cell (radius 1.5 r + dt, z in [z_lo, z_hi]) or, in 6-DoF, the points labelled with the object.
// The reference evaluates one numpy mask over all observed points per target; here one CTA per
// target evaluates the same predicate with the same operation order (fp64, no contraction; the
// world-frame point is `p @ R.T + t` in the host BLAS order, px_common.cuh) and compacts the
// survivors in ascending observed index, which is the order np.nonzero returns.  The organised
// views the nearest-neighbour search needs (pixel map, two-level box hierarchy, per-block leaf
// records, fp32 error bound) are built here as well, with the rules px_targets_upload applies on
// the host -- tests compare both paths bit for bit.
#include "px_kernels.h"

namespace px {

__global__ void obs_world_kernel(const double* __restrict__ pts, long long n, TgtBuildArgs a) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x, y, z;
  apply_pose(a.c2w, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], x, y, z);
  a.world[i] = x, a.world[n + i] = y, a.world[2 * n + i] = z;
}

// membership of observed point i in target t
__device__ __forceinline__ bool tgt_member(const TgtBuildArgs& a, int t, long long i, const double* prm) {
  if (a.mode == 1) return a.obs_labels[i] == a.label_ids[t];
  // search.py:205-214: dx^2 + dy^2 + max(z_lo - z, z - z_hi, 0)^2 <= radius^2
  const double dx = a.world[i] - prm[0], dy = a.world[a.n_obs + i] - prm[1];
  const double pz = a.world[2 * a.n_obs + i];
  const double dz = fmax(fmax(prm[2] - pz, pz - prm[3]), 0.0);
  return dx * dx + dy * dy + dz * dz <= prm[4] * prm[4];
}

// Stride-grid window that contains the projection of every point a capsule can hold: the capsule
// {dx^2 + dy^2 + max(z_lo - z, z - z_hi, 0)^2 <= radius^2} lies inside the ball of radius R = radius + (z_hi - z_lo) / 2
// around its mid point; with the ball in front of the camera (z_c - R > 0) the extreme image coordinates of the ball's
// bounding cube bound the projections.  Two cells of margin on every side; the whole grid when no bound exists.
__device__ __forceinline__ void capsule_window(const TgtBuildArgs& a, const double* prm, int& gx_lo, int& gx_hi, int& gy_lo,
                                               int& gy_hi) {
  const int GW = a.cam.GW, GH = a.cam.GH;
  gx_lo = 0, gy_lo = 0, gx_hi = GW - 1, gy_hi = GH - 1;
  const double R = prm[4] + 0.5 * fabs(prm[3] - prm[2]);
  // capsule mid point in the camera frame: R_c2w^T (c - t_c2w)
  const double wx = prm[0] - a.c2w[3], wy = prm[1] - a.c2w[7], wz = 0.5 * (prm[2] + prm[3]) - a.c2w[11];
  const double xc = a.c2w[0] * wx + a.c2w[4] * wy + a.c2w[8] * wz;
  const double yc = a.c2w[1] * wx + a.c2w[5] * wy + a.c2w[9] * wz;
  const double zc = a.c2w[2] * wx + a.c2w[6] * wy + a.c2w[10] * wz;
  const double zn = zc - R * 1.001 - 1e-6, zf = zc + R * 1.001 + 1e-6;
  if (!(zn > 1e-3) || !isfinite(xc + yc + zc + R)) return;
  const double x0 = xc - R * 1.001, x1 = xc + R * 1.001, y0 = yc - R * 1.001, y1 = yc + R * 1.001;
  const double ulo = a.cam.cx + a.cam.fx * fmin(x0 / zn, x0 / zf), uhi = a.cam.cx + a.cam.fx * fmax(x1 / zn, x1 / zf);
  const double vlo = a.cam.cy + a.cam.fy * fmin(y0 / zn, y0 / zf), vhi = a.cam.cy + a.cam.fy * fmax(y1 / zn, y1 / zf);
  const double st = (double)a.cam.stride;
  // observed point of grid cell g sits at pixel g * stride + 0.5
  const double a0 = floor((ulo - 0.5) / st) - 2.0, a1 = ceil((uhi - 0.5) / st) + 2.0;
  const double b0 = floor((vlo - 0.5) / st) - 2.0, b1 = ceil((vhi - 0.5) / st) + 2.0;
  gx_lo = (int)fmin(fmax(a0, 0.0), (double)GW), gx_hi = (int)fmax(fmin(a1, (double)(GW - 1)), -1.0);
  gy_lo = (int)fmin(fmax(b0, 0.0), (double)GH), gy_hi = (int)fmax(fmin(b1, (double)(GH - 1)), -1.0);
}

// pass 1: member count and grid bounding box of every target
__global__ void __launch_bounds__(256) tgt_count_kernel(TgtBuildArgs a) {
  const int t = blockIdx.x;
  __shared__ double prm[5];
  __shared__ int red[4][8];
  if (a.mode == 0 && threadIdx.x < 5) prm[threadIdx.x] = a.params[5 * (size_t)t + threadIdx.x];
  __syncthreads();
  int cnt = 0, x0 = 1 << 30, y0 = 1 << 30, x1 = -1, y1 = -1;
  if (a.mode == 0) {
    // only the cells inside the capsule's screen window can hold members (the predicate itself is unchanged)
    int gx_lo, gx_hi, gy_lo, gy_hi;
    capsule_window(a, prm, gx_lo, gx_hi, gy_lo, gy_hi);
    const int ww = gx_hi - gx_lo + 1, wh = gy_hi - gy_lo + 1;
    const int ncell = (ww > 0 && wh > 0) ? ww * wh : 0;
    for (int q = threadIdx.x; q < ncell; q += blockDim.x) {
      const int gx = gx_lo + q % ww, gy = gy_lo + q / ww;
      const long long i = a.gidx[gy * a.GW + gx];
      if (i >= 0 && tgt_member(a, t, i, prm)) ++cnt, x0 = min(x0, gx), x1 = max(x1, gx), y0 = min(y0, gy), y1 = max(y1, gy);
    }
  } else {
    for (long long i = threadIdx.x; i < a.n_obs; i += blockDim.x)
      if (tgt_member(a, t, i, prm)) {
        const int cell = a.obs_cell[i], gx = cell % a.GW, gy = cell / a.GW;
        ++cnt, x0 = min(x0, gx), x1 = max(x1, gx), y0 = min(y0, gy), y1 = max(y1, gy);
      }
  }
  for (int o = 16; o; o >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    x0 = min(x0, __shfl_xor_sync(0xffffffffu, x0, o)), y0 = min(y0, __shfl_xor_sync(0xffffffffu, y0, o));
    x1 = max(x1, __shfl_xor_sync(0xffffffffu, x1, o)), y1 = max(y1, __shfl_xor_sync(0xffffffffu, y1, o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[0][w] = cnt, red[1][w] = x0, red[2][w] = y0, red[3][w] = x1 | (y1 << 16);
  __syncthreads();
  if (threadIdx.x == 0) {
    int xx1 = -1, yy1 = -1;
    cnt = 0, x0 = 1 << 30, y0 = 1 << 30;
    for (int q = 0; q < 8; ++q) {
      cnt += red[0][q], x0 = min(x0, red[1][q]), y0 = min(y0, red[2][q]);
      if (red[3][q] >= 0) xx1 = max(xx1, red[3][q] & 0xffff), yy1 = max(yy1, red[3][q] >> 16);
    }
    TgtOrg o{};
    if (cnt > 0) o.gx0 = x0, o.gy0 = y0, o.w = xx1 - x0 + 1, o.h = yy1 - y0 + 1;
    else o.gx0 = o.gy0 = 0, o.w = 1, o.h = 1;
    o.bw = (o.w + PX_BLK - 1) / PX_BLK, o.bh = (o.h + PX_BLK - 1) / PX_BLK;
    o.sw = (o.bw + PX_BLK - 1) / PX_BLK, o.sh = (o.bh + PX_BLK - 1) / PX_BLK;
    a.org[t] = o;
    a.cnt[t] = cnt;
    a.cells[t] = (long long)o.w * o.h;
    const long long ns = (long long)o.sw * o.sh;
    a.nodes[t] = 17 * ns + (ns & 1);  // px_kernels.h: 16 block slots + 1 node per super-block, even count
  }
}

__global__ void tgt_offsets_kernel(TgtBuildArgs a) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.n_targets) return;
  a.org[t].map_off = a.cells_off[t];
  a.org[t].box_off = a.nodes_off[t];
}

// coordinates in the frame of the fp32 pruning structures (TargetsDev::rot)
__device__ __forceinline__ void to_frame(const double* __restrict__ F, double x, double y, double z, double* o) {
  o[0] = F[0] * x + F[1] * y + F[2] * z, o[1] = F[3] * x + F[4] * y + F[5] * z, o[2] = F[6] * x + F[7] * y + F[8] * z;
}

// pass 2: ordered compaction -> obs index, points, map cell of every member; pixel map; error bound
__global__ void __launch_bounds__(256) tgt_fill_kernel(TgtBuildArgs a) {
  const int t = blockIdx.x;
  __shared__ double prm[5];
  __shared__ int wcnt[8];
  __shared__ double wmax[8];
  if (a.mode == 0 && threadIdx.x < 5) prm[threadIdx.x] = a.params[5 * (size_t)t + threadIdx.x];
  __syncthreads();
  const TgtOrg o = a.org[t];
  const long long off = a.offset[t];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int run = 0;
  double m = 0.0;
  // only the cells of the target's grid bounding box (pass 1) can hold members; row-major cell order is
  // ascending observed index, the order np.nonzero returns
  const int ncell = a.cnt[t] > 0 ? o.w * o.h : 0;
  for (int base = 0; base < ncell; base += blockDim.x) {
    const int lc = base + (int)threadIdx.x;
    long long i = -1;
    if (lc < ncell) i = a.gidx[(lc / o.w + o.gy0) * a.GW + lc % o.w + o.gx0];
    const bool in = i >= 0 && tgt_member(a, t, i, prm);
    const unsigned bal = __ballot_sync(0xffffffffu, in);
    if (lane == 0) wcnt[w] = __popc(bal);
    __syncthreads();
    int before = 0, all = 0;
    for (int q = 0; q < 8; ++q) {
      before += q < w ? wcnt[q] : 0;
      all += wcnt[q];
    }
    if (in) {
      const int pos = run + before + __popc(bal & ((1u << lane) - 1u));
      const double x = a.obs_pts[3 * i], y = a.obs_pts[3 * i + 1], z = a.obs_pts[3 * i + 2];
      a.tgt_obs[off + pos] = (int32_t)i;
      a.tgt_pts[3 * (off + pos)] = x, a.tgt_pts[3 * (off + pos) + 1] = y, a.tgt_pts[3 * (off + pos) + 2] = z;
      a.tpix[off + pos] = lc;
      a.tmap[o.map_off + lc] = pos;
      double f[3];
      to_frame(a.frame, x, y, z, f);
      m = fmax(m, fmax(fabs(f[0]), fmax(fabs(f[1]), fabs(f[2]))));
    }
    run += all;
    __syncthreads();
  }
  for (int q = 16; q; q >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, q));
  if (lane == 0) wmax[w] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < 8; ++q) m = fmax(m, wmax[q]);
    // px_targets_upload: bound on the fp32 pruning errors; a query that can still match lies within `gate` of a
    // target point, so its coordinates are bounded by m + gate
    a.org[t].err = ldexp(1.5 * (2.0 * m + a.gate + 1.0), -24);
  }
}

// fp32 pruning copy of a box: lo rounded down, hi rounded up (the fp32 box contains the exact one); an empty node gets
// an inverted far-away box whose distance overflows to +inf and is always pruned
__device__ __forceinline__ void box32(const double* lo, const double* hi, float* lo3, float* hi3, int stride) {
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    float lf = PX_FAR32, hf = -PX_FAR32;
    if (lo[d] <= hi[d]) lf = __double2float_rd(lo[d]), hf = __double2float_ru(hi[d]);
    lo3[d * stride] = lf, hi3[d * stride] = hf;
  }
}

// pass 3: per target, boxes of every block / super-block and the fixed-size leaf record of every block slot
__global__ void __launch_bounds__(256) tgt_tree_kernel(TgtBuildArgs a) {
  const int t = blockIdx.x;
  const TgtOrg o = a.org[t];
  const long long off = a.offset[t];
  const int32_t* map = a.tmap + o.map_off;
  const double* P = a.tgt_pts + 3 * off;
  const int ns = o.sw * o.sh;
  float* bb = a.boxes32 + 6 * o.box_off;  // per super-block 6 planes x 16 block slots, then the super-block nodes
  float* leaves = reinterpret_cast<float*>(a.leaf32) + 48 * o.box_off;  // per block slot: x[16], y[16], z[16] by map cell
  // a thread per block slot / super-block scans the node's map cells
  for (int q = threadIdx.x; q < 17 * ns; q += blockDim.x) {
    const bool sup = q >= 16 * ns;
    const int s_ = sup ? q - 16 * ns : q >> 4, slot = q & 15;
    const int span = sup ? PX_BLK * PX_BLK : PX_BLK;
    const int bx = sup ? s_ % o.sw : (s_ % o.sw) * PX_BLK + (slot & 3), by = sup ? s_ / o.sw : (s_ / o.sw) * PX_BLK + (slot >> 2);
    const int cx0 = bx * span, cy0 = by * span;
    float* rec = leaves + 48 * (size_t)q;  // block slots only
    if (!sup)
      for (int c = 0; c < 48; ++c) rec[c] = PX_FAR32;
    double lo[3] = {CUDART_INF, CUDART_INF, CUDART_INF}, hi[3] = {-CUDART_INF, -CUDART_INF, -CUDART_INF};
    for (int y = cy0; y < min(cy0 + span, o.h); ++y)
      for (int x = cx0; x < min(cx0 + span, o.w); ++x) {
        const int j = map[y * o.w + x];
        if (j < 0) continue;
        double f[3];
        to_frame(a.frame, P[3 * j], P[3 * j + 1], P[3 * j + 2], f);
#pragma unroll
        for (int d = 0; d < 3; ++d) lo[d] = fmin(lo[d], f[d]), hi[d] = fmax(hi[d], f[d]);
        if (!sup) {
          const int c = (y - cy0) * PX_BLK + (x - cx0);
          rec[c] = (float)f[0], rec[16 + c] = (float)f[1], rec[32 + c] = (float)f[2];
        }
      }
    if (sup) {
      float* o6 = bb + 96 * (size_t)ns + 6 * (size_t)s_;
      box32(lo, hi, o6, o6 + 3, 1);
    } else {
      float* blk = bb + 96 * (size_t)s_;
      box32(lo, hi, blk + slot, blk + 48 + slot, 16);
    }
  }
}

cudaError_t launch_tgt_world(const TgtBuildArgs& a, cudaStream_t st) {
  if (a.n_obs > 0 && a.mode == 0)
    obs_world_kernel<<<(unsigned)((a.n_obs + 255) / 256), 256, 0, st>>>(a.obs_pts, a.n_obs, a);
  return cudaGetLastError();
}
cudaError_t launch_tgt_count(const TgtBuildArgs& a, cudaStream_t st) {
  if (a.n_targets > 0) tgt_count_kernel<<<a.n_targets, 256, 0, st>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_tgt_fill(const TgtBuildArgs& a, cudaStream_t st) {
  if (a.n_targets > 0) {
    tgt_offsets_kernel<<<(a.n_targets + 255) / 256, 256, 0, st>>>(a);
    tgt_fill_kernel<<<a.n_targets, 256, 0, st>>>(a);
    tgt_tree_kernel<<<a.n_targets, 256, 0, st>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace px
