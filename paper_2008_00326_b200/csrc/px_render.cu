// px_render.cu -- batched per-candidate render -> occluder mark -> stride cloud -> Lab.
//
// Replaces raster._render_one / _raster_kernel (reference pkg/src/rvpose/
// raster.py:53-134, 239-280) for a whole batch of candidate poses.  One CTA per
// candidate.  Only stride-grid pixels are ever shaded: the batch path reads
// nothing else (raster.py:271-278) and pixels are independent of each other.
//
// Bit-exactness: the reference z-test is `depth < zbuf` in float64 with
// triangles visited in index order, i.e. the owner of a pixel is the triangle
// with the lexicographically smallest (depth, triangle index).  Two equivalent
// evaluations are used:
//   * few triangles (T <= PX_TRI_SMEM): thread per pixel, triangles looped in
//     index order with a strict `<` -- literally the reference recurrence;
//   * many triangles: thread per triangle; pass 1 atomicMin of the raw depth bits
//     (positive doubles order like their 64-bit patterns) into a shared-memory
//     tile, pass 2 atomicMin of the triangle index among the fragments whose
//     depth equals the pass-1 minimum.  A packed fp32-depth|id key would NOT
//     reproduce ownership on near-ties, hence two passes.
// All floating-point expressions keep the reference's operation order; the file
// is compiled with -fmad=false.
#include "px_color.cuh"
#include "px_kernels.h"

namespace px {

struct TriSetup {
  double u0, v0, u1, v1, u2, v2, iz0, iz1, iz2, inv_area;
  int px_lo, px_hi, py_lo, py_hi;
  int ia, ib, ic;  // vertex indices after the winding swap (for colours)
  int ok;
};

__device__ __forceinline__ int clamp_lo(double lo, int n) {  // max(0, int(ceil(x)))
  return lo < 0.0 ? 0 : (lo > (double)n ? n : (int)lo);
}
__device__ __forceinline__ int clamp_hi(double hi, int n) {  // min(n-1, int(floor(x)))
  return hi > (double)(n - 1) ? n - 1 : (hi < -1.0 ? -1 : (int)hi);
}

// raster.py:55-108 for one triangle, from the projected-vertex cache
__device__ __forceinline__ void setup_triangle(int ti, const int32_t* __restrict__ tris, const double* vu,
                                               const double* vv, const double* vz, int W, int H,
                                               TriSetup& s) {
  int ia = tris[3 * ti], ib = tris[3 * ti + 1], ic = tris[3 * ti + 2];
  double z0 = vz[ia], z1 = vz[ib], z2 = vz[ic];
  s.ok = 0;
  if (z0 <= PX_NEAR_PLANE || z1 <= PX_NEAR_PLANE || z2 <= PX_NEAR_PLANE) return;
  double u0 = vu[ia], v0 = vv[ia], u1 = vu[ib], v1 = vv[ib], u2 = vu[ic], v2 = vv[ic];
  double area2 = (u1 - u0) * (v2 - v0) - (v1 - v0) * (u2 - u0);
  if (area2 == 0.0) return;
  if (area2 < 0.0) {
    double t;
    t = u1, u1 = u2, u2 = t;
    t = v1, v1 = v2, v2 = t;
    t = z1, z1 = z2, z2 = t;
    int ti_ = ib;
    ib = ic, ic = ti_;
    area2 = -area2;
  }
  double umin = fmin(u0, fmin(u1, u2)), umax = fmax(u0, fmax(u1, u2));
  double vmin = fmin(v0, fmin(v1, v2)), vmax = fmax(v0, fmax(v1, v2));
  s.px_lo = clamp_lo(ceil(umin - 0.5), W);
  s.px_hi = clamp_hi(floor(umax - 0.5), W);
  s.py_lo = clamp_lo(ceil(vmin - 0.5), H);
  s.py_hi = clamp_hi(floor(vmax - 0.5), H);
  if (s.px_lo > s.px_hi || s.py_lo > s.py_hi) return;
  s.u0 = u0, s.v0 = v0, s.u1 = u1, s.v1 = v1, s.u2 = u2, s.v2 = v2;
  s.iz0 = 1.0 / z0, s.iz1 = 1.0 / z1, s.iz2 = 1.0 / z2;
  s.inv_area = 1.0 / area2;
  s.ia = ia, s.ib = ib, s.ic = ic;
  s.ok = 1;
}

// raster.py:109-125 for one pixel centre; returns false if not covered
__device__ __forceinline__ bool eval_pixel(const TriSetup& s, int px, int py, double& depth, double& b0,
                                           double& b1, double& b2) {
  const double e0u = s.u1 - s.u0, e0v = s.v1 - s.v0;
  const double e1u = s.u2 - s.u1, e1v = s.v2 - s.v1;
  const double e2u = s.u0 - s.u2, e2v = s.v0 - s.v2;
  const double sy = py + 0.5, sx = px + 0.5;
  const double w0 = e1u * (sy - s.v1) - e1v * (sx - s.u1);
  const double w1 = e2u * (sy - s.v2) - e2v * (sx - s.u2);
  const double w2 = e0u * (sy - s.v0) - e0v * (sx - s.u0);
  if (w0 < 0.0 || w1 < 0.0 || w2 < 0.0) return false;
  const bool tl0 = e0v < 0.0 || (e0v == 0.0 && e0u > 0.0);
  const bool tl1 = e1v < 0.0 || (e1v == 0.0 && e1u > 0.0);
  const bool tl2 = e2v < 0.0 || (e2v == 0.0 && e2u > 0.0);
  if ((w0 == 0.0 && !tl1) || (w1 == 0.0 && !tl2) || (w2 == 0.0 && !tl0)) return false;
  b0 = w0 * s.inv_area;
  b1 = w1 * s.inv_area;
  b2 = w2 * s.inv_area;
  const double inv_z = b0 * s.iz0 + b1 * s.iz1 + b2 * s.iz2;
  depth = 1.0 / inv_z;
  return true;
}

// ---------------------------------------------------------------------------
// K0: per-candidate stride-grid bounding box and cloud capacity.  Warp per
// candidate, lanes over vertices.  bbox = (gu_lo, gv_lo, gw, gh) in grid units.

__global__ void __launch_bounds__(256) bbox_kernel(RenderArgs a) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= a.n) return;
  const ModelDev m = a.models[a.model_slot[warp]];
  const double* P = a.poses + 12 * (size_t)warp;
  double p[12];
#pragma unroll
  for (int i = 0; i < 12; ++i) p[i] = P[i];
  double umin = CUDART_INF, umax = -CUDART_INF, vmin = CUDART_INF, vmax = -CUDART_INF;
  for (int i = lane; i < m.V; i += 32) {
    double x, y, z;
    apply_pose(p, m.verts[3 * i], m.verts[3 * i + 1], m.verts[3 * i + 2], x, y, z);
    if (z > PX_NEAR_PLANE) {
      double u = a.cam.fx * x / z + a.cam.cx, v = a.cam.fy * y / z + a.cam.cy;
      umin = fmin(umin, u), umax = fmax(umax, u), vmin = fmin(vmin, v), vmax = fmax(vmax, v);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    umin = fmin(umin, __shfl_xor_sync(0xffffffffu, umin, o));
    umax = fmax(umax, __shfl_xor_sync(0xffffffffu, umax, o));
    vmin = fmin(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
    vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
  }
  if (lane == 0) {
    int4 bb = make_int4(0, 0, 0, 0);
    if (umin <= umax) {
      const int s = a.cam.stride;
      int px_lo = clamp_lo(ceil(umin - 0.5), a.cam.W), px_hi = clamp_hi(floor(umax - 0.5), a.cam.W);
      int py_lo = clamp_lo(ceil(vmin - 0.5), a.cam.H), py_hi = clamp_hi(floor(vmax - 0.5), a.cam.H);
      if (px_lo <= px_hi && py_lo <= py_hi) {
        int gu_lo = (px_lo + s - 1) / s, gu_hi = px_hi / s;
        int gv_lo = (py_lo + s - 1) / s, gv_hi = py_hi / s;
        if (gu_lo <= gu_hi && gv_lo <= gv_hi) bb = make_int4(gu_lo, gv_lo, gu_hi - gu_lo + 1, gv_hi - gv_lo + 1);
      }
    }
    a.bbox[warp] = bb;
    a.cap[warp] = (long long)bb.z * bb.w;
  }
}

// ---------------------------------------------------------------------------
// K1: render.  Dynamic shared memory layout (doubles first):
//   vu[V] vv[V] vz[V]                          projected-vertex cache
//   path A: TriSetup[T]                        (T <= PX_TRI_SMEM)
//   path B: zbits[PX_TILE_PIX] u64, owner[PX_TILE_PIX] i32

template <bool DENSE>
#ifndef PX_RENDER_MINB
#define PX_RENDER_MINB (1024 / PX_RENDER_THREADS)  // 64 registers (swept 3..16 CTAs of 128 threads: 2.6 / 2.1 / 1.9 / 1.7 / 1.5 / 1.5 / 1.7 / 2.6 ms per launch)
#endif
__global__ void __launch_bounds__(PX_RENDER_THREADS, PX_RENDER_MINB) render_kernel(RenderArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int warp_tot[PX_RENDER_THREADS / 32];
  __shared__ int s_base;
  const int c = blockIdx.x;
  const int tid = threadIdx.x;
  const ModelDev m = a.models[a.model_slot[c]];
  const Camera cam = a.cam;
  const int4 bb = a.bbox[c];
  const int gw = bb.z, gh = bb.w;
  if (gw <= 0 || gh <= 0) {
    if (!DENSE && tid == 0) a.count[c] = 0;
    return;
  }
  double* vu = reinterpret_cast<double*>(smem_raw);
  double* vv = vu + m.V;
  double* vz = vv + m.V;
  unsigned char* after = reinterpret_cast<unsigned char*>(vz + m.V);
  __shared__ double sp[12];
  if (tid < 12) sp[tid] = a.poses[12 * (size_t)c + tid];
  __syncthreads();
  for (int i = tid; i < m.V; i += blockDim.x) {
    double x, y, z;
    apply_pose(sp, m.verts[3 * i], m.verts[3 * i + 1], m.verts[3 * i + 2], x, y, z);
    vz[i] = z;
    // raster.py:61-66: (fx * x) / z + cx ; only evaluated for z > near in the reference
    vu[i] = z > PX_NEAR_PLANE ? cam.fx * x / z + cam.cx : 0.0;
    vv[i] = z > PX_NEAR_PLANE ? cam.fy * y / z + cam.cy : 0.0;
  }
  const bool path_a = m.T <= PX_TRI_SMEM;
  TriSetup* tsm = reinterpret_cast<TriSetup*>(after);
  unsigned long long* zbits = reinterpret_cast<unsigned long long*>(after);
  int* owner = reinterpret_cast<int*>(zbits + PX_TILE_PIX);
  __syncthreads();
  if (path_a) {
    for (int ti = tid; ti < m.T; ti += blockDim.x) {
      TriSetup s;
      setup_triangle(ti, m.tris, vu, vv, vz, cam.W, cam.H, s);
      tsm[ti] = s;
    }
    __syncthreads();
  }
  const int st = cam.stride;
  const long long out0 = DENSE ? 0 : a.offset[c];
  if (tid == 0) s_base = 0;
  // tiles are bands of whole grid rows so that tile order == row-major order
  const int rows_per_tile = path_a ? gh : max(1, PX_TILE_PIX / gw);
  for (int r0 = 0; r0 < gh; r0 += rows_per_tile) {
    const int rows = min(rows_per_tile, gh - r0);
    const int npix = rows * gw;
    if (!path_a) {
      for (int i = tid; i < npix; i += blockDim.x) zbits[i] = dbits(CUDART_INF), owner[i] = 0x7fffffff;
      __syncthreads();
      const int py0 = (bb.y + r0) * st, py1 = (bb.y + r0 + rows - 1) * st;
      const int px0 = bb.x * st, px1 = (bb.x + gw - 1) * st;
      for (int pass = 0; pass < 2; ++pass) {
        for (int ti = tid; ti < m.T; ti += blockDim.x) {
          TriSetup s;
          setup_triangle(ti, m.tris, vu, vv, vz, cam.W, cam.H, s);
          if (!s.ok) continue;
          const int ylo = max(s.py_lo, py0), yhi = min(s.py_hi, py1);
          const int xlo = max(s.px_lo, px0), xhi = min(s.px_hi, px1);
          for (int py = ((ylo + st - 1) / st) * st; py <= yhi; py += st)
            for (int px = ((xlo + st - 1) / st) * st; px <= xhi; px += st) {
              double d, b0, b1, b2;
              if (!eval_pixel(s, px, py, d, b0, b1, b2)) continue;
              if (!(d < CUDART_INF)) continue;
              const int li = (py / st - bb.y - r0) * gw + (px / st - bb.x);
              if (pass == 0)
                atomicMin(&zbits[li], dbits(d));
              else if (dbits(d) == zbits[li])
                atomicMin(&owner[li], ti);
            }
        }
        __syncthreads();
      }
    }
    // resolve in row-major chunks of blockDim pixels with an ordered compaction
    for (int base = 0; base < npix; base += blockDim.x) {
      const int li = base + tid;
      bool have = false;
      double depth = 0.0, b0 = 0.0, b1 = 0.0, b2 = 0.0;
      int own = -1, px = 0, py = 0;
      TriSetup s;
      if (li < npix) {
        const int gy = li / gw, gx = li - gy * gw;
        px = (bb.x + gx) * st, py = (bb.y + r0 + gy) * st;
        if (path_a) {
          double best = CUDART_INF;
          for (int ti = 0; ti < m.T; ++ti) {
            const TriSetup& t = tsm[ti];
            if (!t.ok || px < t.px_lo || px > t.px_hi || py < t.py_lo || py > t.py_hi) continue;
            double d, c0, c1, c2;
            if (!eval_pixel(t, px, py, d, c0, c1, c2)) continue;
            if (d < best) best = d, own = ti, b0 = c0, b1 = c1, b2 = c2;
          }
          if (own >= 0) have = true, depth = best, s = tsm[own];
        } else if (owner[li] != 0x7fffffff) {
          own = owner[li];
          setup_triangle(own, m.tris, vu, vv, vz, cam.W, cam.H, s);
          have = eval_pixel(s, px, py, depth, b0, b1, b2);  // same bits as pass 1
        }
        if (have && !DENSE && a.occluder_marking) {  // raster.py:263-270
          const size_t o = (size_t)(bb.y + r0 + gy) * cam.GW + (bb.x + gx);  // the observed planes are stride-grid sampled
          if (a.obs_valid[o] && a.obs_depth[o] < depth - a.delta_occ && a.obs_labels[o] != m.object_id) have = false;
        }
      }
      double cr = 0.0, cg = 0.0, cb = 0.0;
      if (have) {  // raster.py:128-133
        const double s0 = b0 * s.iz0 * depth, s1 = b1 * s.iz1 * depth, s2 = b2 * s.iz2 * depth;
        const double *k0 = m.col + 3 * s.ia, *k1 = m.col + 3 * s.ib, *k2 = m.col + 3 * s.ic;
        cr = s0 * k0[0] + s1 * k1[0] + s2 * k2[0];
        cg = s0 * k0[1] + s1 * k1[1] + s2 * k2[1];
        cb = s0 * k0[2] + s1 * k1[2] + s2 * k2[2];
      }
      if (!DENSE && li < npix) a.slot_map[out0 + (long long)r0 * gw + li] = -1;
      if (DENSE) {
        if (have) {
          const size_t o = (size_t)py * cam.W + px;
          a.dense_z[o] = depth;
          a.dense_c[3 * o] = cr, a.dense_c[3 * o + 1] = cg, a.dense_c[3 * o + 2] = cb;
          a.dense_valid[o] = 1;
          a.dense_owner[o] = own;
        }
        continue;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, have);
      const int wid = tid >> 5, ln = tid & 31;
      if (ln == 0) warp_tot[wid] = __popc(bal);
      __syncthreads();
      int pos = s_base + __popc(bal & ((1u << ln) - 1u));
      for (int w = 0; w < wid; ++w) pos += warp_tot[w];
      int chunk_total = 0;
      for (int w = 0; w < PX_RENDER_THREADS / 32; ++w) chunk_total += warp_tot[w];
      if (have) {  // raster.py:277-279
        const long long o = out0 + pos;
        a.points[3 * o] = ((px + 0.5) - cam.cx) * depth / cam.fx;
        a.points[3 * o + 1] = ((py + 0.5) - cam.cy) * depth / cam.fy;
        a.points[3 * o + 2] = depth;
        if (!a.skip_lab) {  // raster.py:278 (6 pow + 3 cbrt per point: 40 % of this kernel)
          double L, A, B;
          srgb_to_lab(srgb_encode1(cr), srgb_encode1(cg), srgb_encode1(cb), L, A, B);
          a.lab[3 * o] = L, a.lab[3 * o + 1] = A, a.lab[3 * o + 2] = B;
        } else if (a.skip_lab == 2) {
          a.lab[3 * o] = cr, a.lab[3 * o + 1] = cg, a.lab[3 * o + 2] = cb;
        }
        a.src_px[2 * o] = px, a.src_px[2 * o + 1] = py;
        a.slot_map[out0 + (long long)r0 * gw + li] = pos;
      }
      __syncthreads();
      if (tid == 0) s_base += chunk_total;
      __syncthreads();
    }
  }
  if (!DENSE && tid == 0) a.count[c] = s_base;
}

size_t render_smem_bytes(int V, int T) {
  size_t b = sizeof(double) * 3 * (size_t)V;
  size_t extra = T <= PX_TRI_SMEM ? sizeof(TriSetup) * (size_t)T
                                  : (sizeof(unsigned long long) + sizeof(int)) * (size_t)PX_TILE_PIX;
  return b + extra + 16;
}

cudaError_t launch_bbox(const RenderArgs& a, cudaStream_t st) {
  if (a.n == 0) return cudaSuccess;
  const int wpb = 8;
  bbox_kernel<<<(a.n + wpb - 1) / wpb, wpb * 32, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_render(const RenderArgs& a, size_t smem, bool dense, cudaStream_t st) {
  if (a.n == 0) return cudaSuccess;
  cudaError_t e;
  if (dense) {
    e = cudaFuncSetAttribute(render_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    render_kernel<true><<<a.n, PX_RENDER_THREADS, smem, st>>>(a);
  } else {
    e = cudaFuncSetAttribute(render_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    render_kernel<false><<<a.n, PX_RENDER_THREADS, smem, st>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace px
