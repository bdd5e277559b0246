// px_cost.cu -- PERCH explanation cost per candidate, exact kNN, fused argmin.
//
// Replaces search._cost_task, cost.rendered_cost / select_observed /
// observed_cost and neighbors._streamed_kernel (reference pkg/src/rvpose/
// search.py:189-202, cost.py:91-152, neighbors.py:104-134).
//
// Organised path (the search path): the observed cloud is the stride-grid
// unprojection of the depth image (raster.py:197-210), stored here both
// compactly and as a (GH,GW) grid.  For a rendered point q every observed
// point within delta of q projects within
//     r_u = fx*delta*(1+|x_q/z_q|)/(z_q-delta)   pixels of q's projection
// (and likewise r_v), so scanning that pixel window in row-major order with a
// strict `<` yields exactly the reference's global brute-force
// (d2, lowest index) minimum whenever it passes the `d2 <= delta^2` gate; a
// query whose true nearest neighbour is farther than delta is an outlier under
// either search.  Row-major grid order == observed index order.
//
// `explained` is a set (cost.py:131-134): a per-warp bitmap over grid pixels.
// j_o = |selected| - |selected & explained| with `selected` the closed
// inscribed-cylinder test in the candidate's object frame (cost.py:143-144,
// model.py:67-72; evaluated only inside the cylinder's screen bound) or the
// pixel label (search.py:197-199).
#include "px_color.cuh"
#include "px_kernels.h"

namespace px {

__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ int warp_min(int v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_max(int v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

#ifndef PX_COST_MINB
#define PX_COST_MINB (32 / PX_COST_WARPS)  // 64 registers (swept 3..16 CTAs of 4 warps: 4.0 / 3.5 / 3.3 / 3.2 / 2.4 / 2.9 / 3.3 / 3.5 ms)
#endif
__global__ void __launch_bounds__(PX_COST_WARPS * 32, PX_COST_MINB) cost_kernel(CostArgs a) {
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Camera cam = a.cam;
  const int GW = cam.GW, GH = cam.GH, st = cam.stride;
  // persistent warps: warp slot s owns bitmap s and strides over the candidates
  const int slot_id = blockIdx.x * PX_COST_WARPS + wid;
  uint32_t* bm = a.bitmap + (size_t)slot_id * a.bitmap_words;
  for (int c = slot_id; c < a.ren.n; c += gridDim.x * PX_COST_WARPS) {
  const int n = a.ren.count[c];
  const long long off = a.ren.offset[c];
  const double* rp = a.ren.points + 3 * off;
  const double* rl = a.ren.lab + 3 * off;
  const int slot = a.model_slot[c];
  const ModelDev m = a.models[slot];

  // ---- pass 1: rendered points -> nearest observed, gates, explained bits ----
  int within = 0, color_fail = 0;
  double knife_d = CUDART_INF, knife_c = CUDART_INF;  // how close any gate decision came to its threshold
  int e_lo_u = GW, e_hi_u = -1, e_lo_v = GH, e_hi_v = -1;  // bounds of set bits (grid units)
  for (int i = lane; i < n; i += 32) {
    const double qx = rp[3 * i], qy = rp[3 * i + 1], qz = rp[3 * i + 2];
    int gu0 = 0, gv0 = 0, gu1 = GW - 1, gv1 = GH - 1;
    if (qz > a.delta) {
      const double zr = qz - a.delta;
      const double ru = cam.fx * a.delta * (1.0 + fabs(qx / qz)) / zr + 1e-6;
      const double rv = cam.fy * a.delta * (1.0 + fabs(qy / qz)) / zr + 1e-6;
      const double uq = cam.fx * qx / qz + cam.cx, vq = cam.fy * qy / qz + cam.cy;  // continuous pixel coords
      // observed point at grid (gu,gv) sits at continuous pixel (gu*st+0.5, gv*st+0.5); the clamps run in
      // floating point so that huge windows cannot overflow the int conversion
      const double u0 = ceil((uq - ru - 0.5) / st), u1 = floor((uq + ru - 0.5) / st);
      const double v0 = ceil((vq - rv - 0.5) / st), v1 = floor((vq + rv - 0.5) / st);
      gu0 = (int)fmin(fmax(u0, 0.0), (double)GW), gu1 = (int)fmax(fmin(u1, (double)(GW - 1)), -1.0);
      gv0 = (int)fmin(fmax(v0, 0.0), (double)GH), gv1 = (int)fmax(fmin(v1, (double)(GH - 1)), -1.0);
    }  // else: a point closer to the camera than delta has no bounded window -- the whole grid is scanned (exact)
    double best = CUDART_INF;
    int bg = -1;
    for (int gv = gv0; gv <= gv1; ++gv)
      for (int gu = gu0; gu <= gu1; ++gu) {
        const int g = gv * GW + gu;
        const double dx = a.gx[g] - qx, dy = a.gy[g] - qy, dz = a.gz[g] - qz;
        const double d2 = dx * dx + dy * dy + dz * dz;  // NaN where the grid has no point
        if (d2 < best) best = d2, bg = g;
      }
    if (bg >= 0) knife_d = fmin(knife_d, fabs(best - a.delta2));
    if (bg < 0 || !(best <= a.delta2)) continue;
    ++within;
    const int j = a.gidx[bg];
    if (a.use_color) {
      const double* ol = a.obs_lab + 3 * (size_t)j;
      double L = rl[3 * i], A = rl[3 * i + 1], B = rl[3 * i + 2];
      if (a.lab_is_linear)  // raster.py:278 evaluated only for the points that reach the colour gate
        srgb_to_lab(srgb_encode1(L), srgb_encode1(A), srgb_encode1(B), L, A, B);
      const double de = ciede2000(L, A, B, ol[0], ol[1], ol[2]);
      knife_c = fmin(knife_c, fabs(de - a.tau_c));
      if (!(de <= a.tau_c)) {
        ++color_fail;
        continue;
      }
    }
    atomicOr(&bm[bg >> 5], 1u << (bg & 31));
    const int gv = bg / GW, gu = bg - gv * GW;
    e_lo_u = min(e_lo_u, gu), e_hi_u = max(e_hi_u, gu), e_lo_v = min(e_lo_v, gv), e_hi_v = max(e_hi_v, gv);
  }
  within = warp_sum(within);
  color_fail = warp_sum(color_fail);
  if (a.knife) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      knife_d = fmin(knife_d, __shfl_xor_sync(0xffffffffu, knife_d, o));
      knife_c = fmin(knife_c, __shfl_xor_sync(0xffffffffu, knife_c, o));
    }
    if (lane == 0) {  // non-negative doubles order like their bit patterns
      if (knife_d < bits_d(*(volatile unsigned long long*)&a.knife[0])) atomicMin(&a.knife[0], dbits(knife_d));
      if (knife_c < bits_d(*(volatile unsigned long long*)&a.knife[1])) atomicMin(&a.knife[1], dbits(knife_c));
    }
  }
  e_lo_u = warp_min(e_lo_u), e_lo_v = warp_min(e_lo_v), e_hi_u = warp_max(e_hi_u), e_hi_v = warp_max(e_hi_v);
  const int j_r = n - within + color_fail;
  __threadfence();
  __syncwarp();

  // ---- pass 2: observed points selected for this candidate ----
  int j_o = 0, n_foot = 0;
  if (a.cyl_poses) {
    const double* P = a.cyl_poses + 12 * (size_t)c;
    double p[12];
#pragma unroll
    for (int i = 0; i < 12; ++i) p[i] = P[i];
    // screen bound of the cylinder's bounding box (superset of the cylinder)
    const double rad = m.aabb_r;
    double umin = CUDART_INF, umax = -CUDART_INF, vmin = CUDART_INF, vmax = -CUDART_INF;
    bool behind = false;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double ox = (k & 1) ? rad : -rad, oy = (k & 2) ? rad : -rad, oz = (k & 4) ? m.cyl_zmax : m.cyl_zmin;
      const double x = p[0] * ox + p[1] * oy + p[2] * oz + p[3];
      const double y = p[4] * ox + p[5] * oy + p[6] * oz + p[7];
      const double z = p[8] * ox + p[9] * oy + p[10] * oz + p[11];
      if (!(z > 1e-3)) behind = true;
      const double u = cam.fx * x / z + cam.cx, v = cam.fy * y / z + cam.cy;
      umin = fmin(umin, u), umax = fmax(umax, u), vmin = fmin(vmin, v), vmax = fmax(vmax, v);
    }
    int gu0 = 0, gu1 = GW - 1, gv0 = 0, gv1 = GH - 1;
    if (!behind && isfinite(umin) && isfinite(umax) && isfinite(vmin) && isfinite(vmax)) {
      // one full pixel of slack on every side
      const double a0 = floor((umin - 1.5) / st), a1 = ceil((umax + 0.5) / st);
      const double b0 = floor((vmin - 1.5) / st), b1 = ceil((vmax + 0.5) / st);
      gu0 = a0 < 0.0 ? 0 : (a0 > (double)GW ? GW : (int)a0);
      gv0 = b0 < 0.0 ? 0 : (b0 > (double)GH ? GH : (int)b0);
      gu1 = a1 > (double)(GW - 1) ? GW - 1 : (a1 < -1.0 ? -1 : (int)a1);
      gv1 = b1 > (double)(GH - 1) ? GH - 1 : (b1 < -1.0 ? -1 : (int)b1);
    }
    // inverse pose in the reference's rounding (geometry.py:143-145 + :131-134)
    const double ti0 = dot_f012(-p[0], -p[4], -p[8], p[3], p[7], p[11]);
    const double ti1 = dot_f012(-p[1], -p[5], -p[9], p[3], p[7], p[11]);
    const double ti2 = dot_f012(-p[2], -p[6], -p[10], p[3], p[7], p[11]);
    const int w = gu1 - gu0 + 1, h = gv1 - gv0 + 1;
    const int tot = (w > 0 && h > 0) ? w * h : 0;
    for (int q = lane; q < tot; q += 32) {
      const int gv = gv0 + q / w, gu = gu0 + q % w;
      const int g = gv * GW + gu;
      const double ox = a.gx[g], oy = a.gy[g], oz = a.gz[g];
      const double x = dot_f012(ox, oy, oz, p[0], p[4], p[8]) + ti0;
      const double y = dot_f012(ox, oy, oz, p[1], p[5], p[9]) + ti1;
      const double z = dot_f012(ox, oy, oz, p[2], p[6], p[10]) + ti2;
      const bool sel = (x * x + y * y <= m.cyl_r2) && z >= m.cyl_zmin && z <= m.cyl_zmax;  // false on NaN
      n_foot += sel;
      if (sel && !((__ldcg(&bm[g >> 5]) >> (g & 31)) & 1u)) ++j_o;
    }
    j_o = warp_sum(j_o);
    n_foot = warp_sum(n_foot);
  } else {
    // label mode: j_o = count(label == oid) - count(label == oid & explained)
    int hit = 0;
    const int w = e_hi_u - e_lo_u + 1, h = e_hi_v - e_lo_v + 1;
    const int tot = (w > 0 && h > 0) ? w * h : 0;
    for (int q = lane; q < tot; q += 32) {
      const int gv = e_lo_v + q / w, gu = e_lo_u + q % w;
      const int g = gv * GW + gu;
      if ((__ldcg(&bm[g >> 5]) >> (g & 31)) & 1u) {
        const int j = a.gidx[g];
        if (j >= 0 && a.obs_labels[j] == m.object_id) ++hit;
      }
    }
    j_o = a.label_count[slot] - warp_sum(hit);
    n_foot = a.label_count[slot];
  }
  __syncwarp();
  // ---- clear the bits we set (bitmap is clean on entry and exit) ----
  {
    const int w = e_hi_u - e_lo_u + 1, h = e_hi_v - e_lo_v + 1;
    if (w > 0 && h > 0) {
      const int w0 = (e_lo_v * GW + e_lo_u) >> 5, w1 = (e_hi_v * GW + e_hi_u) >> 5;
      for (int q = w0 + lane; q <= w1; q += 32) __stcg(&bm[q], 0u);
    }
  }
  if (lane == 0) {
    a.j_o[c] = j_o;
    a.j_r[c] = j_r;
    if (a.n_match) a.n_match[c] = within;
    if (a.n_foot) a.n_foot[c] = n_foot;
    if (a.best_key) {
      const unsigned long long key = ((unsigned long long)(unsigned)(j_o + j_r) << 32) | (unsigned)a.rank[c];
      atomicMin(&a.best_key[slot], key);
    }
  }
  __syncwarp();
  }  // candidate loop
}

cudaError_t launch_cost(const CostArgs& a, cudaStream_t st) {
  if (a.ren.n == 0) return cudaSuccess;
  int blocks = (a.ren.n + PX_COST_WARPS - 1) / PX_COST_WARPS;
  if (blocks > a.bitmap_slots / PX_COST_WARPS) blocks = a.bitmap_slots / PX_COST_WARPS;
  cost_kernel<<<blocks, PX_COST_WARPS * 32, 0, st>>>(a);
  return cudaGetLastError();
}

// search.py:346-372 on the device: the record of every object's winning candidate (see WinnerArgs)
__global__ void __launch_bounds__(256) winner_kernel(WinnerArgs a) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= a.n) return;
  const int slot = a.model_slot[c];
  unsigned long long* w = a.win + (size_t)slot * PX_WIN_WORDS;
  const unsigned long long nf = (unsigned long long)(unsigned)a.n_final[c];
  if (nf > *(volatile unsigned long long*)&w[27]) atomicMax(&w[27], nf);  // racy read = filter only
  const unsigned long long key = ((unsigned long long)(unsigned)(a.j_o[c] + a.j_r[c]) << 32) | (unsigned)a.rank[c];
  if (key != a.best_key[slot]) return;
  w[0] = key + 1ull;  // 0 = no candidate anywhere
  for (int q = 0; q < 12; ++q) {
    w[1 + q] = dbits(a.refined[12 * (size_t)c + q]);
    w[13 + q] = dbits(a.reg_T[12 * (size_t)c + q]);
  }
  w[25] = (unsigned long long)(unsigned)a.j_o[c];
  w[26] = (unsigned long long)(unsigned)a.j_r[c];
}

cudaError_t launch_winners(const WinnerArgs& a, cudaStream_t st) {
  if (a.n == 0) return cudaSuccess;
  winner_kernel<<<(a.n + 255) / 256, 256, 0, st>>>(a);
  return cudaGetLastError();
}

// colorspace.ciede2000 / srgb_to_lab for arrays (test exports: the device functions the cost and render kernels inline)
__global__ void ciede_kernel(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) out[i] = ciede2000(a[3 * i], a[3 * i + 1], a[3 * i + 2], b[3 * i], b[3 * i + 1], b[3 * i + 2]);
}
__global__ void lab_kernel(const double* __restrict__ rgb, double* __restrict__ out, long long n, int encode_first) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double r = rgb[3 * i], g = rgb[3 * i + 1], b = rgb[3 * i + 2];
  if (encode_first) r = srgb_encode1(r), g = srgb_encode1(g), b = srgb_encode1(b);  // raster.py:278 on linear colours
  srgb_to_lab(r, g, b, out[3 * i], out[3 * i + 1], out[3 * i + 2]);
}
cudaError_t launch_ciede(const double* a, const double* b, double* out, long long n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  ciede_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(a, b, out, n);
  return cudaGetLastError();
}
cudaError_t launch_lab(const double* rgb, double* out, long long n, int encode_first, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  lab_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(rgb, out, n, encode_first);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// exact brute-force kNN (neighbors.py:104-134), thread per query

__global__ void __launch_bounds__(128) knn_kernel(KnnArgs a) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.nq) return;
  double od[PX_KCOV_MAX];
  long long oi[PX_KCOV_MAX];
  const int k = a.k;
  for (int q = 0; q < k; ++q) od[q] = CUDART_INF, oi[q] = -1;
  const double qx = a.q[3 * i], qy = a.q[3 * i + 1], qz = a.q[3 * i + 2];
  int cnt = 0;
  for (long long j = 0; j < a.nt; ++j) {
    const double dx = a.t[3 * j] - qx, dy = a.t[3 * j + 1] - qy, dz = a.t[3 * j + 2] - qz;
    const double d2 = dx * dx + dy * dy + dz * dz;
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
  for (int q = 0; q < k; ++q) a.idx[i * k + q] = oi[q], a.d2[i * k + q] = od[q];
}

cudaError_t launch_knn(const KnnArgs& a, cudaStream_t st) {
  if (a.nq == 0) return cudaSuccess;
  knn_kernel<<<(unsigned)((a.nq + 127) / 128), 128, 0, st>>>(a);
  return cudaGetLastError();
}

// cost.py:91-135 for arbitrary clouds: thread per rendered point, brute force
__global__ void __launch_bounds__(128) generic_cost_kernel(GenericCostArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n_r) return;
  const double qx = a.rp[3 * i], qy = a.rp[3 * i + 1], qz = a.rp[3 * i + 2];
  double best = CUDART_INF;
  long long bj = -1;
  for (long long j = 0; j < a.n_obs; ++j) {
    const double dx = a.op[3 * j] - qx, dy = a.op[3 * j + 1] - qy, dz = a.op[3 * j + 2] - qz;
    const double d2 = dx * dx + dy * dy + dz * dz;
    if (d2 < best) best = d2, bj = j;
  }
  bool outlier = true;
  if (bj >= 0 && best <= a.delta2) {
    outlier = false;
    if (a.use_color) {
      const double* ql = a.rlab + 3 * (size_t)i;
      const double* ol = a.olab + 3 * (size_t)bj;
      if (!(ciede2000(ql[0], ql[1], ql[2], ol[0], ol[1], ol[2]) <= a.tau_c)) outlier = true;
    }
    if (!outlier) a.explained[bj] = 1;
  }
  if (outlier) atomicAdd(a.j_r, 1);
}

cudaError_t launch_generic_cost(const GenericCostArgs& a, cudaStream_t st) {
  if (a.n_r == 0) return cudaSuccess;
  generic_cost_kernel<<<(a.n_r + 127) / 128, 128, 0, st>>>(a);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// plumbing kernels: exclusive scan of capacities (single CTA), dense fill

__global__ void __launch_bounds__(1024) scan_kernel(const long long* in, long long* out, long long* total, int n) {
  __shared__ long long part[1024];
  const int tid = threadIdx.x;
  const int per = (n + 1023) / 1024;
  const int lo = min(n, tid * per), hi = min(n, lo + per);
  long long s = 0;
  for (int i = lo; i < hi; ++i) s += in[i];
  part[tid] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    long long v = tid >= o ? part[tid - o] : 0;
    __syncthreads();
    part[tid] += v;
    __syncthreads();
  }
  long long run = tid ? part[tid - 1] : 0;
  for (int i = lo; i < hi; ++i) {
    out[i] = run;
    run += in[i];
  }
  if (tid == 1023) *total = part[1023];
}

cudaError_t launch_scan(const long long* in, long long* out_excl, long long* total, int n, cudaStream_t st) {
  scan_kernel<<<1, 1024, 0, st>>>(in, out_excl, total, n);
  return cudaGetLastError();
}

__global__ void fill_dense_kernel(double* z, double* c, uint8_t* valid, int32_t* owner, size_t npix) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npix) return;
  z[i] = CUDART_INF;
  c[3 * i] = c[3 * i + 1] = c[3 * i + 2] = 0.0;
  valid[i] = 0;
  owner[i] = -1;
}

cudaError_t launch_fill_dense(double* z, double* c, uint8_t* valid, int32_t* owner, size_t npix, cudaStream_t st) {
  fill_dense_kernel<<<(unsigned)((npix + 255) / 256), 256, 0, st>>>(z, c, valid, owner, npix);
  return cudaGetLastError();
}

}  // namespace px
