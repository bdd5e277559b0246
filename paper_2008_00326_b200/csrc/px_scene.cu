// px_scene.cu -- per-scene set-up on the device.
//
//  * the observed cloud of a frame: raster.frame_to_cloud / _grid_cloud and cloud_labels (reference
//    pkg/src/rvpose/raster.py:191-217) -- stride-grid sampling of the valid mask, row-major compaction
//    (np.nonzero order), unprojection at the pixel centre (geometry.py:222-231, same operation order:
//    ((u + 0.5) - cx) * z / fx), sRGB -> Lab (colorspace.py:41-55), label per point; plus the organised
//    grid views the cost and target kernels read.  Points / pixels / labels are bit-identical to the host
//    path, Lab agrees to ~1e-12 (libdevice pow / cbrt vs numpy) and only feeds the dE gate.
//  * the candidate lattice: proposals.grid_proposals_3dof / pose_proposals_6dof are outer x inner products
//    (proposals.py:163-210); the per-candidate camera pose `world_to_cam.compose(pose_i)` (search.py:253-255) is
//    formed here in the host BLAS rounding order (px_common.cuh), so a search uploads O(outer + inner) numbers
//    per object instead of 108 bytes per candidate.  The shard of a rank (dist.shard_index: outer index modulo
//    world size) is generated directly.
#include "px_color.cuh"
#include "px_kernels.h"

namespace px {

// valid stride-grid pixels of every grid row (warp per row)
__global__ void __launch_bounds__(128) scene_count_kernel(SceneCloudArgs a) {
  const int gv = blockIdx.x * 4 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (gv >= a.GH) return;
  const uint8_t* row = a.valid + (size_t)gv * a.GW;
  int cnt = 0;
  for (int gu = lane; gu < a.GW; gu += 32) cnt += row[gu] != 0;
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if (lane == 0) a.row_count[gv] = cnt;
}

__global__ void __launch_bounds__(128) scene_fill_kernel(SceneCloudArgs a) {
  const int gv = blockIdx.x * 4 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (gv >= a.GH) return;
  const int v = gv * a.stride;
  long long base = a.row_offset[gv];
  for (int g0 = 0; g0 < a.GW; g0 += 32) {
    const int gu = g0 + lane;
    const int u = gu * a.stride;
    const bool in = gu < a.GW;
    const bool ok = in && a.valid[(size_t)gv * a.GW + gu] != 0;
    const unsigned m = __ballot_sync(0xffffffffu, ok);
    const long long i = base + __popc(m & ((1u << lane) - 1u));
    base += __popc(m);
    if (!in) continue;
    const size_t cell = (size_t)gv * a.GW + gu;
    if (!ok) {
      a.gx[cell] = a.gy[cell] = a.gz[cell] = CUDART_NAN;
      a.gidx[cell] = -1;
      continue;
    }
    const double z = a.depth[cell];
    const double x = (((double)u + 0.5) - a.cx) * z / a.fx;  // geometry.py:231
    const double y = (((double)v + 0.5) - a.cy) * z / a.fy;
    a.pts[3 * i] = x, a.pts[3 * i + 1] = y, a.pts[3 * i + 2] = z;
    a.gx[cell] = x, a.gy[cell] = y, a.gz[cell] = z;
    a.gidx[cell] = (int32_t)i;
    a.src[2 * i] = u, a.src[2 * i + 1] = v;
    a.cell[i] = (int32_t)cell;
    a.labels_out[i] = a.labels[cell];  // raster.py:217
    const double* c = a.color_grid + 3 * cell;
    double L, A, B;
    srgb_to_lab(c[0], c[1], c[2], L, A, B);
    a.lab[3 * i] = L, a.lab[3 * i + 1] = A, a.lab[3 * i + 2] = B;
  }
}

cudaError_t launch_scene_count(const SceneCloudArgs& a, cudaStream_t st) {
  scene_count_kernel<<<(a.GH + 3) / 4, 128, 0, st>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_scene_fill(const SceneCloudArgs& a, cudaStream_t st) {
  scene_fill_kernel<<<(a.GH + 3) / 4, 128, 0, st>>>(a);
  return cudaGetLastError();
}

// count(label == object id) per model slot (cost.py:147-152 in label mode needs |selected|)
__global__ void label_count_kernel(const int32_t* __restrict__ labels, long long n, const ModelDev* models, int n_models,
                                   int32_t* __restrict__ out) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int l = labels[i];
  for (int s = 0; s < n_models; ++s)
    if (models[s].object_id == l) atomicAdd(&out[s], 1);
}
cudaError_t launch_label_count(const int32_t* labels, long long n, const ModelDev* models, int n_models, int32_t* out,
                               cudaStream_t st) {
  if (n <= 0 || n_models <= 0) return cudaSuccess;
  label_count_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(labels, n, models, n_models, out);
  return cudaGetLastError();
}

// ---- candidate lattice ---------------------------------------------------------------------------

__global__ void __launch_bounds__(256) lattice_kernel(LatticeArgs a) {
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= a.n_local) return;
  int o = 0;
  while (o + 1 < a.n_objects && c >= a.objs[o + 1].cand_off) ++o;
  const LatticeObjDev L = a.objs[o];
  const long long q = c - L.cand_off;
  const int k = (int)(q / L.n_inner), b = (int)(q - (long long)k * L.n_inner);
  const int outer = a.rank + k * a.world;  // dist.shard_index: outer index modulo world size
  double pose[12];
  if (a.mode3dof) {
    // search.py:253-255: world_to_cam.compose(lift(x, y, yaw)); rotation = yaw spin b, translation = cell `outer`
    const double* R = a.rotations + 9 * (L.rot_off + b);
    const double* t = a.translations + 3 * (L.tr_off + outer);
    const double lift[12] = {R[0], R[1], R[2], t[0], R[3], R[4], R[5], t[1], R[6], R[7], R[8], t[2]};
    compose_pose(a.w2c, lift, a.w2c_vec_order, pose);
  } else {
    // search.py:257: 6-DoF hypotheses live in the camera frame already; rotation `outer`, translation b
    const double* R = a.rotations + 9 * (L.rot_off + outer);
    const double* t = a.translations + 3 * (L.tr_off + b);
    for (int i = 0; i < 3; ++i) pose[4 * i] = R[3 * i], pose[4 * i + 1] = R[3 * i + 1], pose[4 * i + 2] = R[3 * i + 2], pose[4 * i + 3] = t[i];
  }
  for (int i = 0; i < 12; ++i) a.poses[12 * c + i] = pose[i];
  a.slot[c] = L.slot;
  a.rank_in_object[c] = (int32_t)((long long)outer * L.n_inner + b);
  if (a.tidx) a.tidx[c] = a.mode3dof ? L.tgt_off + k : L.tgt_off;
  if (a.capsules && a.mode3dof && b == 0) {  // search.py:407-426: one capsule target per (object, grid cell)
    const double* t = a.translations + 3 * (L.tr_off + outer);
    double* p = a.capsules + 5 * (size_t)(L.tgt_off + k);
    p[0] = t[0], p[1] = t[1], p[2] = L.z_lo, p[3] = L.z_hi, p[4] = L.radius;
  }
}

cudaError_t launch_lattice(const LatticeArgs& a, cudaStream_t st) {
  if (a.n_local <= 0) return cudaSuccess;
  lattice_kernel<<<(unsigned)((a.n_local + 255) / 256), 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace px
