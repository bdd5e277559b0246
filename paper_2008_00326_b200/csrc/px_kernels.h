// px_kernels.h -- kernel argument blocks and launchers shared by the libpx
// translation units (internal; the public C-ABI is include/px.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "px_common.cuh"

#ifndef PX_RENDER_THREADS
#define PX_RENDER_THREADS 64   // swept 32 / 64 / 128 / 256 at 64 registers: 1.40 / 1.43 / 1.50 / 1.74 ms per launch (32 slows the NN kernel's neighbours in the L2)
#endif
#define PX_TRI_SMEM 64      // meshes up to this many triangles use the per-pixel path
#define PX_TILE_PIX 4096    // stride-grid pixels per shared-memory z tile (atomic path)
#ifndef PX_GICP_WARPS
#define PX_GICP_WARPS 2     // candidates (warps) per CTA in the GICP linearise kernel (tuned by sweep)
#endif
#ifndef PX_GICP_MINB
#define PX_GICP_MINB 8      // min resident CTAs per SM requested from ptxas (register budget: 128/thread)
#endif
#ifndef PX_COST_WARPS
#define PX_COST_WARPS 16      // persistent warps per CTA, 148 x 32 of them in all (swept 2 / 4 / 8 / 16: 3.5 / 2.5 / 2.3 / 2.2 ms)
#endif
#define PX_KCOV_MAX 32

namespace px {

struct ModelDev {
  const double* verts;  // (V,3) object frame
  const double* col;    // (V,3) linear-light colour
  const int32_t* tris;  // (T,3)
  int V, T;
  int32_t object_id;
  int pad_;
  double cyl_r2, cyl_zmin, cyl_zmax;
  double aabb_r;        // sqrt(cyl_r2) upper bound used only for screen bounds
};

struct RenderArgs {
  Camera cam;
  const ModelDev* models;
  const int32_t* model_slot;  // (n)
  const double* poses;        // (n,12)
  int n;
  int occluder_marking;
  int skip_lab;               // 1: leave `lab` unwritten (first render of a refining search: GICP reads points only);
                              // 2: store the linear-light colour there instead (the cost kernel converts on demand)
  double delta_occ;
  const double* obs_depth;    // (GH,GW): the observed planes at the stride-grid pixels (all the batch path ever reads)
  const uint8_t* obs_valid;
  const int32_t* obs_labels;
  int4* bbox;                 // (n) out of K0 / in of K1
  long long* cap;             // (n) out of K0
  const long long* offset;    // (n) exclusive scan of cap
  int32_t* count;             // (n) out
  double* points;             // (sum cap,3)
  double* lab;                // (sum cap,3)
  int32_t* src_px;            // (sum cap,2)
  int32_t* slot_map;          // (sum cap) out: compact index of every screen-box slot, -1 = empty
  // dense single-view output (px_rasterize)
  double* dense_z;
  double* dense_c;
  uint8_t* dense_valid;
  int32_t* dense_owner;
};

size_t render_smem_bytes(int V, int T);
cudaError_t launch_bbox(const RenderArgs& a, cudaStream_t st);
cudaError_t launch_render(const RenderArgs& a, size_t smem, bool dense, cudaStream_t st);
cudaError_t launch_scan(const long long* in, long long* out_excl, long long* total, int n, cudaStream_t st);
cudaError_t launch_fill_dense(double* z, double* c, uint8_t* valid, int32_t* owner, size_t npix, cudaStream_t st);

struct GicpCfgDev {
  int k_cov, max_iter;
  double eps, tol_t2, tol_r2, gate2;
};

// ragged cloud batch on the device: candidate c owns slots [offset[c], offset[c]+count[c])
struct CloudsDev {
  int n;
  const long long* offset;
  const int32_t* count;
  const double* points;
  const double* lab;
  const int32_t* src_px;
  const int32_t* slot_map;  // (sum cap) compact index per screen-box slot or -1; null for uploaded clouds
  const int4* bbox;         // (n) screen box (gu_lo, gv_lo, gw, gh); null for uploaded clouds
};

// Organised view of one target: its points are observed-cloud points, i.e. they
// sit on stride-grid pixels of the frame.  map[(gy-gy0)*w + (gx-gx0)] = local
// index or -1.  w == 0: not organised (generic cloud) -> linear scans.
// boxes: 3-D bounding boxes {lo xyz, hi xyz} of the points of every PX_BLK x
// PX_BLK block of map cells (bh x bw of them) followed by those of every PX_BLK x
// PX_BLK group of blocks (sh x sw).
#define PX_BLK 4
#define PX_GATE_MAX 1e3   // metres: larger gates are refused (PX_E_LIMIT) so that every fp32 pruning threshold stays finite
#define PX_FAR32 1e30f  // coordinate of an absent leaf point / bound of an empty box: every distance to it overflows to +inf
struct TgtOrg {
  int gx0, gy0, w, h;
  int bw, bh, sw, sh;
  long long map_off;
  long long box_off;  // first node of the target in boxes32 (units of 6 floats) / leaf32 (units of 48 floats)
  double err;         // bound on every fp32 rounding error of the pruning tests for this target (metres)
};

struct TargetsDev {
  int n_targets;
  const long long* offset;  // (n_targets+1)
  const double* points;     // (sum,3)
  const double* cov;        // (sum,9)
  const TgtOrg* org;        // (n_targets) or null
  const int32_t* tmap;
  const float* boxes32;       // per node {lo xyz, hi xyz}: fp32 3-D box, lo rounded down / hi rounded up (SoA per super-block)
  const float4* leaf32;       // per block slot (node numbering of boxes32): fp32 planes x[16], y[16], z[16] of the block's
                              //   4x4 map cells (row-major; PX_FAR32 where the cell holds no point) -- 12 float4 = 192 B
  const double* soa;          // 6 planes of `plane` doubles: x, y, z and the normal v0 the covariance I - f v0 v0^T is
  long long plane;            //   made of -- coherent-gather copy for the linearise kernel, which rebuilds the matrix
  double f;                   // 1 - epsilon the target covariances were built with
  // Frame of the fp32 pruning structures (boxes32, leaf32): x' = rot * x.  Axis-aligned boxes of a tilted plane are
  // fat (a 4x4-cell patch of a table seen at 60 degrees of incidence is 1.9 x 1.9 x 3.3 cm in the camera frame, and
  // its corners reach 1.6 cm off the plane); in a frame with the dominant plane axis-aligned they are thin, so their
  // distance to a query is close to the true distance and far fewer blocks / leaves are opened.  The rotation only
  // moves the conservative fp32 filter -- every surviving point is still evaluated in fp64 on the ORIGINAL
  // coordinates -- so results do not depend on it.  Identity unless the builder knows better (3-DoF: camera -> world).
  double rot[9];
};

// Device-side construction of GICP targets as subsets of the uploaded organised observed cloud
// (px_targets.cu; search.py:393-426).
struct TgtBuildArgs {
  int n_targets;
  int mode;                   // 0: capsule crops (3-DoF), 1: label sub-clouds (6-DoF)
  const double* params;       // mode 0: (n,5) cell x, cell y, z_lo, z_hi, radius (world frame)
  const int32_t* label_ids;   // mode 1: (n) object ids
  double c2w[12];             // camera -> world (mode 0)
  double gate;                // max_correspondence_distance (enters the fp32 pruning error bound)
  double frame[9];            // TargetsDev::rot: frame of the fp32 pruning structures
  Camera cam;                 // intrinsics + grid size (mode 0: screen window of a capsule)
  // scene
  const double* obs_pts;      // (n_obs,3) camera frame
  const int32_t* obs_labels;  // (n_obs)
  const int32_t* obs_cell;    // (n_obs) stride-grid cell gy*GW+gx of every observed point
  const int32_t* gidx;        // (GH*GW) observed index of every stride-grid cell or -1
  long long n_obs;
  int GW;
  double* world;              // scratch: 3 planes of n_obs (mode 0)
  // per-target sizes and their exclusive scans
  long long* cnt;             // (n)
  long long* cells;           // (n) w*h
  long long* nodes;           // (n) bw*bh + sw*sh
  const long long* offset;    // (n+1) scan of cnt      = TargetsDev::offset
  const long long* cells_off; // (n+1)
  const long long* nodes_off; // (n+1)
  // outputs (same layout as px_targets_upload produces on the host)
  TgtOrg* org;
  int32_t* tgt_obs;           // (sum) observed index of every target point
  double* tgt_pts;            // (sum,3)
  int32_t* tpix;              // (sum) map cell
  int32_t* tmap;              // (sum cells), -1 on entry
  float* boxes32;             // (sum nodes,6)
  float4* leaf32;             // (sum nodes,12)
};
cudaError_t launch_tgt_world(const TgtBuildArgs& a, cudaStream_t st);
cudaError_t launch_tgt_count(const TgtBuildArgs& a, cudaStream_t st);
cudaError_t launch_tgt_fill(const TgtBuildArgs& a, cudaStream_t st);  // offsets -> fill -> tree

struct CovArgs {  // covariances of a list of clouds (targets), thread per point
  int n_clouds;
  const long long* offset;  // (n_clouds+1) or per-cloud offsets with counts
  const int32_t* count;     // nullable: if null, count = offset[i+1]-offset[i]
  const double* points;
  double* cov;              // (sum,9)
  double* v0;               // (sum,3) nullable: the normal each covariance was made of
  int k;
  double eps;
  // organised targets (nullable): ring search instead of the linear scan
  const TgtOrg* org;
  const int32_t* tmap;
  const int32_t* tpix;      // (sum) map cell (y*w+x) of every target point
  double ray_k;
  Camera cam;               // ray_k is re-derived per target over its own grid window when cam.stride > 0
};
cudaError_t launch_cov(const CovArgs& a, long long total_points, cudaStream_t st);
// (n,3) points + (n,3) covariance normals -> 6 planes of n doubles (TargetsDev::soa)
cudaError_t launch_soa(const double* pts, const double* v0, double* soa, long long n, cudaStream_t st);

struct RefineArgs {
  CloudsDev src;
  TargetsDev tgt;
  const int32_t* target_idx;  // (n)
  const double* init_T;       // (n,12) or null = identity
  GicpCfgDev cfg;
  Camera cam;
  // scratch, indexed by the source slot offsets; structure-of-arrays with plane stride `plane`
  long long plane;            // >= sum cap
  double* src_soa;            // 6 planes: x, y, z and the covariance normal v0 of every source point
  double* w_buf;              // 10 planes, matched points compacted in index order: W = (Cb + R Ca R^T)^-1 (9), packed (source index | target index << 32)
  int32_t* nn;                // (sum cap) gated nearest neighbours of the current iteration (next iteration's search seeds)
  double* st_pose;            // (n,20) current iterate [R (9) | t (3)], step xi (6), f0, pad
  int32_t* st_i;              // (n,8) per-candidate integer state (px_gicp.cu: ST_*)
  double* st_hg;              // (n,44) normal equations of the current iteration: H (36), g (6), f0, pad
  // outputs
  double* out_T;              // (n,12) [orthonormalize(R)|t]
  int32_t* out_iters;
  int32_t* out_flags;         // low byte failure code, bit 8 converged
  double* out_resid;          // nullable: rms residual (registration.py:59-67)
  double* out_trace;          // nullable: (n, max_iter, 2) objective trace (f0, f_try)
  int32_t* out_ntrace;        // nullable: accepted steps per candidate
  int32_t* out_ncorr_sum;     // nullable: sum over iterations of the correspondence count (roofline accounting)
  // refine-apply (search.py:291-301); poses_in null => skip
  const double* poses_in;     // (n,12) candidate poses
  double* poses_out;          // (n,12) refined candidate poses
  int mode3dof;
  double c2w[12], w2c[12];
  int c2w_vec_order, w2c_vec_order;
  double fixed_z;
};
// Launch order: init, (nn, lin + solve, halve) x max_iter, finish.  `marks` (nullable) receives one event
// before every launch and one after the last: 3 + 3 * max_iter events.
cudaError_t launch_refine(const RefineArgs& a, cudaStream_t st, int* launches, cudaEvent_t* marks = nullptr);
// init + the nearest-neighbour and linearise kernels of iteration 1 only (px_gicp_linearize, a test export)
cudaError_t launch_linearize_once(const RefineArgs& a, cudaStream_t st);

struct CostArgs {
  CloudsDev ren;
  Camera cam;
  const ModelDev* models;
  const int32_t* model_slot;   // (n)
  const double* cyl_poses;     // (n,12) or null -> label mode
  // organised observed cloud
  const double* gx;            // (GH*GW) NaN where no point
  const double* gy;
  const double* gz;
  const int32_t* gidx;         // (GH*GW) observed index or -1
  const double* obs_lab;       // (n_obs,3)
  const int32_t* obs_labels;   // (n_obs)
  const int32_t* label_count;  // per model slot: count(obs_labels == oid)
  double delta, delta2, tau_c;
  int use_color;
  int lab_is_linear;           // ren.lab holds linear-light colours (RenderArgs::skip_lab == 2): convert matched points only
  uint32_t* bitmap;            // scratch: (#warp slots) x bitmap_words, zero on entry and exit
  int bitmap_words;
  int bitmap_slots;            // number of warp slots the bitmap scratch holds (multiple of PX_COST_WARPS)
  int32_t* j_o;                // (n) out
  int32_t* j_r;                // (n) out
  int32_t* n_match;            // (n) out, nullable: rendered points with an observed neighbour within delta (SURVEY 8(d) n_m)
  int32_t* n_foot;             // (n) out, nullable: observed points selected for the candidate (n_fp)
  unsigned long long* knife;   // nullable: [0] min |d2 - delta^2| over all gated neighbours, [1] min |dE - tau_c| (double bits)
  // fused argmin (search.py:178-183): key = total<<32 | rank
  const int32_t* rank;         // (n) rank of the candidate inside its object, nullable
  unsigned long long* best_key;  // per model slot, nullable
};
cudaError_t launch_cost(const CostArgs& a, cudaStream_t st);

// Per-object winner records after the (all-reduced) argmin keys are known (search.py:346-372): the candidate whose
// packed key equals best_key[slot] writes its record; every other record stays zero, so an all-reduce(MAX) over the
// raw 64-bit words across ranks delivers the owner's bits unchanged.
#define PX_WIN_WORDS 28  // key + 1 | refined pose (12) | applied correction (12) | j_o | j_r | max points in the final render
struct WinnerArgs {
  int n;
  const int32_t* model_slot;          // (n)
  const int32_t* rank;                // (n) rank in object
  const int32_t* j_o;
  const int32_t* j_r;
  const int32_t* n_final;             // (n) points in the final render
  const double* refined;              // (n,12)
  const double* reg_T;                // (n,12)
  const unsigned long long* best_key; // per model slot (global after the reduction)
  unsigned long long* win;            // (n_models, PX_WIN_WORDS), zero on entry
};
cudaError_t launch_winners(const WinnerArgs& a, cudaStream_t st);

// raster.frame_to_cloud + cloud_labels on the device (px_scene.cu)
struct SceneCloudArgs {
  int H, W, stride, GW, GH;
  double fx, fy, cx, cy;
  const double* depth;        // (GH,GW) stride-grid samples of the frame planes
  const uint8_t* valid;       // (GH,GW)
  const int32_t* labels;      // (GH,GW)
  const double* color_grid;   // (GH,GW,3) sRGB of the stride-grid pixels
  long long* row_count;       // (GH) out of the count pass
  const long long* row_offset;  // (GH) exclusive scan
  double* pts;                // (n,3)
  double* lab;                // (n,3)
  int32_t* src;               // (n,2) (u,v)
  int32_t* labels_out;        // (n)
  int32_t* cell;              // (n)
  double *gx, *gy, *gz;       // (GH*GW), NaN where no point
  int32_t* gidx;              // (GH*GW), -1 where no point
};
cudaError_t launch_scene_count(const SceneCloudArgs& a, cudaStream_t st);
cudaError_t launch_scene_fill(const SceneCloudArgs& a, cudaStream_t st);
cudaError_t launch_label_count(const int32_t* labels, long long n, const ModelDev* models, int n_models, int32_t* out,
                               cudaStream_t st);

// candidate lattice of one search, generated on the device (px_scene.cu)
struct LatticeObjDev {
  int slot;               // model slot
  int n_outer, n_inner;   // 3-DoF: cells x yaws; 6-DoF: rotations x translations
  int n_outer_local;      // outer items owned by this rank
  long long cand_off;     // first local candidate of the object
  long long rot_off, tr_off;  // into LatticeArgs::rotations (units of 9) / translations (units of 3)
  int tgt_off;            // 3-DoF: first local GICP target of the object; 6-DoF: the object's target
  int pad_;
  double z_lo, z_hi, radius;  // 3-DoF capsule of the per-cell target
};
struct LatticeArgs {
  int mode3dof, n_objects, rank, world;
  long long n_local;
  const LatticeObjDev* objs;
  const double* rotations;
  const double* translations;
  double w2c[12];
  int w2c_vec_order;
  int32_t* slot;            // (n_local) out
  double* poses;            // (n_local,12) out
  int32_t* rank_in_object;  // (n_local) out
  int32_t* tidx;            // (n_local) out, nullable
  double* capsules;         // (n_targets,5) out, nullable
};
cudaError_t launch_lattice(const LatticeArgs& a, cudaStream_t st);

cudaError_t launch_ciede(const double* lab_a, const double* lab_b, double* out, long long n, cudaStream_t st);
cudaError_t launch_lab(const double* rgb, double* out, long long n, int encode_first, cudaStream_t st);

struct KnnArgs {  // exact brute-force kNN, k <= PX_KCOV_MAX (neighbors.py:104-134)
  const double* q;
  long long nq;
  const double* t;
  long long nt;
  int k;
  long long* idx;  // (nq,k)
  double* d2;      // (nq,k)
};
cudaError_t launch_knn(const KnnArgs& a, cudaStream_t st);

struct GenericCostArgs {  // cost.py:91-135 on arbitrary (non-organised) clouds
  const double* rp;
  const double* rlab;
  int n_r;
  const double* op;
  const double* olab;
  long long n_obs;
  double delta2, tau_c;
  int use_color;
  uint8_t* explained;  // (n_obs) zeroed by the caller
  int32_t* j_r;        // single int, zeroed by the caller -> counts outliers
};
cudaError_t launch_generic_cost(const GenericCostArgs& a, cudaStream_t st);

}  // namespace px
