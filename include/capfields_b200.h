/*
 * capfields_b200 — C-ABI of the B200-native Instant-NVR render back-end hot path.
 *
 * Every entry point takes plain device pointers + sizes and a caller-supplied
 * stream (`void* stream` = cudaStream_t, NULL = legacy default stream). All calls
 * are stream-ordered and asynchronous unless stated; none allocate on the hot
 * call (handles own their storage, sized at create time). No torch types.
 *
 * Status codes map 1:1 onto the reference's exception classes (the Python shim
 * re-raises them):
 *   CF_E_OUT_OF_SUPPORT  -> capfields.edgraph.OutOfSupportError   (edgraph.py:27)
 *   CF_E_DUPLICATE_FRAME -> ValueError "frame already registered"  (knnfield.py:132-133)
 *   CF_E_BAD_ARG         -> ValueError                             (knnfield.py:56-57,134-135)
 *   CF_E_DEGENERATE      -> capfields.transforms.DegenerateWeightsError (transforms.py:15)
 *   CF_E_CUDA            -> RuntimeError (device fault / launch failure)
 *   CF_E_FORMAT          -> capfields.records.RecordFormatError      (records.py:24)
 * cf_last_error() returns a thread-local message for the last non-zero status.
 *
 * Reference interfaces replaced (the reference has no FFI; these are the Python
 * functions whose bodies the calls stand in for — see INTEGRATION.md):
 *   cf_deform_nodes            <- edgraph.deformed_nodes            edgraph.py:134-136
 *   cf_dq_blend / cf_dq_status <- transforms.dq_blend                transforms.py:180-196
 *   cf_dq_apply                <- transforms.dq_apply                transforms.py:174-177
 *   cf_knn_warp                <- edgraph.warp_backward_batch       edgraph.py:174-183
 *                                 edgraph.warp_forward_batch        edgraph.py:154-162
 *                                 knnfield.brute_force_query        knnfield.py:32-42
 *                                 knnfield.brute_force_neighbors_batch knnfield.py:25-29
 *   cf_knnfield_build          <- KnnField._build_canonical_field   knnfield.py:93-120
 *   cf_knnfield_update         <- KnnField.update_live_map          knnfield.py:124-167
 *                                 KnnField._dilate_once             knnfield.py:169-188
 *   cf_knnfield_query          <- KnnField.query_motion_batch       knnfield.py:197-222
 *   cf_lbs_forward             <- skeleton.lbs_batch                skeleton.py:142-149
 *   cf_lbs_backward            <- (builder-defined inverse of lbs_batch)
 *   cf_hashgrid_encode(_bwd)   <- SPEC nrf.hash_encode
 *   cf_field_forward           <- SPEC nrf E_g/E_c/DeformNet
 *   cf_render_*                <- SPEC nrf.volume_render/render_view SPEC.md:381-407
 */
#ifndef CAPFIELDS_B200_H
#define CAPFIELDS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CF_OK 0
#define CF_E_BAD_ARG 1
#define CF_E_OUT_OF_SUPPORT 2
#define CF_E_DUPLICATE_FRAME 3
#define CF_E_DEGENERATE 4
#define CF_E_CUDA 5
#define CF_E_FORMAT 6

int cf_version(void);
const char* cf_last_error(void);
/* number of SMs of the current device (grid sizing helper for hosts) */
int cf_device_sm_count(void);
/* self-test of the shared-denominator division used by the warp kernels:
 * n random (a, b) pairs (seeded; log-uniform magnitudes incl. adversarial
 * significands) divided both ways on the device; *mismatches = number of
 * results not bit-equal to IEEE a / b. Synchronous. */
int cf_selftest_exact_div(int64_t n, uint64_t seed, int64_t* mismatches);

/* ---------------------------------------------------------------- deformation */

/* anchors[i] = dq_apply(dqs[i], nodes[i]) in float64, bit-identical to the
 * reference's numpy evaluation order (edgraph.py:134-136). */
int cf_deform_nodes(const double* nodes, const double* dqs, int64_t n, double* anchors, void* stream);
/* dq_blend drop-in (transforms.py:180-196): n rows of k (weight, dq) pairs -> (n, 8) unit dual
 * quaternions, bit-exact with the reference's numpy evaluation order; *err (device int, zeroed
 * by the caller, optional) receives 2 for a negative weight, 1 for a row summing to <= 0 */
int cf_dq_blend(const double* weights, const double* dqs, int64_t n, int k, double* out, int* err, void* stream);
/* synchronises the stream and maps cf_dq_blend's *err to a status: CF_E_BAD_ARG (ValueError,
 * negative weights), CF_E_DEGENERATE (DegenerateWeightsError, zero weights) or CF_OK */
int cf_dq_status(const int* err, void* stream);
/* dq_apply drop-in (transforms.py:174-177): row i = dq[i * dq_stride] applied to p[i * p_stride]
 * (a stride of 0 broadcasts one dq / one point) */
int cf_dq_apply(const double* dq, int64_t dq_stride, const double* p, int64_t p_stride, int64_t n, double* out,
                void* stream);
/* graphs of n <= 1024 nodes: the deformed nodes plus the frame's anchor block read by
 * cf_human_canon (float64 + fp32 copies, bbox; cf_anchor_block_bytes(n) bytes, 16-byte aligned) */
int cf_anchor_block_bytes(int64_t n, int64_t* bytes);
/* candidate grid of a frame's anchors (n <= 1024), hierarchical k-NN: grid_res cells along the
 * longest side of the anchors' bbox grown by the ED support radius sqrt(-ln 1e-6) radius; per cell
 * the nodes that can be among the k nearest of any point in it (float64, ties included), up to
 * cmax ids (fuller cells fall back to every node). Reads the anchor block (cf_deform_nodes_block). */
int cf_cand_grid_bytes(int grid_res, int cmax, int64_t* bytes);
int cf_cand_grid_build(const void* block, int64_t n, int k, double radius, int grid_res, int cmax, void* cand,
                       void* stream);
int cf_deform_nodes_block(const double* nodes, const double* dqs, int64_t n, double* anchors, void* block,
                          void* stream);

/* Coarse voxel buckets over a point set (ED anchors or posed skin vertices):
 * counting sort of point ids into a uniform grid, rebuilt per frame into
 * storage sized at create time. */
typedef struct cf_buckets cf_buckets_t;
int cf_buckets_create(int64_t max_points, int max_grid_res, cf_buckets_t** out);
int cf_buckets_destroy(cf_buckets_t* b);
/* stream-ordered destroy: the buffers are freed after the work queued on `stream`, no host sync */
int cf_buckets_destroy_async(cf_buckets_t* b, void* stream);
/* grid_res <= 0 picks a resolution from n (~4 points per occupied cell). */
int cf_buckets_build(cf_buckets_t* b, const double* pts, int64_t n, int grid_res, void* stream);
/* Optional second level, after cf_buckets_build: per cell, the exact candidate
 * list of points that can be among the k nearest of any query in the cell
 * (radius d_k(centre) + 2 half-diagonals). cf_knn_warp then scans one list per
 * query (ring search only outside the grid box); results stay bit-identical. */
int cf_buckets_build_candidates(cf_buckets_t* b, int k, void* stream);

/* Exact k-NN (ties by index, squared distance evaluated as the reference's
 * sum((p - a)**2)) over `anchors` followed by the dual-quaternion blend.
 *   mode CF_WARP_BACKWARD  : warp_backward_batch  (safe_w = valid ? w : 1, DQB^-1 applied)
 *   mode CF_WARP_FORWARD   : warp_forward_batch   (safe_w = valid ? w : 1, DQB applied)
 *   mode CF_BRUTE_QUERY    : brute_force_query    (max(w,1e-300), DQB^-1 applied)
 *   mode CF_NEIGHBORS_ONLY : brute_force_neighbors_batch (idx only)
 * `buckets` NULL -> exhaustive scan (trivially-correct brute-force kernel);
 * otherwise the hierarchical bucket ring search (bit-identical results).
 * Any of idx_out (int64, N*k), w_out (N*k), pc_out (N*3), valid_out (N) may be NULL. */
#define CF_WARP_BACKWARD 0
#define CF_WARP_FORWARD 1
#define CF_BRUTE_QUERY 2
#define CF_NEIGHBORS_ONLY 3
int cf_knn_warp(const cf_buckets_t* buckets, const double* anchors, const double* dqs, int64_t n_nodes,
                int k, double radius, int mode, const double* pts, int64_t n_pts,
                int64_t* idx_out, double* w_out, double* pc_out, uint8_t* valid_out, void* stream);
/* Hierarchical exact k-NN warp for graphs of up to 8192 nodes (k <= 8): queries
 * are visited in `order` (optional permutation, e.g. by Morton code of the query
 * position, so that each warp's 32 queries are neighbours); each warp culls the
 * nodes against its queries' box and ranks survivors fp32-first, float64-exact.
 * Same outputs and modes as cf_knn_warp, bit-identical indices. */
int cf_knn_warp_cull(const double* anchors, const double* dqs, int64_t n_nodes, int k, double radius, int mode,
                     const double* pts, const int* order, int64_t n_pts, int64_t* idx_out, double* w_out,
                     double* pc_out, uint8_t* valid_out, void* stream);

/* ------------------------------------------------------------------ KnnField */

/* neighbor_idx (res^3, s) int32, -1 outside support (knnfield.py:93-120). */
int cf_knnfield_build(const double* nodes, int64_t n, int s, int res, const double* bbox_min,
                      double voxel_size, double support_radius, int32_t* neighbor_idx, void* stream);
/* live map of one frame (knnfield.py:124-188). scratch_u64: res^3 uint64;
 * scratch_i32: res^3 int32 (pre-dilation map). */
int cf_knnfield_update(const double* nodes, const double* dqs, int64_t n, const int32_t* neighbor_idx, int s,
                       int res, const double* bbox_min, double voxel_size, double radius, int32_t* live_out,
                       uint64_t* scratch_u64, int32_t* scratch_i32, void* stream);
/* O(1) query (knnfield.py:197-222): anchors_frame = deformed nodes of the frame,
 * dqs_frame = the frame's LUT block. nbr_out int64 (N,s). */
int cf_knnfield_query(const int32_t* live, const int32_t* neighbor_idx, const double* dqs_frame,
                      const double* anchors_frame, int s, int res, const double* bbox_min, double voxel_size,
                      double radius, const double* pts, int64_t n_pts, int64_t* nbr_out, double* w_out,
                      double* pc_out, uint8_t* valid_out, void* stream);
/* Sparse live maps (a frame's map is mostly empty space: 512 MiB dense per frame at
 * 512^3): bricks of 8^3 voxels. brick_index: B^3 int32 (B = ceil(res / 8), brick
 * (bi, bj, bk) at (bi*B + bj)*B + bk) = the brick's block in `bricks` (512 int32, voxel
 * (x, y, z) of the brick at (x*8 + y)*8 + z) or -1 if all its voxels are empty.
 * cf_knnfield_brick_count: B^3. cf_knnfield_brick_index: brick_index and the number of
 * set bricks (device int32) from a dense map; cf_knnfield_brick_pack: the set bricks;
 * cf_knnfield_brick_unpack: back to the dense map. cf_knnfield_query_sparse: the
 * query of cf_knnfield_query on a sparse map (same results). */
int cf_knnfield_brick_count(int res, int64_t* n_bricks_total);
int cf_knnfield_brick_index(const int32_t* live_dense, int res, int32_t* brick_index, int32_t* n_set, void* stream);
int cf_knnfield_brick_pack(const int32_t* live_dense, int res, const int32_t* brick_index, int32_t* bricks,
                           void* stream);
int cf_knnfield_brick_unpack(const int32_t* brick_index, const int32_t* bricks, int res, int32_t* live_dense,
                             void* stream);
int cf_knnfield_query_sparse(const int32_t* brick_index, const int32_t* bricks, const int32_t* neighbor_idx,
                             const double* dqs_frame, const double* anchors_frame, int s, int res,
                             const double* bbox_min, double voxel_size, double radius, const double* pts,
                             int64_t n_pts, int64_t* nbr_out, double* w_out, double* pc_out, uint8_t* valid_out,
                             void* stream);

/* ------------------------------------------------------------------ skeleton */

/* forward LBS (skeleton.py:142-149): A (J,4,4) float64, weights (N,J). */
int cf_lbs_forward(const double* A, int J, const double* pts, const double* weights, int64_t n_pts, double* out,
                   void* stream);
/* pose Jacobian of forward LBS by central differences (tracking.py:244-256): A_pm
 * (2T, J, 4, 4) = bone transforms at theta +/- fd_step e_k (k-major, + first);
 * out (n, 3, T) = (LBS(A+) - LBS(A-)) / (2 fd_step) */
int cf_lbs_theta_jacobian(const double* A_pm, int n_theta, int J, const double* pts, const double* weights,
                          int64_t n_pts, double fd_step, double* out, void* stream);
/* per-frame vertex transforms for the backward warp: T_v = sum_j W[v,j] A_j[:3,:],
 * Tinv_v its inverse, both (V,3,4) row-major; T_out may be NULL. */
int cf_lbs_vertex_transforms(const double* A, int J, const double* vert_weights, int64_t n_verts, double* T_out,
                             double* Tinv_out, void* stream);
/* per-frame skin setup in one kernel: cf_lbs_vertex_transforms (T, Tinv) plus
 * the posed vertices of cf_lbs_forward with the same weights (J <= 64); posed_box
 * (6 x uint64, may be NULL) receives the posed vertices' bounding box in the
 * order-preserving key form cf_human_lbs_fallback reads */
int cf_lbs_setup(const double* A, int J, const double* verts, const double* vert_weights, int64_t n_verts,
                 double* T_out, double* Tinv_out, double* posed_out, uint64_t* posed_box, void* stream);
/* backward LBS (builder-defined): nearest posed skin vertex
 * v* (exact 1-NN, ties by index; vert_buckets built over verts_posed, or NULL
 * for an exhaustive scan) -> p_c = Tinv_{v*} [p, 1];
 * valid = |p - v*|^2 <= max_dist^2. */
int cf_lbs_backward(const cf_buckets_t* vert_buckets, const double* verts_posed, const double* vert_Tinv,
                    int64_t n_verts, double max_dist, const double* pts, int64_t n_pts, int64_t* vert_out,
                    double* pc_out, uint8_t* valid_out, void* stream);

/* ------------------------------------------------------------------ hash grid */

#define CF_MAX_LEVELS 16
typedef struct cf_hashgrid_desc {
  int n_levels;       /* L */
  int n_features;     /* F (2 or 4) */
  int log2_table;     /* log2 T */
  int base_resolution;
  int max_resolution;
  int resolution[CF_MAX_LEVELS]; /* N_l */
  int dense[CF_MAX_LEVELS];      /* 1: dense (N_l+1)^3 indexing */
  int64_t offset[CF_MAX_LEVELS + 1]; /* entry offsets of each level, offset[L] = total entries */
} cf_hashgrid_desc;

/* fill desc from (L, F, log2T, N_min, N_max) */
int cf_hashgrid_init(cf_hashgrid_desc* desc, int n_levels, int n_features, int log2_table, int base_res,
                     int max_res);
/* pts (N,3) float32 in [0,1]^3 (clamped); table (entries, F) float32;
 * feat_out (N, L*F) float32. */
int cf_hashgrid_encode(const cf_hashgrid_desc* desc, const float* table, const float* pts, int64_t n_pts,
                       float* feat_out, void* stream);
/* table_grad += dL/dtable, atomics (dfeat (N, L*F)). */
int cf_hashgrid_encode_bwd(const cf_hashgrid_desc* desc, const float* pts, const float* dfeat, int64_t n_pts,
                           float* table_grad, void* stream);
/* parity probe: idx_out (N, L, 8) uint32 entry indices within each level,
 * w_out (N, L, 8) float32 trilinear weights. */
int cf_hashgrid_indices(const cf_hashgrid_desc* desc, const float* pts, int64_t n_pts, uint32_t* idx_out,
                        float* w_out, void* stream);

/* ------------------------------------------------------------------ tiny MLPs */

/* Fused MLP chain on tcgen05 (fp16 operands, fp32 TMEM accumulation):
 * y = L_n(relu(...relu(L_1(x)))). widths[0..n_layers]; layer l weight is the
 * (N_l x K_l) fp16 matrix (K_l, N_l = widths padded to 16, <= 128) packed in the
 * UMMA canonical K-major layout, concatenated into wblob;
 * bias (n_layers x 128) fp32, row l used where has_bias[l] (host array).
 * x (N, widths[0]) fp32, y (N, widths[n_layers]) fp32. */
int cf_mlp_forward(int n_layers, const int* widths, const uint8_t* wblob, int w_bytes, const float* bias,
                   const int* has_bias, const float* x, int64_t n_rows, float* y, void* stream);

/* ------------------------------------------------------------------ render path */

/* pinhole camera, CV axes (camera.py:94-108): R camera-to-world row-major */
typedef struct cf_camera {
  double R[9];
  double fx, fy, cx, cy;
  int width, height;
  const double* params; /* optional device double[13] = R[9], fx, fy, cx, cy read by the kernel
                           instead of the fields above (a captured CUDA graph replays with new
                           cameras by rewriting this block); NULL = use the fields */
  int row0, row_stride; /* row shard: local row j is image row row0 + j * row_stride (height =
                           local rows; row_stride <= 0 means 1). Multi-GPU renders deal the rows
                           of one frame round-robin; the directions equal the full frame's. */
} cf_camera;

/* cubic occupancy bit grid: res^3 cells of edge `cell` from `min`, x-major
 * flat index (i*res + j)*res + k, 32 cells per uint32 word */
typedef struct cf_occ_grid {
  double min[3];
  double cell;
  int res;
} cf_occ_grid;

/* uniform march of n_samples per ray over [t_near, t_far]: t_i = t_near + (i+0.5) dt */
typedef struct cf_march_desc {
  double origin[3];
  int64_t n_rays;
  int n_samples;
  double t_near, t_far, dt;
  cf_occ_grid human_grid;   /* live-space occupancy of the human field */
  cf_occ_grid object_grid;  /* object-local occupancy of the rigid object */
  double obj_R[9], obj_t[3]; /* object pose (object-to-world) */
  double obj_min[3], obj_inv_side; /* object unit-cube normalisation */
  const int* human_cell_bbox;      /* device int[6] (lo xyz, hi xyz) of set live cells, or NULL */
  const double* sample_t;          /* training: explicit depth of compacted sample s (NULL = uniform t_i);
                                      delta_s = t_{s+1} - t_s within a ray, dt for its last sample */
  const double* frame;             /* optional device double[15] = origin[3], obj_R[9], obj_t[3] read by
                                      the kernels instead of the fields (graph-replayable frames);
                                      NULL = use the fields */
} cf_march_desc;

/* compacted samples of one field: records (capacity) = ray << 8 | i, grouped
 * per ray in ascending i; counters: int[4] — [0] = total emitted, [1] = overflow
 * flag, [2..3] = work ticket of the per-sample kernels (zeroed by the producer,
 * re-armed by each consumer launch) */
typedef struct cf_march_out {
  uint32_t* records;
  int* ray_offset;
  int* ray_count;
  int* counters;
  int64_t capacity;
} cf_march_out;

/* per-frame human warp state (hybrid deformation) */
typedef struct cf_human_warp {
  const double* dqs;        /* (n,8) node motion of the frame */
  int k;                    /* ED neighbours */
  double r2;                /* ED radius^2 */
  const double* vert_Tinv;  /* (V,12) inverse blended bone transforms, NULL = no LBS fallback */
  double lbs_max_d2;
  double canon_min[3];      /* canonical unit-cube normalisation */
  double inv_side;
  const double* anchors;    /* (n,3) deformed nodes of the frame */
  int n_nodes;
  const void* anchor_block; /* n_nodes <= 1024: the frame's anchor block (cf_deform_nodes_block), which the
                               k-NN scans with warp-cooperative culling (anchor_buckets may be NULL) */
  const void* cand_grid;    /* optional, with anchor_block: the frame's candidate grid (cf_cand_grid_build);
                               each sample then ranks only its cell's candidate nodes */
} cf_human_warp;

int cf_camera_rays(const cf_camera* cam, double* dirs, void* stream);
/* occupancy from geometry: cells whose centre is within radius of a bucketed point */
int cf_occ_from_points(const cf_buckets_t* pts, const cf_occ_grid* g, double radius, uint32_t* bits, void* stream);
/* occupancy of a solid origin-centred box dilated by shell: sdf(centre) <= shell */
int cf_occ_box_shell(const cf_occ_grid* g, const double* half_extents, double shell, uint32_t* bits, void* stream);
/* per-frame live occupancy: forward ED warp of every occupied canonical cell
 * centre (node_buckets over the CANONICAL nodes), 3x3x3 live cells set */
int cf_occ_splat(const uint32_t* canon_bits, const cf_occ_grid* cg, const cf_buckets_t* node_buckets,
                 const double* dqs, int k, double radius, const cf_occ_grid* lg, uint32_t* live_bits, void* stream);
/* once per sequence: the static part of the splat — every occupied canonical
 * cell whose forward warp is valid, with its exact canonical k-NN (ties by
 * index) and Gaussian weights (edgraph.canonical_blend_info, edgraph.py:186-195).
 * cells (cap), nbr (cap*k), w (cap*k); count = cells written (device int). */
int cf_occ_cache(const uint32_t* canon_bits, const cf_occ_grid* cg, const cf_buckets_t* node_buckets, int k,
                 double radius, int64_t capacity, int* cells, int* nbr, double* w, int* count, void* stream);
/* per frame, same live bits as cf_occ_splat from the cache: blend + apply the
 * frame's dqs, set the centre cells in a 1-padded scratch grid
 * ((res+2)^3/32 + 3 words), then a word-parallel 3x3x3 dilation; live_bbox (int[6],
 * may be NULL) receives the cell bbox of the live set as cf_occ_bbox would */
int cf_occ_splat_cached(const int* cells, const int* nbr, const double* w, const int* count, int64_t capacity, int k,
                        const double* dqs, const cf_occ_grid* cg, const cf_occ_grid* lg, uint32_t* scratch_bits,
                        uint32_t* live_bits, int* live_bbox, void* stream);
/* bounding box (cell coords, int[6] lo xyz, hi xyz; lo > hi if empty) of the set cells */
int cf_occ_bbox(const uint32_t* bits, const cf_occ_grid* g, int* bbox, void* stream);
/* occupancy-skipped compaction of the samples of every ray (one or two fields);
 * each ray only tests the samples inside its entry/exit interval of the
 * occupied box (the live cell bbox, the object grid box), with a one-sample
 * margin, so decisions equal a test of every sample */
int cf_march(const cf_march_desc* M, const double* dirs, const uint32_t* human_bits, const uint32_t* object_bits,
             const cf_march_out* human, const cf_march_out* object, void* stream);
/* cf_camera_rays + cf_march in one kernel: each ray's direction is generated
 * (and written to dirs) by the thread that marches it; n_rays = width * height */
int cf_rays_march(const cf_camera* cam, const cf_march_desc* M, double* dirs, const uint32_t* human_bits,
                  const uint32_t* object_bits, const cf_march_out* human, const cf_march_out* object, void* stream);
/* human samples -> canonical unit cube (xu: float4 x,y,z,flag; flag 1 = ED, 2 = LBS, 0 = invalid) */
int cf_human_canon(const cf_march_desc* M, const double* dirs, const cf_march_out* F, const cf_human_warp* W,
                   const cf_buckets_t* anchor_buckets, const cf_buckets_t* vert_buckets, float* xu, void* stream);
/* the backward-LBS fallback of cf_human_canon as a separate pass: with vert_buckets = NULL
 * cf_human_canon leaves the samples no ED warp reaches at flag 0; this pass gives them
 * their LBS canonical position (flag 2) — output identical to the fused call. It needs
 * no vertex buckets: a warp scans the posed vertices (verts_posed, n_verts) for each
 * flag-0 sample within lbs_max_dist of their box (posed_box of cf_lbs_setup); exact
 * 1-NN with ties by index, as the bucket search. The render runs the canonicalisation
 * as soon as the march and the ED chain are done and this pass after the LBS setup. */
int cf_human_lbs_fallback(const cf_march_desc* M, const double* dirs, const cf_march_out* F, const cf_human_warp* W,
                          const double* verts_posed, int64_t n_verts, const uint64_t* posed_box, float* xu,
                          void* stream);
int cf_object_canon(const cf_march_desc* M, const double* dirs, const cf_march_out* F, float* xu, void* stream);
/* front-to-back compositing of field outputs (float4 sigma,r,g,b per sample) */
int cf_composite(const cf_march_desc* M, const cf_march_out* F, const float* field, float t_term, float* rgb,
                 float* depth, float* opacity, void* stream);
/* per pixel: nearer layer among those with opacity > 0.5, else background; layer 0 bg, 1 human, 2 object */
int cf_composite_layers(int64_t n, const float* h_rgb, const float* h_depth, const float* h_opac, const float* o_rgb,
                        const float* o_depth, const float* o_opac, const float* bg, float* out, uint8_t* layer,
                        void* stream);
/* cf_composite of the human field fused with cf_composite_layers against an
 * already composited object layer (o_* may be NULL: no object) */
int cf_composite_final(const cf_march_desc* M, const cf_march_out* F, const float* field, float t_term, float* rgb,
                       float* depth, float* opacity, const float* o_rgb, const float* o_depth, const float* o_opac,
                       const float* bg, float* out, uint8_t* layer, void* stream);

/* fused radiance field of one field: hash grids + MLPs on tcgen05.
 * wblob = fp16 canonical-layout weights, in order
 *   [has_deform: D1 128x32, D2..D4 128x128, D5 16x128] G1 64x32, G2 16x64, C1 64x32, C2 64x64, C3 16x64 */
typedef struct cf_field_desc {
  int has_deform;
  cf_hashgrid_desc dgrid;   /* deformation grid (L*F = 32, F = 4) */
  const void* dtable;       /* fp16 (entries, F): the fp16 copy of the fp32 parameters */
  cf_hashgrid_desc cgrid;   /* canonical grid (L*F = 32, F = 2) */
  const void* ctable;       /* fp32 (entries, F) */
  const uint8_t* wblob;
  int w_bytes;
  const float* dbias;       /* DeformNet layer-1 bias (128), pose theta folded in */
  float delta_scale;        /* |dv| bound, metres (0.05) */
  float inv_side;           /* metres -> unit cube */
  void* save_h;             /* training: DeformNet hidden activations h1..h4, feature-major (512, S) fp16
                               (row = layer * 128 + unit, S = capacity), or NULL */
  float* save_o;            /* training: DeformNet raw outputs (o0, o1, o2, 0) float4 per sample, or NULL */
  uint32_t* save_mask;      /* training: ReLU bits of layers 1..4, (S,16) uint32 = [layer][half][2], or NULL */
  int precise;              /* 1 = "fp32" mode: fp32 tables and features, split-fp16 (hi + lo) MLP operands
                               (3 MMA chains per layer); 0 = "fp16" mode (fp16 operands, fp16 deform-table copy) */
  const uint8_t* wblob_lo;  /* precise: the residual blob fp16(W - fp16(W)), same layout as wblob */
  int train;                /* 1 = the training forward: 32-bit semantics (as precise) plus the fp16 saves of
                               the backward, feature-major in the scratch (cf_field_train_layout) */
  int split_stages;         /* precise render: 0 = the hash lookups run inside the MLP kernels (the deformation
                               grid in DeformNet, the canonical grid in E_g / E_c: stages 0 and 2 are empty);
                               1 = separate hash kernels, features in the scratch (stage-by-stage inspection) */
  int max_ctas;             /* precise render: cap on the persistent E_g / E_c kernel's CTAs (0 = one per SM);
                               a field rendered on a side stream beside another leaves it the other SMs */
} cf_field_desc;
/* occupancy from the trained density (the builder's K12; SPEC.md:429 leaves ray-marching
 * acceleration open): per cell of a res^3 grid over the field's unit cube, the E_g density
 * logit g0 at the centre u = (i + 0.5) / res, exact fp32 (hash features as cf_hash_encode,
 * W1 (64 x 32) / W2 (16 x 64, row 0) fp32 master weights, un-contracted sequential sums);
 * logits (res^3, init -inf) = max(logits + log_decay, g0); bits = (logits > log_threshold)
 * dilated by `dilate` cells per axis (Chebyshev; the DeformNet offset bound for the human).
 * x-major cells ((x * res + y) * res + z), 32 z-cells per word; res % 32 == 0; scratch = res^3/32 words */
int cf_density_grid_update(const cf_hashgrid_desc* G, const float* table, const float* W1, const float* W2, int res,
                           float log_decay, float log_threshold, int dilate, float* logits, uint32_t* bits,
                           uint32_t* scratch, void* stream);
/* device scratch needed by cf_field_forward for `capacity` samples */
int cf_field_scratch_bytes(const cf_field_desc* F, int64_t capacity, int64_t* bytes);
/* scratch layout (S = capacity): fp16 mode: cfeat (S,32) fp16 | dfeat (S,32) fp16 | xc (S) float4;
 * precise mode: cfeat (S,32) fp32 | dfeat (S,32) fp32 | xc (S) float4 (dfeat / xc human only);
 * training (train = 1, S % 8 == 0): byte offsets from cf_field_train_layout:
 * [0] cfeat16 (32,S) fp16 feature-major, [1] dfeat16 (33,S) fp16 feature-major with row 32 = 1,
 * [2] xc (S) float4, [3] dfeat32 (S,32) fp32, [4] cfeat32 (S,32) fp32, [5] total bytes */
int cf_field_train_layout(int64_t capacity, int64_t* offsets);
/* out: float4 (sigma, r, g, b) per compacted sample of S (count read on device).
 * Stages: hash (fp16 features) [-> DeformNet -> hash] -> E_g/E_c, see field.cu */
int cf_field_forward(const cf_field_desc* F, const cf_march_out* S, const double* dirs, const float* xu, float* out,
                     void* scratch, void* stream);
/* one stage of cf_field_forward (so hosts can time / overlap them):
 * 0 deform-grid hash, 1 DeformNet, 2 canonical-grid hash, 3 E_g/E_c (0-1 human only) */
int cf_field_stage(const cf_field_desc* F, const cf_march_out* S, const double* dirs, const float* xu, float* out,
                   void* scratch, int stage, void* stream);

/* ------------------------------------------------------------------ training (SPEC train_step) */

/* valid-sample compaction (training): C gets the samples of F whose flag (xu.w) > 0 —
 * records and xu, in C->records / xu_c, count in C->counters[0] (reset here) — with
 * vidx[j] = the full index of compacted sample j and inv[s] = the compacted index of
 * sample s or -1. The field forward / backward then run on C; cf_scatter_rows puts
 * their per-sample outputs (float4) back in F's order (zero for invalid samples) and
 * cf_gather_rows takes per-sample float4 rows of F (the composite's gradients) to C. */
int cf_compact_valid(const cf_march_out* F, const float* xu, const cf_march_out* C, float* xu_c, int* vidx, int* inv,
                     void* stream);
int cf_scatter_rows(const cf_march_out* F, const int* inv, const float* src, float* dst, void* stream);
int cf_gather_rows(const cf_march_out* C, const int* vidx, const float* src, float* dst, void* stream);

/* training rays of one key frame (device ray-batch sampler): n_rays pixels drawn
 * uniformly with replacement from fg_pixels (the frame's foreground pixel ids) by a
 * counter-based hash of (seed, i); gathers rgb (H*W,3), depth, masks at those pixels
 * and writes each pixel's exact camera ray (same directions as cf_camera_rays);
 * pix_out (optional) = the drawn pixel ids; seed_offset (optional, device) is added to
 * seed (a captured training step draws new rays every replay) */
int cf_keyframe_rays(const cf_camera* cam, const int* fg_pixels, int64_t n_fg, int64_t n_rays, uint64_t seed,
                     const uint64_t* seed_offset, const float* rgb, const float* depth, const uint8_t* mask_h, const uint8_t* mask_o, int* pix_out,
                     double* dirs, float* rgb_out, float* depth_out, uint8_t* mask_h_out, uint8_t* mask_o_out,
                     void* stream);
/* depth-guided samples of the masked rays: fills F (records, per-ray
 * offset/count, counters) and t_out (float64 depth per compacted sample; pass it as
 * M->sample_t to the canonicalisation / field / composite calls); the stratum jitter of ray i
 * is a counter-based hash of (seed + *seed_offset, ray_id0 + i): a ray draws the same samples
 * whichever shard of a data-parallel batch it is in */
int cf_train_sample(const cf_march_desc* M, const float* gt_depth, const uint8_t* mask, int n_guided, int n_uniform,
                    int n_empty, double sigma_d, uint64_t seed, const uint64_t* seed_offset, int64_t ray_id0,
                    const cf_march_out* F, double* t_out, void* stream);
/* masked L2 colour + lambda * L1 depth (lambda_depth = 0.1) and the
 * compositing backward: grad = grad_scale * float4 (dL/dsigma, dL/dr, dL/dg, dL/db) per
 * sample; norm (device, 4 floats) = [1 / n_masked, 1 / n_depth_valid, grad_scale, loss weight]
 * (cf_train_norms; grad_scale: a power of two keeping the fp16 backward operands in
 * range — loss scaling, divided out by the optimiser); loss[0] += L_color,
 * loss[1] += L_depth (normalised, times the loss weight, unscaled) */
int cf_loss_composite_bwd(const cf_march_desc* M, const cf_march_out* F, const float* field, float t_term,
                          const float* gt_rgb, const float* gt_depth, const uint8_t* mask, float lambda_depth,
                          const float* norm, float* grad, float* loss, void* stream);

/* saved activations (fp16 rows) and gradients of the E_g/E_c backward (S = capacity) */
typedef struct cf_color_bwd_io {
  void* h1;    /* (S,64) */
  void* cin;   /* (S,32) */
  void* c1;    /* (S,64) */
  void* c2;    /* (S,64) */
  void* d_o;   /* (S,16) */
  void* dc2;   /* (S,64) */
  void* dc1;   /* (S,64) */
  void* dg;    /* (S,16) */
  void* dh1;   /* (S,64) */
  float* dfeat; /* (S,32) fp32 dL/d(canonical hash features) */
} cf_color_bwd_io;
/* E_g/E_c backward on tcgen05 (forward recomputed per tile from the features that
 * cf_field_forward left in `scratch`): dX chain with the transposed weights
 * wt_blob = [C3^T 64x16, C2^T 64x64, C1^T 32x64, G2^T 64x16, G1^T 32x64] */
int cf_color_backward(const cf_field_desc* F, const uint8_t* wt_blob, const cf_march_out* S, const double* dirs,
                      const float* xu, const float* grad_out, const void* scratch, const cf_color_bwd_io* io,
                      void* stream);
/* canonical hash-grid backward at the positions the forward used (xc / xu);
 * dx_out (optional, float4 per sample): dL/dx of those positions (unit-cube
 * coordinates), the spatial gradient of the trilinear interpolation that
 * carries the loss into DeformNet */
int cf_field_hash_backward(const cf_field_desc* F, const cf_march_out* S, const float* xu, const void* scratch,
                           const float* dfeat, float* table_grad, float* dx_out, void* stream);
/* DeformNet backward buffers (S = capacity) */
typedef struct cf_deform_bwd_io {
  const void* save_h;  /* (512,S) fp16 forward h1..h4 (cf_field_desc.save_h; read by the dW GEMMs, not here) */
  const float* save_o; /* float4 per sample: raw outputs (cf_field_desc.save_o) */
  const uint32_t* save_mask; /* (S,16) ReLU bits of layers 1..4 (cf_field_desc.save_mask) */
  void* d_o;           /* (S,16) fp16 dL/d(raw outputs) */
  void* dpre;          /* (512,S) fp16 dL/d(pre-activations) of layers 1..4, feature-major as save_h */
  float* d_dfeat;      /* (S,32) fp32 dL/d(deform hash features) */
} cf_deform_bwd_io;
/* DeformNet backward on tcgen05: from dL/dxc (dxc, float4 per sample, the
 * canonical hash backward's dx_out) through xc = xu + delta_scale tanh(o) inv_side
 * and the 5 layers with the transposed weights
 * wt_blob = [W5^T 128x16, W4^T, W3^T, W2^T 128x128, W1x^T 32x128] */
int cf_deform_backward(const cf_field_desc* F, const uint8_t* wt_blob, const cf_march_out* S, const float* xu,
                       const float* dxc, const cf_deform_bwd_io* io, void* stream);
/* deformation-grid hash backward at xu: table_grad += corner weight * d_dfeat */
int cf_deform_hash_backward(const cf_field_desc* F, const cf_march_out* S, const float* xu, const float* d_dfeat,
                            float* table_grad, void* stream);
/* Adam: p -= lr * mhat / (sqrt(vhat) + eps), m/v in place; grads scaled by grad_scale */
int cf_adam(float* p, const float* g, float* m, float* v, int64_t n, float lr, float beta1, float beta2, float eps,
            int step, float grad_scale, void* stream);
/* split-K weight-gradient GEMM on tcgen05: C[128 x n_cols] += A[128 x K] B[n_cols x K]^T,
 * A / B fp16 K-major (row strides lda / ldb elements), C fp32 row-major (ldc);
 * n_cols in {32, 64, 128} */
int cf_gemm_kmajor_f16(const void* A, int64_t lda, const void* B, int64_t ldb, int n_cols, int64_t K, float* C,
                       int ldc, void* stream);
/* ---- the training step's device-side control (graph-capturable: no host syncs) */
/* one weight-gradient problem: C[m x n] += A[m x K] B[n x K]^T, A / B fp16 K-blocked
 * feature-major (the training saves): a matrix of a_rows (b_rows) rows stored as
 * capacity / 64 blocks of (rows, 64), element (r, k) at ((k / 64) * rows + r) * 64 + k % 64,
 * 16-byte aligned; the first m (n) rows are the operand; C fp32 row-major (ldc);
 * m, n in 1..128 */
typedef struct cf_dw_problem {
  const void* A;
  int64_t a_rows;
  int m;
  const void* B;
  int64_t b_rows;
  int n;
  float* C;
  int ldc;
} cf_dw_problem;
/* up to 10 problems in one tcgen05 launch (capacity % 64 == 0), K = min(*count, capacity)
 * read on the device (the frame's sample count); the operands' columns K .. roundup(K, 64) must be
 * finite with zero in A or B (the training kernels write every lane of a tile) */
int cf_dw_grouped(const cf_dw_problem* problems, int n, const int* count, int64_t capacity, void* stream);
/* masked / depth-valid ray counts of n_frames key-frame batches (frame f's rays at
 * f * frame_stride): counts (n_frames, 4) int32 = [n_m human, n_d human, n_m object, n_d object] */
int cf_train_counts(const uint8_t* mask_h, const uint8_t* mask_o, const float* gt_depth, int64_t n_rays,
                    int n_frames, int64_t frame_stride, int* counts, void* stream);
/* per-step normalisers from the counts (after the data-parallel sum over ranks):
 * norms (2 fields, n_frames, 4) = [1/n_m, 1/n_d, loss scale, 1/n_frames] (cf_loss_composite_bwd's
 * norm), adam_scale (2) = 1 / (n_frames * loss scale), stats (2 fields x 2) zeroed, ++*step,
 * *seed (optional) = the step's sampling seed offset */
int cf_train_norms(const int* counts, int n_frames, float* norms, float* adam_scale, float* stats, int* step,
                   uint64_t* seed, void* stream);
/* DeformNet layer-1 dW from the GEMM over [features | 1]: G[:, :n_x] += tmp[:, :n_x],
 * G[:, n_x + j] += tmp[:, n_x] * theta[j]; tmp (rows, ldt) zeroed */
int cf_dw_pose_cols(float* tmp, int rows, int ldt, int n_x, const float* theta, int n_theta, float* G, int ldg,
                    void* stream);
/* one tensor of cf_adam_multi; p16 (optional) receives fp16(p) after the update */
typedef struct cf_adam_tensor {
  float* p;
  float* g;
  float* m;
  float* v;
  void* p16;
  int64_t n;
  float lr;
  int scale_idx;  /* gradient scale = scale[scale_idx] */
} cf_adam_tensor;
/* Adam over up to 24 tensors in one launch: bias corrections from the device step
 * counter, gradients multiplied by the device scale (NULL = 1) and zeroed after use */
int cf_adam_multi(const cf_adam_tensor* tensors, int n, float beta1, float beta2, float eps, const int* step,
                  const float* scale, void* stream);
/* one matrix of cf_pack_multi: the packed matrix P (rows x cols) is W[r][col0 + c]
 * (transpose = 0) or W[c][col0 + r] (transpose = 1), W row stride ldw; blob_lo optional */
typedef struct cf_pack_item {
  const float* w;
  uint8_t* blob;
  uint8_t* blob_lo;
  int rows, cols, ldw, col0, transpose;
} cf_pack_item;
int cf_pack_multi(const cf_pack_item* items, int n, void* stream);
/* fp32 (n x k) row-major weight -> fp16 UMMA canonical K-major blob (n, k padded to 16) */
int cf_pack_weight(const float* w, int n, int k, uint8_t* blob, void* stream);
/* as cf_pack_weight, plus the residual fp16(W - fp16(W)) into blob_lo (same layout):
 * the B operand halves of the "fp32" precision mode */
int cf_pack_weight_split(const float* w, int n, int k, uint8_t* blob, uint8_t* blob_lo, void* stream);

/* device -> pinned host (cudaHostAlloc'd, UVA-mapped) copy by `ctas` CTAs of stores
 * instead of a copy-engine memcpy (overlaps the next view's uploads); 16-byte aligned */
int cf_store_to_host(const void* src, void* dst_host, int64_t bytes, int ctas, void* stream);
/* up to CF_COPY_BATCH_MAX small copies in one kernel launch (sources: device memory or
 * pinned host memory, read through its mapping); one CTA per entry */
#define CF_COPY_BATCH_MAX 8
typedef struct cf_copy_list {
  int n;
  const void* src[CF_COPY_BATCH_MAX];
  void* dst[CF_COPY_BATCH_MAX];
  int64_t bytes[CF_COPY_BATCH_MAX];
} cf_copy_list;
int cf_copy_batch(const cf_copy_list* list, void* stream);
/* small pinned host -> device upload by one CTA (not queued behind copy-engine transfers) */
int cf_load_from_host(void* dst, const void* src_host, int64_t bytes, void* stream);

/* ------------------------------------------------- motion-prior ingestion */
/* CFMP v1 motion-prior stream (records.py:98-147): "CFMP", u32 version, u32
 * n_nodes, u32 n_theta, then per frame i64 frame_id and four length-prefixed
 * float64 arrays (dqs n_nodes*8, theta n_theta, rotation 9, translation 3).
 * The codec is host code (no GPU needed); the arrays it fills are caller-owned
 * (pin them for one upload into the device LUT). */
typedef struct cf_mp_info {
  int64_t n_frames;
  int32_t n_nodes;
  int32_t n_theta;
  int64_t bytes;
} cf_mp_info;
/* validate a stream and count its frames (load_motion_priors, records.py:128-147);
 * CF_E_FORMAT on a bad magic / version / array length or a truncated frame */
int cf_mp_scan(const char* path, cf_mp_info* info);
/* decode frames [first, first + count) into host arrays: frame_ids (count) int64,
 * dqs (count, n_nodes, 8), theta (count, n_theta), rot (count, 3, 3), trans (count, 3) float64 */
int cf_mp_read(const char* path, int64_t first, int64_t count, int64_t* frame_ids, double* dqs, double* theta,
               double* rot, double* trans);
/* encode (MotionPriorWriter, records.py:98-120): create (header + frames) or append
 * `count` frames; appending checks the stream's n_nodes / n_theta */
int cf_mp_write(const char* path, int create, int32_t n_nodes, int32_t n_theta, int64_t count,
                const int64_t* frame_ids, const double* dqs, const double* theta, const double* rot,
                const double* trans);
/* per-frame skeleton FK on the device (skinning_transforms, skeleton.py:121-139):
 * theta (n_frames, 3J) device float64 -> A (n_frames, J, 4, 4) device float64,
 * A_j = G_j(theta) G_j(0)^-1. parents (J) int32 and offsets (J, 3) float64 are HOST
 * arrays (parents[j] < j, -1 = root), J <= 64. */
/* DeformNet layer-1 pose bias of a frame: out[i] = sum_j W[i * ldw + col0 + j] * (float)theta[j]
 * (fp32, j ascending) — the theta fold of DESIGN.md §3, run per frame on the device */
int cf_pose_bias(const float* W, int ldw, int col0, int n_out, const double* theta, int n_theta, float* out,
                 void* stream);
int cf_skinning_transforms(const double* theta, int64_t n_frames, const int32_t* parents, const double* offsets,
                           int32_t n_joints, double* A, void* stream);

/* ------------------------------------------------------ key-frame selection */
/* SPEC.md:434-519 (module keyframes), Eq. 5-7.
 * No reference code exists; the exact evaluation order is frozen in
 * oracle/keyframes.py and DESIGN.md §3.6. All pointers are device pointers. */
/* Crete-Roffet blur score of an 8-bit RGB image (H, W, 3), 0 = sharp, 1 = blurred;
 * sums = 4 x u64 device scratch (s_F / s_V per axis, exact); score = 1 double */
int cf_blur_score(const uint8_t* rgb, int height, int width, unsigned long long* sums, double* score, void* stream);
typedef struct cf_vis_camera {
  double R[9]; /* world -> camera rotation (row-major) */
  double t[3]; /* world -> camera translation */
  double fx, fy, cx, cy;
} cf_vis_camera;
/* Eq. 5 visibility map of n nodes (n,3) against a depth map (H, W) float64 metres
 * (0 = invalid): bits (ceil(n/32) words), bit i = node i visible */
int cf_visibility_map(const double* nodes, int n, const double* depth, int height, int width,
                      const cf_vis_camera* cam, double eps, uint32_t* bits, void* stream);
#define CF_POOL_HUMAN 0
#define CF_POOL_OBJECT 1
typedef struct cf_pool_desc {
  int kind;             /* CF_POOL_HUMAN (Eq. 6) or CF_POOL_OBJECT (Eq. 7) */
  int count, capacity;  /* entries in use, capacity (100) */
  int n_theta;          /* pose components (72) */
  int vis_words;        /* visibility words per entry */
  const double* theta;  /* (capacity, n_theta) */
  const uint32_t* vis;  /* (capacity, vis_words) */
  const int64_t* t;     /* (capacity) frame index / insertion time */
  const double* d;      /* (capacity, 3) object translations */
  const double* beta_pose; /* (n_theta) Eq. 6 pose weights */
  double beta_vis, beta_t, beta_d, gamma;
} cf_pool_desc;
typedef struct cf_pool_entry {
  const double* theta;
  const uint32_t* vis;
  int64_t t;
  const double* d;
} cf_pool_entry;
typedef struct cf_pool_decision {
  int insert;        /* 1: push the candidate */
  int evict;         /* entry to evict first, or -1 */
  int nearest;       /* least dissimilar entry (ties -> oldest), -1 if empty */
  int pad;
  double min_dissim;
} cf_pool_decision;
/* dissimilarity of a candidate to every pool entry (dissim: count doubles) and
 * the pool-update decision, one launch */
int cf_pool_scan(const cf_pool_desc* pool, const cf_pool_entry* cand, double* dissim, cf_pool_decision* decision,
                 void* stream);

/* --------------------------------------------- rigid-object TSDF (tsdf.py) */
/* SURVEY §8(f) 4 (tracking front-end): TsdfVolume (tsdf.py:17-171) on the device.
 * tsdf / weight: (r, r, r) float64 device arrays (x-major, as the reference's
 * meshgrid(indexing="ij")); truncation band `trunc`; weights saturate at 64. */
typedef struct cf_tsdf_desc {
  double* tsdf;
  double* weight;
  int resolution;
  int pad;
  double voxel;
  double origin[3];
  double trunc;
} cf_tsdf_desc;
typedef struct cf_rigid { /* p' = R p + t, R row-major */
  double R[9];
  double t[3];
} cf_rigid;
typedef struct cf_pinhole {
  double fx, fy, cx, cy;
  int width, height;
} cf_pinhole;
/* integrate (tsdf.py:33-61): vol_to_world = the object pose, world_to_cam = the
 * camera's inverse pose; depth (H, W) float64 metres; mask (H, W) u8 or NULL */
int cf_tsdf_integrate(const cf_tsdf_desc* V, const double* depth, int height, int width, const uint8_t* mask,
                      const cf_rigid* vol_to_world, const cf_rigid* world_to_cam, const cf_pinhole* cam, void* stream);
/* sample (tsdf.py:63-88) and/or gradient (tsdf.py:90-100) at n points (n,3):
 * val (n) + valid (n) u8 and/or grad (n,3); any output may be NULL (not both) */
int cf_tsdf_sample(const cf_tsdf_desc* V, const double* pts, int64_t n, double* val, uint8_t* valid, double* grad,
                   void* stream);
/* ray cast (tsdf.py:134-171) of every `stride`-th pixel: cam_rot = camera-to-world
 * rotation (t ignored), vol_rot = world-to-volume rotation, origin = the camera centre
 * in volume coordinates (device double[3]); per ray: pts / nrm (3) and hit (u8) */
int cf_tsdf_raycast(const cf_tsdf_desc* V, const cf_pinhole* cam, const cf_rigid* cam_rot, const cf_rigid* vol_rot,
                    const double* origin, int stride, double t0, double step, double max_t, double* pts, double* nrm,
                    uint8_t* hit, void* stream);
/* zero crossings along `axis` (tsdf.py:102-132): per voxel pair of the slice
 * ((r-1) along axis, row-major) a flag and the interpolated point (pts (n,3)) */
int cf_tsdf_crossings(const cf_tsdf_desc* V, int axis, double* pts, uint8_t* flag, void* stream);

/* ------------------------------------- non-rigid tracking solve (tracking.py) */
/* depth_normals (tracking.py:60-80): camera-facing world normals (H, W, 3) of a depth
 * map (H, W) float64 by central differences of the backprojected points (0 = invalid);
 * cam_pose = camera-to-world */
int cf_depth_normals(const double* depth, int height, int width, const cf_pinhole* cam, const cf_rigid* cam_pose,
                     double* normals, void* stream);
/* find_correspondences (tracking.py:83-150) per model point (n,3) with normals (n,3):
 * keep (n) u8, and for kept points the (subpixel) target (n,3) and depth normal n_u
 * (n,3); mask (H, W) u8 or NULL; world_to_cam = the camera pose's inverse;
 * cos_max = cos(normal gate) */
int cf_find_correspondences(const double* pts, const double* pt_normals, int64_t n, const double* depth, int height,
                            int width, const uint8_t* mask, const double* normals_map, const cf_pinhole* cam,
                            const cf_rigid* cam_pose, const cf_rigid* world_to_cam, double tau, double cos_max,
                            double* target, double* n_u, uint8_t* keep, void* stream);
/* rigid_icp (tracking.py:560-620) building blocks: transform model points / normals by
 * T; point-to-plane residuals of the kept correspondences (0 elsewhere); the Huber-
 * weighted 6x6 normal equations sums[0..21) = upper triangle of Jr^T Jr (row-major),
 * sums[21..27) = Jr^T (w r) (zeroed here, accumulated with fp64 atomics) */
int cf_rigid_transform(const double* pts, const double* normals, int64_t n, const cf_rigid* T, double* out_pts,
                       double* out_normals, void* stream);
int cf_icp_residuals(const double* live, const uint8_t* keep, const double* target, const double* n_u, int64_t n,
                     double* r, void* stream);
int cf_icp_normal_equations(const double* live, const uint8_t* keep, const double* n_u, const double* r, int64_t n,
                            double knee, double* sums, void* stream);
/* Non-rigid tracker (tracking.py:270-508) on the device. cf_nr_warp: apply_blended
 * (edgraph.py:198-205) of n samples with fixed neighbours idx (n,k) int32 and weights
 * w (n,k). cf_nr_terms: the data / bind / reg / pose terms of energy_terms
 * (unweighted sums -> energy[0..4)) and, when val != NULL, their Jacobian rows in CSR
 * (val / col at each term's entry offset, residuals at its row offset; rows: data 6k
 * entries, bind 6+T, reg 12, pose T). cf_nr_step: _apply_step's node update. */
typedef struct cf_nr_system {
  const double* dqs;
  const double* nodes;
  int n_nodes, n_theta;
  const double* warped;
  const int64_t* data_idx;
  const double* data_u;
  const double* data_n;
  int64_t n_data;
  const int* blend_idx;
  const double* blend_wn;
  int k;
  double w_data;
  int64_t data_row0, data_entry0;
  int do_bind;
  const double* node_lbs;
  const double* node_jth;
  double s_bind;
  int64_t bind_row0, bind_entry0;
  const int64_t* edges;
  int64_t n_edges;
  double s_reg;
  int64_t reg_row0, reg_entry0;
  const double* pose_lbs;
  const double* pose_u;
  const double* pose_n;
  const double* pose_jth;
  int64_t n_pose;
  double w_pose;
  int64_t pose_row0, pose_entry0;
  double* val;
  int* col;
  double* res;
  double* energy;   /* [data, bind, reg, pose] energies, each a fixed-order sum (deterministic) */
  int jac_terms;    /* with val: bit 0 data, 1 bind, 2 reg, 3 pose = write that term's Jacobian rows */
} cf_nr_system;
int cf_nr_warp(const double* dqs, const int* idx, const double* w, int k, const double* pts, const double* normals,
               int64_t n, double* out_pts, double* out_normals, void* stream);
int cf_nr_terms(const cf_nr_system* S, void* stream);
int cf_nr_step(const double* dqs, const double* delta, int n, double* out, void* stream);
/* CSR matrix on the device (int32 indices) */
typedef struct cf_csr {
  const double* val;
  const int* col;
  const int* rowptr; /* rows + 1 */
  int rows, cols;
  int64_t nnz;
} cf_csr;
/* workspace (doubles) cf_pcg_solve needs for a rows x cols Jacobian */
int cf_pcg_workspace_doubles(int rows, int cols, int64_t* n_doubles);
/* pcg_solve (tracking.py:158-193): Jacobi-PCG on (J^T J + lambda diag(J^T J)) x = -J^T r,
 * at most max_iters iterations, stop when |res| <= tol |b|; one cooperative launch.
 * JT = J transposed (CSR); x (cols) out; iters (device int) = iterations run, or NULL */
int cf_pcg_solve(const cf_csr* J, const cf_csr* JT, const double* r, double lm_lambda, int max_iters, double tol,
                 double* x, double* work, int* iters, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CAPFIELDS_B200_H */
