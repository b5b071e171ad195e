/*
 * agr.h -- C ABI of the B200-native batched ray caster (libagr.so).
 *
 * The hot path of the Aerial Gym Simulator renderer (arxiv 2503.01471,
 * PAPER.md §III.D.1 "Exteroceptive Sensors", lines 226-228): per-environment
 * meshes made of transformed sub-meshes, a bounding volume hierarchy over
 * them, and rays "cast outwards per-pixel to evaluate intersection",
 * reporting range (ToF / LiDAR) or depth (camera), segmentation and face
 * index images (Fig. 3).
 *
 * Design: the paper's per-env merged mesh M_{i,t} = T o M^base
 * is represented as instances of shared asset meshes.  Each asset gets a
 * bottom-level BVH (BLAS, LBVH: 30-bit Morton codes, on-device radix sort,
 * Karras hierarchy) built once at create; each environment gets a top-level
 * BVH (TLAS) over its instances, rebuilt by agr_build or refit in place by
 * agr_refit after agr_set_instance_transforms.  Casts are hand-written CUDA
 * kernels for sm_100a; results equal the plain definition of DESIGN.md §3.
 *
 * Conventions (DESIGN.md §4 "Readings"):
 *  - transforms are row-major float[3][4] T = [A | b], x' = A x + b
 *    (object -> env-local for instances; sensor -> env-local for poses; the
 *    columns of a pose's A are the sensor axes x forward, y left, z up);
 *  - pinhole pixel (u, v) has its centre at (u + 0.5, v + 0.5), u to the
 *    right (-y), v downward (-z); sensor-frame direction
 *    d_s = (1, -(u + 0.5 - cx)/fx, -(v + 0.5 - cy)/fy);
 *  - DEPTH reports t for d_s as written (= distance from the image plane);
 *    RANGE and beams report t for the unit direction (= Euclidean range);
 *  - a hit needs 0 < t <= max_range on a closed, double-sided triangle; the
 *    smallest t wins, equal t goes to the lowest per-env face index;
 *  - misses write max_range, seg -1, face -1;
 *  - per-env face index = sum of face counts of the env's earlier instances
 *    (creation order) + the asset-local face index; seg = instance label.
 *
 * Errors: every call returns agr_status.  Host-checkable argument errors
 * return before any launch and leave the scene unchanged.  CUDA launch
 * errors return AGR_ECUDA; asynchronous device faults surface at the
 * caller's next synchronisation or at the next agr call.  No exceptions
 * cross the ABI and the library never aborts.  agr_last_error() returns a
 * thread-local message for the last failing call on this thread.
 *
 * Ownership: host arrays passed to agr_scene_create are copied before it
 * returns.  Device buffers passed to set/cast calls are caller-owned and
 * must stay alive until the work on `stream` completes; the library never
 * frees them.  The library owns every BVH / instance buffer it allocates
 * and frees them in agr_scene_destroy.  All device work is asynchronous on
 * the caller's stream (a cudaStream_t passed as void*, NULL = legacy default
 * stream) with no hidden synchronisation, except where a call says so.  One
 * scene must be used by one stream at a time; different scenes may be used
 * concurrently from different threads.
 *
 * CUDA graphs: agr_set_instance_transforms, agr_build, agr_refit, the device
 * casts, agr_checksum and agr_sim_kinematic_step enqueue only kernels,
 * device copies and event records, so a step made of them can be captured
 * (cudaStreamBeginCapture / torch.cuda.graph) and replayed -- bench.py's
 * Table-II env step does.  agr_update_mesh(es) uploads host-side tables
 * through a staging buffer that later calls overwrite, and the *_host casts
 * synchronise: do not capture those.
 */
#ifndef AGR_H
#define AGR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AGR_ABI_VERSION 4

typedef int32_t agr_status;
enum {
    AGR_OK = 0,
    AGR_EINVAL = -1,       /* bad argument (null pointer, size, index)      */
    AGR_ENOMEM = -2,       /* device or host allocation failed              */
    AGR_ECUDA = -3,        /* CUDA runtime error (message in agr_last_error) */
    AGR_ESTATE = -4,       /* call not valid in this state (e.g. no build)  */
    AGR_EUNSUPPORTED = -5  /* a size beyond a documented limit              */
};

/* Documented limits. */
#define AGR_MAX_INSTANCES_PER_ENV 1024 /* per-env TLAS is built in one CTA   */
#define AGR_MAX_BVH_DEPTH 94           /* binary BLAS depth accepted at create
                                          (the traversal stack holds 96
                                          entries).  A mesh update that makes a
                                          BLAS deeper is still correct: a ray
                                          whose stack would overflow is
                                          re-solved by an FP64 test of every
                                          triangle of its env (counter [5];
                                          agr_scene_get_info reports the new
                                          blas_max_depth).                  */

typedef struct agr_scene_s* agr_scene;

/* One asset mesh (a sub-mesh M_j of PAPER.md:226), host memory. */
typedef struct {
    const float* verts;   /* [n_verts][3] object-space vertices (metres)    */
    int32_t n_verts;      /* >= 3                                            */
    const int32_t* faces; /* [n_faces][3] vertex indices in [0, n_verts)     */
    int32_t n_faces;      /* >= 1; zero-area faces are kept for numbering
                             and are never hit                               */
} agr_mesh;

/* One instance of an asset in an environment. */
typedef struct {
    int32_t asset;        /* index into the meshes array                     */
    int32_t label;        /* segmentation id written for its hits (>= 0)     */
} agr_instance;

/* Pinhole intrinsics in pixels. */
typedef struct {
    int32_t width, height;
    float fx, fy, cx, cy;
} agr_pinhole;

typedef enum { AGR_DEPTH = 0, AGR_RANGE = 1 } agr_distance;

/* Output images.  Each pointer is caller-owned memory (device memory for
 * the device casts, host memory for the *_host casts) laid out
 * [n_envs][n_sensors][rows][cols] (pinhole rows = height, cols = width;
 * beams rows = C channels, cols = K columns; rays: [n_envs][R]), with a
 * trailing vector dimension for normal / bary / point.  Any pointer may be
 * NULL to skip that channel.  Channels after `face` are the per-hit data
 * of PAPER.md:218 / :228 (surface normals, barycentric coordinates, point
 * clouds), computed in FP64 from the winning triangle. */
typedef struct {
    float* dist;          /* depth / range (metres); max_range on a miss     */
    int32_t* seg;         /* instance label, -1 on a miss                    */
    int32_t* face;        /* per-env face index, -1 on a miss                */
    float* normal;        /* [..][3] unit geometric normal of the hit face in
                             the env frame, oriented towards the ray origin
                             (n . d < 0); (0,0,0) on a miss                  */
    float* bary;          /* [..][2] (b1, b2): hit = (1-b1-b2) v0 + b1 v1 +
                             b2 v2 over the face's vertices in face order;
                             (-1,-1) on a miss                               */
    float* point;         /* [..][3] o + dist * d in the env frame (the hit
                             point; the max-range point on a miss)           */
    int32_t* valid;       /* stereo shadow mask: 0 if the
                             segment from the hit point to the second sensor
                             (agr_set_stereo) hits the scene at a distance in
                             (eps, L - eps) from the hit point, else 1; 1 on
                             a miss.  Pinhole and beam casts only (explicit
                             rays write 1).                                  */
    float* annot;         /* [..][k] vertex annotations of the hit face
                             (agr_set_vertex_annotations) interpolated with
                             its barycentrics: (1-b1-b2) A(v0) + b1 A(v1) +
                             b2 A(v2); NaN on a miss or on an asset without
                             annotations.  EINVAL if none were set.          */
} agr_outputs;

/* Scene statistics (sizes in elements / bytes of library-owned memory). */
typedef struct {
    int32_t n_assets, n_envs;
    int64_t n_instances, n_blas_nodes, n_blas_tris, n_tlas_nodes;
    int32_t blas_max_depth, tlas_max_depth;
    int64_t device_bytes;
    int32_t built;        /* 1 after the first agr_build                     */
    int32_t n_parts;      /* BLAS parts over all assets (>= n_assets; see
                             agr_create_options.part_policy)                 */
    int64_t n_items;      /* TLAS leaves over all envs: (instance, part)     */
} agr_scene_info;

int32_t agr_abi_version(void);

/* Thread-local message describing the last failing call ("" if none). */
const char* agr_last_error(void);

/*
 * Create a scene on CUDA device `device`: copies the asset meshes and the
 * instance table, builds every BLAS (synchronous; returns when done).
 *   env_offsets: host int64 [n_envs + 1], env e owns instances
 *                [env_offsets[e], env_offsets[e+1]); env_offsets[0] == 0.
 *   inst:        host [env_offsets[n_envs]] instance table.
 * Instance transforms start as identity; call agr_set_instance_transforms
 * and agr_build before the first cast.
 * EINVAL: null pointers, n_meshes < 1, n_envs < 1, a face index out of
 * range, a non-finite vertex, an asset index out of range, a negative
 * label, non-monotone env_offsets.  EUNSUPPORTED: an env with more than
 * AGR_MAX_INSTANCES_PER_ENV instances or a BLAS deeper than the traversal
 * stack.  On error *out is set to NULL.
 */
agr_status agr_scene_create(int32_t device, const agr_mesh* meshes, int32_t n_meshes,
                            int32_t n_envs, const int64_t* env_offsets,
                            const agr_instance* inst, agr_scene* out);

/* Creation options (agr_scene_create uses the defaults). */
typedef struct {
    int32_t trbvh_rounds; /* treelet-restructuring passes applied to every
                             BLAS after the LBVH (Karras & Aila 2013; SAH-
                             optimal treelets of 7 subtrees), 0..16; default 3.
                             0 keeps the plain Karras LBVH.                  */
    int32_t part_policy;  /* 0 (default): an asset whose faces form several
                             connected components that fill much less than
                             their common box (a tree's trunk and canopy) is
                             split into up to 4 parts, each with its own BLAS
                             and its own TLAS leaf per instance, so rays only
                             enter the parts they approach; kept when the
                             parts' box areas sum to < 0.85 of the whole
                             box's and no env exceeds 2048 TLAS leaves.
                             Results are identical either way (the BVH only
                             accelerates the plain definition).
                             1: one BLAS per asset.                          */
    int32_t node_width;   /* width of the wide BVH copy kept beside the 4-wide
                             BVH every traversal uses, for the interval-packet
                             camera / LiDAR traversal: 8 (256-B nodes) or 16
                             (512-B nodes: lanes 0-15 test the children, 16-31
                             order them) or 32 (1-KB nodes: every lane tests
                             one child, ordered by the tile's entry bound);
                             0 (default): 32 (c3 +5 % over 8; an env of at
                             most 32 TLAS items is one wide node: c4 +2 %,
                             c5 +4 %);
                             4: no wide copy (half the node memory and no wide
                             collapse in builds / refits -- for scenes cast one
                             ray per lane).                                  */
    int32_t reserved[5];  /* must be 0                                        */
} agr_create_options;

agr_status agr_scene_create_ex(int32_t device, const agr_mesh* meshes, int32_t n_meshes,
                               int32_t n_envs, const int64_t* env_offsets,
                               const agr_instance* inst, const agr_create_options* opts,
                               agr_scene* out);

/* Free all device memory of the scene (synchronises its device). NULL: no-op. */
agr_status agr_scene_destroy(agr_scene scene);

agr_status agr_scene_get_info(agr_scene scene, agr_scene_info* info);

/*
 * PAPER.md:226 (§III.D.1): "transformations for each sub-mesh at time t are
 * maintained as T_{i,t} = {T_{j,t}}" and "the vertices of the mesh are
 * transformed to match the obstacles in the simulator at time t as
 * M_{i,t} = T^T_{i,t} o M^base_i".  Here the transform is applied to the rays instead
 * (instancing): copy new instance transforms (device float
 * [n_instances][3][4], row-major object -> env-local x' = A x + b; A must
 * be invertible; EINVAL for a NULL T with instances) into the scene and
 * recompute the per-instance ray transforms and bounds.  Async on
 * `stream`; T may be reused once the stream passes this point.  The TLAS is
 * stale until agr_build or agr_refit.
 */
agr_status agr_set_instance_transforms(agr_scene scene, const float* T, void* stream);

/*
 * Replace the vertices of asset `asset` (device float [n_verts][3], same
 * count and face topology as at create) and rebuild its BLAS on `stream`
 * (Morton codes, radix sort, Karras, fit, collapse -- all on the device,
 * no host round trip), then recompute every instance's bounds.  This is the
 * paper's per-env mesh update at reset ("performing this
 * exclusively for randomization of static environments"): give each env
 * its own asset for per-env unique or deforming meshes.  Faces that become
 * (non-)degenerate are handled (numbering is kept).  The TLAS is stale
 * until agr_build / agr_refit.  Non-finite vertices give unspecified
 * results for that asset.
 */
agr_status agr_update_mesh(agr_scene scene, int32_t asset, const float* verts, int32_t n_verts,
                           void* stream);

/*
 * Per-vertex annotations of asset `asset` ("embed vertex-level
 * annotations that can be queried"): `values` device float [n_verts][k],
 * k in [1, AGR_MAX_ANNOT], the same k for every asset of the scene (fixed
 * by the first call).  Copied into library memory on `stream` (async;
 * `values` may be reused once the stream passes this point).  Assets never
 * given annotations read NaN.  Casts with out.annot interpolate them.
 * EINVAL on a bad asset, a vertex-count mismatch or a k mismatch.
 */
#define AGR_MAX_ANNOT 8
agr_status agr_set_vertex_annotations(agr_scene scene, int32_t asset, const float* values, int32_t n_verts,
                                      int32_t k, void* stream);

/*
 * Batched agr_update_mesh: replace the vertices of the n distinct assets
 * `assets` (host int32 [n]) with `verts` (device float [sum of their vertex
 * counts][3], the assets' vertex arrays concatenated in the order of
 * `assets`) and rebuild all n BLAS in ONE set of launches (the build's
 * kernels run over the concatenated faces; each asset's tree is exactly the
 * one agr_update_mesh would build).  This is the reset path for per-env
 * unique meshes: n = number of envs being reset.
 * EINVAL on n < 0, a NULL pointer with n > 0, an asset out of range or
 * listed twice.  Async on `stream`; `assets` is read before return.
 */
agr_status agr_update_meshes(agr_scene scene, int32_t n, const int32_t* assets, const float* verts,
                             void* stream);

/* "a bounding volume hierarchy is calculated for M_{i,t} for
 * efficient ray-casting" -- here the per-env top level over the instances
 * (the per-asset bottom levels are built at create / agr_update_mesh(es)).
 * Full per-env TLAS rebuild (one CTA per env: LBVH -- Morton order + Karras
 * hierarchy -- or, after agr_set_tlas_builder(scene, 1), a binned-SAH
 * top-down split of the instance boxes), bottom-up fit and 4- / 8-wide
 * collapse.  Async; EINVAL for a NULL scene. */
agr_status agr_build(agr_scene scene, void* stream);

/* In-place TLAS refit (the transformations T_{i,t} change with
 * t while the env's sub-meshes M^base_i stay): keeps the topology of the last
 * agr_build and recomputes all boxes bottom-up.  Async.  ESTATE before the
 * first agr_build. */
agr_status agr_refit(agr_scene scene, void* stream);

/*
 * Pinhole camera cast.  poses: device float
 * [n_envs][n_sensors][3][4] (sensor -> env-local).  Outputs
 * [n_envs][n_sensors][height][width].  max_range > 0 in the reported unit.
 * ESTATE if transforms were set after the last build/refit.
 */
agr_status agr_cast_pinhole(agr_scene scene, const agr_pinhole* cam, agr_distance kind,
                            const float* poses, int32_t n_sensors, float max_range,
                            agr_outputs out, void* stream);

/*
 * Beam-table cast for LiDARs and other central projections (PAPER.md:215,
 * :228 "customizable projection models (e.g., Dome LiDAR)").  dirs: device
 * float [C][K][3] sensor-frame directions (normalised in FP64 by the
 * library; need not be exactly unit).  Always reports range.  Outputs
 * [n_envs][n_sensors][C][K].
 */
agr_status agr_cast_beams(agr_scene scene, const float* dirs, int32_t C, int32_t K,
                          const float* poses, int32_t n_sensors, float max_range,
                          agr_outputs out, void* stream);

/*
 * Explicit rays (test / debug entry, SPEC cast_rays): orig, dir device
 * float [n_envs][R][3] in env-local coordinates; t is reported in units of
 * |dir| (no normalisation).  Outputs [n_envs][R].
 */
agr_status agr_cast_rays(agr_scene scene, const float* orig, const float* dir, int32_t R,
                         float max_range, agr_outputs out, void* stream);

/*
 * End-to-end pinhole cast through HOST buffers: copies `poses_host`
 * (pageable or pinned host memory) to the device, casts, and copies the
 * images back into the host pointers of `out_host`, pipelining the
 * device->host copies with the casts of later env chunks on internal
 * streams.  The internal streams first wait (cudaStreamWaitEvent, no host
 * sync) for the scene work of the last agr_set_instance_transforms /
 * agr_update_mesh(es) / agr_set_vertex_annotations / agr_build / agr_refit
 * on whatever stream it was queued, so no caller-side sync is needed
 * between those calls and this one.  Synchronous: returns when out_host
 * is filled.  EINVAL on bad intrinsics or an invalid `kind`.
 */
agr_status agr_cast_pinhole_host(agr_scene scene, const agr_pinhole* cam, agr_distance kind,
                                 const float* poses_host, int32_t n_sensors, float max_range,
                                 agr_outputs out_host);

/* End-to-end beams cast through host buffers (see agr_cast_pinhole_host). */
agr_status agr_cast_beams_host(agr_scene scene, const float* dirs_host, int32_t C, int32_t K,
                               const float* poses_host, int32_t n_sensors, float max_range,
                               agr_outputs out_host);

/*
 * Per-env order-independent 64-bit checksums of an output image set
 * (device pointers as produced by a cast; NULL channels are skipped):
 * sums[e] = sum over the env's elements of mix64(index, dist bits, seg,
 * face).  sums: device uint64 [n_envs].  Used to compare runs bitwise
 * across GPU counts without moving images.  Async.
 */
agr_status agr_checksum(agr_scene scene, agr_outputs out, int64_t elems_per_env,
                        uint64_t* sums, void* stream);

/*
 * Second sensor of a stereo pair for the `valid` output channel: its origin
 * is (ox, oy, oz) in each pose's sensor frame (x forward, y left, z up;
 * e.g. (0, -0.095, 0) for a right camera 95 mm away), and eps > 0 is the
 * self-hit guard in metres.  Defaults: (0, -0.095, 0), 1e-4.
 */
agr_status agr_set_stereo(agr_scene scene, float ox, float oy, float oz, float eps);

/*
 * Numerics mode (test hook): 0 = FP32 filter + FP64 arbitration (default);
 * 1 = exact mode, every leaf test in FP64 (slow; results must be identical).
 */
agr_status agr_set_exact_mode(agr_scene scene, int32_t exact);

/* TLAS builder used by the next agr_build: 0 = LBVH (default), 1 = binned
 * SAH.  Results are identical either way; only the speed differs (on the c3
 * forest the SAH TLAS saves 4 % of the TLAS node visits but its build costs
 * ~1 ms per 1024 envs, so LBVH is the default). */
agr_status agr_set_tlas_builder(agr_scene scene, int32_t builder);

/*
 * Traversal schedule (results are identical either way): 0 = auto (default;
 * the 32 rays of a 4x8 pinhole tile (8 columns x 4 channels for beam
 * tables) traverse as one warp packet: a
 * node is visited when the interval of the tile's ray directions may reach
 * a child, and every lane still tests each visited leaf on its own ray;
 * stereo shadow segments, whose origins differ per lane, visit the union
 * of the lanes' own box tests; on the 8-wide node copy when it exists,
 * agr_create_options.node_width; a pinhole whose 4x8 tile spans more than
 * 0.12 rad -- 4 / fx or 8 / fy, i.e. fx or fy below ~67 px: small images
 * with a wide field of view -- is cast one ray per lane instead, because a
 * wide direction interval culls little), 1 = one independent ray per lane
 * (faster when a tile's rays diverge, e.g. terrain seen at grazing angles),
 * 2 = the packets of mode 0 on the 4-wide nodes, for every camera
 * (comparison / testing), 3 = the packets of mode 0 on the 8-wide nodes
 * (the 4-wide ones if there is no BVH8 copy) for every camera.
 * Explicit rays always use 1.  EINVAL outside 0..3.
 */
agr_status agr_set_traversal(agr_scene scene, int32_t mode);

/*
 * Counters of the last cast (test / profiling hook; device-side counters
 * are collected only when enabled):  counters[0] rays, [1] internal nodes
 * visited, [2] leaf (triangle) tests, [3] instance entries, [4] FP64
 * arbitration tests, [5] candidate-list overflows / stack fallbacks,
 * [6] internal nodes visited at the TLAS level, [7] instance entries whose
 * BLAS root test hit no child for the lane's own ray (node and leaf counts
 * are per lane: in packet mode every lane counts each warp visit; [7] is
 * counted in mode 1 only).
 */
agr_status agr_enable_counters(agr_scene scene, int32_t enable);
agr_status agr_get_counters(agr_scene scene, int64_t counters[8]);

/*
 * Debug export of one asset's BLAS for structural tests (synchronous):
 * nodes float [n_nodes][16] (packed 64-byte nodes), leaf_face int32
 * [n_leaves] (asset-local face of each leaf in BVH order), morton uint32
 * [n_leaves] (sorted codes).  Pass NULL to query sizes via *n_nodes and
 * *n_leaves.  Node child refs: >= 0 node index relative to the asset's
 * first node, < 0 leaf ~index relative to the asset's first leaf,
 * INT32_MIN empty.  The binary nodes are packed by the create-time build
 * only: after agr_update_mesh(es) of this asset, a request for `nodes`
 * returns AGR_ESTATE (leaf_face and morton stay available).
 * AGR_EUNSUPPORTED for an asset split into several BLAS parts
 * (agr_create_options.part_policy).
 */
agr_status agr_debug_export_blas(agr_scene scene, int32_t asset, float* nodes,
                                 int32_t* leaf_face, uint32_t* morton,
                                 int64_t* n_nodes, int64_t* n_leaves);

/*
 * Debug export of the traversal BVH4 (synchronous).  which >= 0: the BLAS of
 * asset `which` (AGR_EUNSUPPORTED if it is split into parts); which < 0:
 * the TLAS of env (-1 - which) (after agr_build).
 * nodes float [n_nodes][32]: per node lo.x[4] hi.x[4] lo.y[4] hi.y[4]
 * lo.z[4] hi.z[4] ref[4] (int bits) cnt; refs are global (>= 0 node index,
 * < 0 ~leaf: triangle record, or global TLAS item = (instance, part) in
 * instance order; INT32_MIN empty).
 * *root = global index of node 0 of the export.  NULL nodes: size query.
 * A BLAS export holds exactly the nodes reachable from its root (the BVH4
 * is compacted at every build); a TLAS export holds one node per binary
 * node, unreachable ones included.
 */
agr_status agr_debug_export_bvh4(agr_scene scene, int32_t which, float* nodes, int32_t* root,
                                 int64_t* n_nodes);

/*
 * Debug export of asset `asset`'s BLAS parts (agr_create_options.
 * part_policy): *n_parts, and, if part_of_face is not NULL, the part
 * (0 .. n_parts - 1) of each of its faces (host int32 [n_faces]).
 */
agr_status agr_debug_asset_parts(agr_scene scene, int32_t asset, int32_t* part_of_face, int32_t* n_parts);

#ifdef __cplusplus
}
#endif
#endif /* AGR_H */
