// agr_internal.cuh -- device data layouts and small helpers shared by the
// libagr.so translation units (BLAS build, TLAS build/refit, casts, ABI).
//
// Nothing here is shared with oracle/ (the oracle and the CUDA
// path share no code).
//
// HBM layout:
//   nodes   BVH4 nodes, float4[8] = 128 B, BLAS nodes of every asset first,
//           then every env's TLAS nodes.  A BLAS's BVH4 holds only the
//           nodes reachable from its root: BVH4 node k (from node_base) is
//           the greedy 4-wide collapse of the k-th reachable binary node in
//           binary order (root = 0; BlasInfo.n_nodes4 in use).  A TLAS's
//           BVH4 node j is the collapse of its binary node j (reachable or
//           not).  Boxes of the 4 children stored per axis:
//             f0 = lo.x[4], f1 = hi.x[4], f2 = lo.y[4], f3 = hi.y[4],
//             f4 = lo.z[4], f5 = hi.z[4], f6 = ref[4] (int bits), f7 = (n, -)
//           ref >= 0: global node index; ref < 0: leaf ~x (TLAS: x = global
//           item; BLAS: x = first | (count - 1) << LEAF_SHIFT, a leaf of
//           `count` <= LEAF_MAX consecutive triangle records whose box is
//           their union -- a binary subtree over at most LEAF_MAX
//           consecutive leaves is referenced as one such leaf instead of
//           getting BVH4 nodes of its own); REF_EMPTY: no child (its box is
//           +inf everywhere, never hit).
//   bnodes  the binary LBVH of every BLAS (64-B nodes: child boxes + refs),
//           kept for structural checks (agr_debug_export_blas).
//   tris    float4[3] per BLAS leaf, 48 B (FP32 filter test, object space):
//             t0 = (v0.xyz, inv_min_alt)   inv_min_alt = 1 / min altitude
//             t1 = (e1.xyz, two_area)      e1 = v1 - v0, two_area = |e1 x e2|
//             t2 = (e2.xyz, local face id as int bits)
//   triv    float4[3] per BLAS leaf: the exact FP32 input vertices v0 v1 v2 (w = 0)
//           (read only by the FP64 arbitration / epilogue).
//   irec    float4[4] per TLAS item, 64 B (ray -> object space):
//             r0..r2 = rows of [Ainv | binv] (FP64 inverse rounded to FP32)
//             r3 = (blas root node (int bits), nAinv, err_off, instance (int bits))
//
// Parts and items.  An asset whose faces form several connected components
// spread over a much larger box than they fill (a tree: thin trunk + round
// canopy) is split at create into up to MAX_PARTS parts, each with a BLAS
// of its own (a "part" = one BLAS; BlasInfo is per part).  The TLAS leaves
// are ITEMS = (instance, part) pairs, so a ray enters only the parts whose
// world boxes it crosses.  Triangle records keep the asset-local face id, so
// face numbering, labels and every output are unchanged.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define AGR_HD __host__ __device__ __forceinline__

namespace agr {

constexpr int REF_EMPTY = (int)0x80000000;  // INT32_MIN
#ifndef AGR_LEAF_MAX
#define AGR_LEAF_MAX 2
#endif
constexpr int LEAF_MAX = AGR_LEAF_MAX;      // triangles per BLAS leaf (1..4)
constexpr int LEAF_SHIFT = 29;              // BLAS leaf ref: count - 1 in bits 29-30
constexpr int LEAF_MASK = (1 << LEAF_SHIFT) - 1;  // first record (faces_total < LEAF_MASK - 4, abi.cu)
constexpr int STACK_SIZE = 96;              // traversal stack entries per ray
constexpr int MAX_PARTS = 4;                // BLAS parts per asset
constexpr int MAX_TLAS_N = 2048;            // TLAS leaves (items) per env: one-CTA build

// Relative error budget of the FP32 object-space ray:
// position error <= K_ERR * (nAinv * (|o|_1 + |b|_1 + t_max |d|_1) + r_asset).
constexpr float K_ERR = 7.62939453125e-06f;  // 2^-17
// Relative slack on FP32 t values (ray direction rounding etc.).
constexpr float T_REL = 9.5367431640625e-07f;  // 2^-20

// One BLAS (an asset part).
struct BlasInfo {
    int node_base;   // global index of the BLAS root node
    int leaf_base;   // global index of its first leaf record
    int n_leaves;    // non-degenerate triangles in the BLAS
    int n_faces;     // faces of the part
    float lo[3], hi[3];  // root box (object space, exact min/max)
    float radius;    // max |v| over the vertices of the part's faces (object units)
    int depth;       // BLAS depth (edges from root to deepest leaf)
    int n_nodes4;    // BVH4 nodes in use from node_base (the reachable collapse, compacted)
};

// Read-only view of a scene passed by value to kernels.
struct SceneView {
    const float4* nodes;      // [n_nodes][8] BVH4
    int wide_w;               // width of the wide copy: 8, 16 or 32 (0: none)
    const float4* nodesw;     // [n_nodes][2 wide_w] BVH8 / BVH16 copy (its own numbering; BLAS roots and TLAS nodes at the
                              // same indices as the BVH4), or null
    const float4* tris;       // [n_leaves][3]
    const float* triv;        // [n_leaves][3] float4 (v.xyz, 0)
    const float4* irec;       // [n_items][4] (TLAS leaf ~item)
    const float* inst_T;      // [n_inst][12] forward transforms (FP32 input)
    const int* inst_face_off; // [n_inst] per-env face offset of the instance
    const int* inst_label;    // [n_inst]
    const int* env_off;       // [n_envs + 1]
    const int* tlas_root;     // [n_envs] global node index of the env's TLAS root
    const int* inst_asset;    // [n_inst]
    const BlasInfo* parts;    // [n_parts]
    const int* part_off;      // [n_assets + 1] parts of asset a: [part_off[a], part_off[a+1])
    int n_envs;
    // vertex annotations (f1): [sum V][annot_k] by asset vertex, NaN = none
    const float* annot;
    int annot_k;
    const int* mesh_faces;    // [sum F][3] asset-local vertex ids (face order)
    const int* asset_voff;    // [n_assets] first vertex of each asset in annot rows
    const int* asset_foff;    // [n_assets] first face of each asset in mesh_faces
};

// ---- small vector helpers --------------------------------------------------
struct f3 { float x, y, z; };
struct d3 { double x, y, z; };

AGR_HD f3 mk(float x, float y, float z) { f3 r; r.x = x; r.y = y; r.z = z; return r; }
AGR_HD f3 sub(f3 a, f3 b) { return mk(a.x - b.x, a.y - b.y, a.z - b.z); }
AGR_HD float dot(f3 a, f3 b) { return fmaf(a.x, b.x, fmaf(a.y, b.y, a.z * b.z)); }
AGR_HD f3 cross(f3 a, f3 b) {
    return mk(fmaf(a.y, b.z, -a.z * b.y), fmaf(a.z, b.x, -a.x * b.z), fmaf(a.x, b.y, -a.y * b.x));
}
AGR_HD d3 mkd(double x, double y, double z) { d3 r; r.x = x; r.y = y; r.z = z; return r; }
AGR_HD d3 subd(d3 a, d3 b) { return mkd(a.x - b.x, a.y - b.y, a.z - b.z); }
AGR_HD double dotd(d3 a, d3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
AGR_HD d3 crossd(d3 a, d3 b) {
    return mkd(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}

// ---- 30-bit Morton code (10 bits per axis) -------------------------------
AGR_HD uint32_t expand_bits10(uint32_t v) {
    v = (v * 0x00010001u) & 0xFF0000FFu;
    v = (v * 0x00000101u) & 0x0F00F00Fu;
    v = (v * 0x00000011u) & 0xC30C30C3u;
    v = (v * 0x00000005u) & 0x49249249u;
    return v;
}
// x, y, z in [0, 1]: quantise min(floor(x * 1024), 1023); x in bit 2 of
// each triple (x most significant), as in Karras 2012.
AGR_HD uint32_t morton30(float x, float y, float z) {
    uint32_t xi = (uint32_t)fminf(fmaxf(floorf(x * 1024.0f), 0.0f), 1023.0f);
    uint32_t yi = (uint32_t)fminf(fmaxf(floorf(y * 1024.0f), 0.0f), 1023.0f);
    uint32_t zi = (uint32_t)fminf(fmaxf(floorf(z * 1024.0f), 0.0f), 1023.0f);
    return (expand_bits10(xi) << 2) | (expand_bits10(yi) << 1) | expand_bits10(zi);
}

// Normalise a centroid coordinate to the centroid bounds; a zero-extent axis
// uses extent 1.
AGR_HD float unit_coord(float c, float lo, float hi) {
    float ext = hi - lo;
    return ext > 0.0f ? (c - lo) / ext : 0.0f;
}

// ---- float <-> orderable uint for atomic min/max ---------------------------
__device__ __forceinline__ uint32_t float_to_ordered(float f) {
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ordered_to_float(uint32_t u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
}

// ---- 4-wide collapse of a binary LBVH node -----------------------------------------
AGR_HD float half_area(const float b[6]) {
    float dx = b[3] - b[0], dy = b[4] - b[1], dz = b[5] - b[2];
    return dx * dy + dy * dz + dz * dx;
}

// Greedy collapse of binary node j into up to W children (W = 4: the BVH4 of
// every traversal mode; W = 8: the BVH8 of the interval-packet traversal):
// repeatedly open the internal child with the largest surface area (the
// SAH's choice), keeping the children in left-to-right (Morton) order.  Refs
// are local: >= 0 binary internal node, < 0 leaf.  child(r, side) and box(r,
// b[6]) read the binary tree.  Returns the number of children; unused refs
// are REF_EMPTY.
template <int W, class CHILD, class BOX>
__device__ __forceinline__ int collapse_w(int j, const CHILD& child, const BOX& box, int refs[W],
                                          bool keep_pairs = false) {
    refs[0] = child(j, 0);
    refs[1] = child(j, 1);
#pragma unroll
    for (int k = 2; k < W; ++k) refs[k] = REF_EMPTY;
    int cnt = 2;
    bool open = true;
    // static indices and selects only, so refs[] stays in registers
#pragma unroll
    for (int step = 2; step < W; ++step) {
        int best = -1, r = 0;
        float best_a = -1.0f;
#pragma unroll
        for (int k = 0; k < W; ++k) {
            // keep_pairs: a node over two leaves stays closed (it becomes a
            // pair leaf) and the slot goes to a larger subtree
            if (k < step && refs[k] >= 0 && !(keep_pairs && child(refs[k], 0) < 0 && child(refs[k], 1) < 0)) {
                float b[6];
                box(refs[k], b);
                float a = half_area(b);
                if (a > best_a) { best_a = a; best = k; r = refs[k]; }
            }
        }
        open = open && best >= 0;
        if (!open) continue;
        const int c0 = child(r, 0), c1 = child(r, 1);
#pragma unroll
        for (int k = W - 1; k >= 0; --k) {
            const int kk = k > 0 ? k - 1 : 0;
            refs[k] = (k > best + 1 && k <= step) ? refs[kk] : k == best ? c0 : k == best + 1 ? c1 : refs[k];
        }
        cnt = step + 1;
    }
    return cnt;
}

template <class CHILD, class BOX>
__device__ __forceinline__ int collapse4(int j, const CHILD& child, const BOX& box, int refs[4],
                                         bool keep_pairs = false) {
    return collapse_w<4>(j, child, box, refs, keep_pairs);
}

// Wide node of the interval-packet traversal (W = 8: 256 B, W = 16: 512 B):
// child k's record is the 32 B at k: (lo.x, lo.y, lo.z, hi.x), (hi.y, hi.z,
// ref, -), so lane k of a warp fetches its child with two 128-bit loads and
// lanes 0..W-1 read the node's W x 32 B.
constexpr int NODE8_F4 = 16;  // float4 per BVH8 node
__device__ __forceinline__ void write_childw(float4* nodesw, int W, int g, int k, const float b[6], int ref) {
    float4* p = nodesw + 2 * (size_t)W * g + 2 * k;
    p[0] = make_float4(b[0], b[1], b[2], b[3]);
    p[1] = make_float4(b[4], b[5], __int_as_float(ref), 0.0f);
}
__device__ __forceinline__ void write_child8(float4* nodesw, int g, int k, const float b[6], int ref) {
    write_childw(nodesw, 8, g, k, b, ref);
}

// Writes BVH4 node g: boxes b[k][6] (lo xyz, hi xyz) and global refs.
__device__ __forceinline__ void write_node4(float4* nodes, int g, const float b[4][6], const int ref[4], int cnt) {
    float4* p = nodes + 8 * (size_t)g;
    p[0] = make_float4(b[0][0], b[1][0], b[2][0], b[3][0]);
    p[1] = make_float4(b[0][3], b[1][3], b[2][3], b[3][3]);
    p[2] = make_float4(b[0][1], b[1][1], b[2][1], b[3][1]);
    p[3] = make_float4(b[0][4], b[1][4], b[2][4], b[3][4]);
    p[4] = make_float4(b[0][2], b[1][2], b[2][2], b[3][2]);
    p[5] = make_float4(b[0][5], b[1][5], b[2][5], b[3][5]);
    p[6] = make_float4(__int_as_float(ref[0]), __int_as_float(ref[1]), __int_as_float(ref[2]), __int_as_float(ref[3]));
    p[7] = make_float4(__int_as_float(cnt), 0.0f, 0.0f, 0.0f);
}

}  // namespace agr

// Host launch wrappers implemented in the .cu files (all async on `stream`).
namespace agr {
// One BLAS (asset part) of a batched BLAS build: all kernels of the build
// run once over the concatenation of the batch's faces (face g of the batch
// belongs to the segment whose [off, off + n_faces) contains it).
struct BlasSeg {
    const float* verts;    // device [V][3] (the asset's vertices)
    const int* faces;      // device [F][3], asset-local vertex ids (this part's faces)
    const int* face_ids;   // device [F]: asset-local face id of each face, or null (identity)
    int n_verts, n_faces;
    int off;               // first batch face of this asset (set by blas_build_batch)
    int node_base;         // global index of this asset's first node (F - 1 reserved, >= 1)
    int leaf_base;         // global leaf-record index of this asset's first leaf (F reserved)
    BlasInfo* info;        // this part's BlasInfo (device)
};
struct BlasBatchArgs {
    float4* nodes;         // global BVH4 node array
    float4* nodesw;        // global wide node array (compacted like the BVH4; root at node_base), or null
    int wide_w;            // its width: 8, 16 or 32
    float4* bnodes;        // global binary BLAS node array (debug export)
    float4* tris;          // global tri record array
    float* triv;           // global exact-vertex array
    uint32_t* dbg_morton;  // optional: sorted codes at leaf_base + p (device) or null
    int trbvh_rounds;      // treelet-restructuring passes after the LBVH (0 = plain LBVH)
    int opt_collapse;      // 1: SAH-optimal BVH8 collapse (creation-time builds); 0: greedy (mesh updates)
    void* h_stage;         // optional pinned host staging for the segment / sort-block tables
    size_t h_stage_bytes;
    cudaEvent_t stage_free;  // recorded after each upload from h_stage
};
// Builds the BLAS of every asset in h_segs[0, n) (host array; `off` is
// filled in) in one set of launches.  `scratch` must hold
// blas_scratch_bytes(sum of n_faces, n) bytes.  Async on `stream`.
size_t blas_scratch_bytes(int64_t total_faces, int n_segs, int wide_w);
// Pinned host staging a batch of n_segs segments over total_faces faces needs
// (BlasBatchArgs.h_stage).
size_t blas_stage_bytes(int64_t total_faces, int n_segs);
cudaError_t blas_build_batch(BlasSeg* h_segs, int n_segs, const BlasBatchArgs& a, void* scratch,
                             cudaStream_t stream);

struct TlasArgs {
    float4* nodes;            // global node array (TLAS part written)
    float4* nodesw;           // global wide node array (TLAS part written), or null
    int wide_w;               // its width: 8, 16 or 32
    float4* irec;             // [n_items][4] written
    float* item_box;          // [n_items][6] written
    const float* inst_T;      // [n_inst][12]
    const int* item_inst;     // [n_items] instance of each item
    const int* item_part;     // [n_items] part (BLAS) of each item
    const BlasInfo* parts;    // [n_parts]
    const int* item_off;      // [n_envs+1] items of env e: [item_off[e], item_off[e+1])
    const int* tlas_off;      // [n_envs] offset of the env's first node within the TLAS part
    int nb_blas;              // number of BLAS nodes (TLAS node j of env e is global
                              // node nb_blas + tlas_off[e] + j)
    int* tlas_child;          // [2 * n_tlas_nodes] local child refs (>=0 node, <0 ~local item)
    int* tlas_item_parent;    // [n_items] local parent (internal node) of each item leaf
    int* tlas_node_parent;    // [n_tlas_nodes] local parent of each internal node
    int* tlas_depth;          // [n_envs] depth of each env's TLAS (written by build)
    int* tlas_refs4;          // [n_tlas_nodes][4] the BVH4 collapse of each node (binary refs), kept by refits
    int* tlas_refsw;          // [n_tlas_nodes][wide_w] the wide collapse, kept by refits (or null)
    int n_envs;
    int max_n;                // max items in one env (sizes shared memory)
    int builder;              // 0: LBVH (Morton + Karras), 1: binned SAH (default)
};
cudaError_t items_update(const TlasArgs& a, int n_items, cudaStream_t stream);
cudaError_t tlas_build(const TlasArgs& a, bool rebuild, cudaStream_t stream);

// Casts.  Model: 0 rays, 1 pinhole, 2 beams.
struct CastArgs {
    SceneView sv;
    int model;
    int kind;             // pinhole: 0 depth, 1 range
    int W, H;             // pinhole image / beams (W = K columns, H = C channels)
    float fx, fy, cx, cy;
    double inv_fx64, inv_fy64;  // 1 / (double)fx, 1 / (double)fy (FP64 raygen)
    const float* beams;   // [C][K][3]
    const float* poses;   // [n_envs][S][12]
    int S;
    const float* orig;    // rays [n_envs][R][3]
    const float* dir;
    int R;
    float max_range;
    float* out_dist;
    int* out_seg;
    int* out_face;
    float* out_normal;    // [..][3]
    float* out_bary;      // [..][2]
    float* out_point;     // [..][3]
    int* out_valid;       // stereo shadow mask (1 valid, 0 shadowed)
    float* out_annot;     // [..][annot_k] interpolated vertex annotations
    float stereo[3];      // second sensor origin in the sensor frame
    float stereo_eps;     // self-hit guard (metres)
    int env_begin, env_end;  // envs cast by this launch (chunking)
    int out_env_base;        // outputs are indexed from this env (0: global indexing)
    unsigned long long* counters;  // optional [8]
    int exact;
    int packet;           // 1: warp-packet traversal for pinhole / beams tiles
    int wide;             // 1: interval packets over the BVH8 copy (sv.nodesw)
    // filled by cast_launch: n / d = (n * m) >> s for n < 2^31 (tile decode
    // of tiles_img, tiles_x, S without integer division)
    unsigned div_m[3];
    int div_s[3];
};
cudaError_t cast_launch(const CastArgs& a, cudaStream_t stream);

cudaError_t checksum_launch(const float* dist, const int* seg, const int* face,
                            int64_t elems_per_env, int n_envs, unsigned long long* sums,
                            cudaStream_t stream);
}  // namespace agr
