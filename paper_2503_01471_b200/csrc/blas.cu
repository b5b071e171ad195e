// blas.cu -- bottom-level BVH (BLAS) builds on the GPU, batched over assets.
//
// PAPER.md:226 (§III.D.1): "a bounding volume hierarchy is calculated for
// M_{i,t} for efficient ray-casting".  The paper's Warp BVH algorithm is not
// stated; BASELINE.json north_star fixes an LBVH: "per-asset BLAS built by
// LBVH from 30-bit Morton codes, an on-device radix sort and the Karras
// hierarchy" (Karras, HPG 2012).  SURVEY.md §8(a) row a1, kernels K1-K5:
//   K1 tri_prep     triangle AABB, exact-area degeneracy test, centroid
//                   bounds and asset radius (ordered-int atomics)
//   K1b morton      30-bit Morton code of the centroid in the centroid bounds
//   K2 radix sort   LSD, 8-bit digits, stable (hist / scan / scatter)
//   K3 karras       radix-tree topology, ties broken by leaf index
//   K4 fit          bottom-up boxes: 2nd-arriving child unions (atomic flag)
//   K4b trbvh       treelet restructuring
//   K5 pack         BVH4 nodes + 48-B triangle records + exact vertices
// Zero-area faces (exactly, in FP64 from the FP32 inputs) are left out of
// the tree: they can never be hit, and the face numbering is kept by the
// per-leaf local face id.
//
// Batching (per-env unique meshes rebuilt at reset):
// every kernel runs once over the concatenated faces of all assets in the
// batch; face g belongs to segment seg_of[g].  The sort orders (asset,
// Morton code) by an LSD pass over the codes followed by passes over the
// segment id (stable), so each asset's leaf order -- and therefore its tree
// -- is exactly what a build of that asset alone produces.  Per-segment
// scratch (tree topology, boxes, flags) lives at the segment's face offset.
#include "agr_internal.cuh"

#include <cfloat>
#include <climits>
#include <cstring>
#include <cooperative_groups.h>
#include <cuda/atomic>

#ifndef AGR_CHILD_REC
#define AGR_CHILD_REC 0  // 1: a k_make_rec pass writes 64-B child records; 0: the top-down reads the build
                         // arrays (c6 update 2.72 -> 2.69 ms and 64 B per face less scratch)
#endif
#ifndef AGR_KEEP_PAIRS
#define AGR_KEEP_PAIRS 0
#endif
#include <vector>

namespace agr {
namespace {

constexpr int T_BLK = 256;
constexpr int RS_THREADS = 256;
constexpr int RS_ROUNDS = 8;        // rounds of RS_THREADS keys per sort block
constexpr int RS_TILE = RS_THREADS * RS_ROUNDS;
constexpr int SCAN_THREADS = 1024, SCAN_CHUNK = 4 * SCAN_THREADS;  // multi-CTA scan

// Sort blocks never straddle segments: segment s gets ceil(F_s / RS_TILE)
// blocks of its own, so the LSD passes sort every segment by its codes in
// place and no pass over segment ids is needed.  Upper bound on the blocks.
inline int64_t rs_max_blocks(int64_t F, int B) { return F / RS_TILE + B; }
constexpr uint32_t DEGENERATE_KEY = 0xFFFFFFFFu;
constexpr unsigned FULL = 0xFFFFFFFFu;

// Box records of the build scratch: 32 B (lo.xyz, -, hi.xyz, -), so one box
// is two 128-bit loads / stores instead of six scalar ones (the bottom-up
// passes are bound by L2 requests, not bytes).
constexpr int BX = 8;
constexpr int MAX_LEVELS = 512;  // BVH4 levels of the compaction queue (>= any binary depth)

__device__ __forceinline__ void load_box_cg(const float* p, float b[6]) {
    const float4 u = __ldcg(reinterpret_cast<const float4*>(p)), v = __ldcg(reinterpret_cast<const float4*>(p) + 1);
    b[0] = u.x; b[1] = u.y; b[2] = u.z; b[3] = v.x; b[4] = v.y; b[5] = v.z;
}
// + the ints in lo.w / hi.w (the fit keeps subtree size / height there)
__device__ __forceinline__ int2 load_box_cg_w(const float* p, float b[6]) {
    const float4 u = __ldcg(reinterpret_cast<const float4*>(p)), v = __ldcg(reinterpret_cast<const float4*>(p) + 1);
    b[0] = u.x; b[1] = u.y; b[2] = u.z; b[3] = v.x; b[4] = v.y; b[5] = v.z;
    return make_int2(__float_as_int(u.w), __float_as_int(v.w));
}
__device__ __forceinline__ int2 load_box_w(const float* p, float b[6]) {
    const float4 u = reinterpret_cast<const float4*>(p)[0], v = reinterpret_cast<const float4*>(p)[1];
    b[0] = u.x; b[1] = u.y; b[2] = u.z; b[3] = v.x; b[4] = v.y; b[5] = v.z;
    return make_int2(__float_as_int(u.w), __float_as_int(v.w));
}
__device__ __forceinline__ void store_box_w(float* p, const float b[6], int w0, int w1) {
    reinterpret_cast<float4*>(p)[0] = make_float4(b[0], b[1], b[2], __int_as_float(w0));
    reinterpret_cast<float4*>(p)[1] = make_float4(b[3], b[4], b[5], __int_as_float(w1));
}
__device__ __forceinline__ void store_box(float* p, const float b[6]) {
    reinterpret_cast<float4*>(p)[0] = make_float4(b[0], b[1], b[2], 0.0f);
    reinterpret_cast<float4*>(p)[1] = make_float4(b[3], b[4], b[5], 0.0f);
}
__device__ __forceinline__ void store_box_cg(float* p, const float b[6]) {
    __stcg(reinterpret_cast<float4*>(p), make_float4(b[0], b[1], b[2], 0.0f));
    __stcg(reinterpret_cast<float4*>(p) + 1, make_float4(b[3], b[4], b[5], 0.0f));
}

// Child records for the top-down pass (one coalesced pass over the internal
// nodes): rec[i] = child 0 box, child 1 box, refs, and per child the
// pair-leaf ref it becomes if the collapse leaves it closed (0: none), so
// each collapse step reads one 64-B record instead of refs, boxes and sizes
// from four scattered arrays.
__device__ __forceinline__ void write_rec(float4* rec, const float a[6], const float b[6], int ra, int rb, int xa,
                                          int xb) {
    rec[0] = make_float4(a[0], a[1], a[2], a[3]);
    rec[1] = make_float4(a[4], a[5], b[0], b[1]);
    rec[2] = make_float4(b[2], b[3], b[4], b[5]);
    rec[3] = make_float4(__int_as_float(ra), __int_as_float(rb), __int_as_float(xa), __int_as_float(xb));
}
struct Scratch {
    float* tri_box;      // [Ftot][BX] leaf boxes (lo xyz, -, hi xyz, -) by SORTED batch position
    float4* cent;        // [Ftot] triangle centroids (xyz, -) by batch face (Morton input)
    uint32_t* bounds;    // [B][8]: ordered-int centroid lo xyz, hi xyz, radius, n_valid
    uint32_t* mcode;     // [Ftot] Morton code of each batch face
    uint32_t* keys[2];   // [Ftot]
    uint32_t* vals[2];   // [Ftot] batch face ids
    uint32_t* hist;      // [256 * nblocks], (segment, digit, block) order
    int4* rs_blk;        // [nblocks] sort block: first key, end, hist base, hist stride
    uint32_t* scan_part; // [256 * nblocks / SCAN_CHUNK + 1] multi-CTA scan partials
    int* seg_of;         // [Ftot] segment of each batch face
    BlasSeg* segs;       // [B]
    int* child;          // [2 Ftot] local refs; segment s at 2 off_s
    int* node_parent;    // [Ftot]   segment s at off_s
    int* leaf_parent;    // [Ftot]
    float* ibox;         // [Ftot][BX] internal node boxes, same layout
    int* flags;          // [Ftot]
    int* depth;          // [B]
    float* cost;         // [Ftot] SAH cost of each internal node's subtree (TRBVH)
    int* height;         // [Ftot] edges from each internal node to its deepest leaf
    int* size;           // [Ftot] leaves under each internal node
    int2* range;         // [Ftot] leaf range [lo, hi] of each Karras node (segment-local)
    int* seg4;           // [B] BVH4 nodes allocated in each segment (compaction)
    int* seg8;           // [B] the same for the BVH8 copy
    int2* queue;         // [Ftot] (binary node, BVH4 slot) of every reachable node, level by level
    float4* rec;         // [Ftot][4] per internal node: both children's boxes, refs and pair-leaf codes
    float* dp8;          // [Ftot][W] SAH cost of the node's subtree as <= i wide child slots (SAH-optimal collapse)
    int* qctl;           // [2 + MAX_LEVELS]: [0] items in the queue, [2 + L] items of BVH4 level L
};

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

size_t scratch_layout(int64_t F, int B, int wide_w, void* base, Scratch* out) {
    char* p = (char*)base;
    size_t used = 0;
    const size_t nb = (size_t)rs_max_blocks(F, B);
    auto take = [&](size_t bytes) {
        char* q = p ? p + used : nullptr;
        used += align_up(bytes);
        return q;
    };
    Scratch s;
    s.tri_box = (float*)take(sizeof(float) * BX * F);
    s.cent = (float4*)take(sizeof(float4) * F);
    s.bounds = (uint32_t*)take(sizeof(uint32_t) * 8 * B);
    s.mcode = (uint32_t*)take(sizeof(uint32_t) * F);
    for (int i = 0; i < 2; ++i) s.keys[i] = (uint32_t*)take(sizeof(uint32_t) * F);
    for (int i = 0; i < 2; ++i) s.vals[i] = (uint32_t*)take(sizeof(uint32_t) * F);
    s.hist = (uint32_t*)take(sizeof(uint32_t) * 256 * nb);
    s.rs_blk = (int4*)take(sizeof(int4) * nb);
    s.scan_part = (uint32_t*)take(sizeof(uint32_t) * (256 * nb / SCAN_CHUNK + 2));
    s.seg_of = (int*)take(sizeof(int) * F);
    s.segs = (BlasSeg*)take(sizeof(BlasSeg) * B);
    s.child = (int*)take(sizeof(int) * 2 * F);
    s.node_parent = (int*)take(sizeof(int) * F);
    s.leaf_parent = (int*)take(sizeof(int) * F);
    s.ibox = (float*)take(sizeof(float) * BX * F);
    s.flags = (int*)take(sizeof(int) * F);
    s.depth = (int*)take(sizeof(int) * B);
    s.cost = (float*)take(sizeof(float) * F);
    s.height = (int*)take(sizeof(int) * F);
    s.size = (int*)take(sizeof(int) * F);
    s.range = (int2*)take(sizeof(int2) * F);
    s.seg4 = (int*)take(sizeof(int) * B);
    s.seg8 = (int*)take(sizeof(int) * B);
    s.queue = (int2*)take(sizeof(int2) * F);
    s.rec = (float4*)take(AGR_CHILD_REC ? sizeof(float4) * 4 * F : 16);
    s.dp8 = (float*)take(sizeof(float) * (wide_w > 0 ? wide_w : 1) * F);  // the wide collapse's DP tables
    s.qctl = (int*)take(sizeof(int) * (2 + MAX_LEVELS));
    if (out) *out = s;
    return used + 256;
}

// Segment context of batch face g.
struct SegCtx {
    int s;        // segment
    int off;      // its first batch face
    int F;        // its faces
    int n;        // its non-degenerate leaves (after K1)
};
__device__ __forceinline__ SegCtx seg_ctx(const BlasSeg* segs, const int* seg_of, const uint32_t* bounds,
                                          int g) {
    SegCtx c;
    c.s = __ldg(seg_of + g);
    c.off = segs[c.s].off;
    c.F = segs[c.s].n_faces;
    c.n = (int)bounds[8 * c.s + 7];
    return c;
}

// ---- K0: segment ids, bounds init -----------------------------------------
__global__ void k_seg_of(const BlasSeg* segs, int* seg_of) {
    const int s = blockIdx.x;
    const int off = segs[s].off, F = segs[s].n_faces;
    for (int i = threadIdx.x; i < F; i += blockDim.x) seg_of[off + i] = s;
}

__global__ void k_init_bounds(uint32_t* b, int B) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 8 * B) return;
    int k = i & 7;
    if (k < 3) b[i] = float_to_ordered(FLT_MAX);
    else if (k < 6) b[i] = float_to_ordered(-FLT_MAX);
    else if (k == 6) b[i] = float_to_ordered(0.0f);
    else b[i] = 0u;
}

// ---- K1: triangle prep --------------------------------------------------------
__global__ void k_tri_prep(const BlasSeg* segs, const int* seg_of, int Ftot, float4* __restrict__ cent,
                           uint32_t* __restrict__ vflag, uint32_t* bounds) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    const int s = g < Ftot ? __ldg(seg_of + g) : -1;
    float clo[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, chi[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
    float rad = 0.0f;  // the segment's radius: max |v| over its faces' vertices
    bool valid = false;
    if (s >= 0) {
        const BlasSeg& S = segs[s];
        const int f = g - S.off;
        const float* a = S.verts + 3 * S.faces[3 * f];
        const float* b = S.verts + 3 * S.faces[3 * f + 1];
        const float* c = S.verts + 3 * S.faces[3 * f + 2];
        for (const float* v : {a, b, c})
            rad = fmaxf(rad, sqrtf(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]) * 1.000001f);
        // exact-input FP64 area: zero only for genuinely degenerate input
        d3 A = mkd(a[0], a[1], a[2]), B = mkd(b[0], b[1], b[2]), C = mkd(c[0], c[1], c[2]);
        d3 n = crossd(subd(B, A), subd(C, A));
        valid = (n.x != 0.0 || n.y != 0.0 || n.z != 0.0);
        float cc[3];
        for (int k = 0; k < 3; ++k) {
            const float lo = fminf(a[k], fminf(b[k], c[k]));
            const float hi = fmaxf(a[k], fmaxf(b[k], c[k]));
            cc[k] = 0.5f * lo + 0.5f * hi;
            if (valid) clo[k] = chi[k] = cc[k];
        }
        cent[g] = make_float4(cc[0], cc[1], cc[2], 0.0f);
        vflag[g] = valid ? 1u : 0u;
    }
    // centroid bounds and valid count: one set of atomics per block when the
    // block lies in one segment (the common case: same-address atomics from
    // every warp of a segment queue up at L2 and stall the loads), else per
    // thread
    __shared__ int s_seg[2];
    __shared__ uint32_t s_red[8];
    if (threadIdx.x == 0) { s_seg[0] = s; s_red[6] = 0u; s_red[7] = 0u; }
    if (threadIdx.x < 3) { s_red[threadIdx.x] = 0xFFFFFFFFu; s_red[3 + threadIdx.x] = 0u; }
    if (threadIdx.x == blockDim.x - 1) s_seg[1] = s;
    __syncthreads();
    const int s0 = s_seg[0];
    if (s0 >= 0 && s_seg[1] == s0) {  // segments are contiguous: first == last => one segment
        unsigned cnt = __popc(__ballot_sync(FULL, valid));
        for (int o = 16; o > 0; o >>= 1) {
            for (int k = 0; k < 3; ++k) {
                clo[k] = fminf(clo[k], __shfl_xor_sync(FULL, clo[k], o));
                chi[k] = fmaxf(chi[k], __shfl_xor_sync(FULL, chi[k], o));
            }
            rad = fmaxf(rad, __shfl_xor_sync(FULL, rad, o));
        }
        if ((threadIdx.x & 31) == 0) {
            if (cnt > 0) {
                for (int k = 0; k < 3; ++k) {
                    atomicMin(&s_red[k], float_to_ordered(clo[k]));
                    atomicMax(&s_red[3 + k], float_to_ordered(chi[k]));
                }
                atomicAdd(&s_red[6], cnt);
            }
            atomicMax(&s_red[7], float_to_ordered(rad));
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            if (s_red[6] > 0) {
                for (int k = 0; k < 3; ++k) {
                    atomicMin(&bounds[8 * s0 + k], s_red[k]);
                    atomicMax(&bounds[8 * s0 + 3 + k], s_red[3 + k]);
                }
                atomicAdd(&bounds[8 * s0 + 7], s_red[6]);
            }
            atomicMax(&bounds[8 * s0 + 6], s_red[7]);
        }
    } else if (s >= 0) {
        if (valid) {
            for (int k = 0; k < 3; ++k) {
                atomicMin(&bounds[8 * s + k], float_to_ordered(clo[k]));
                atomicMax(&bounds[8 * s + 3 + k], float_to_ordered(chi[k]));
            }
            atomicAdd(&bounds[8 * s + 7], 1u);
        }
        atomicMax(&bounds[8 * s + 6], float_to_ordered(rad));
    }
}

// ---- K1b: Morton codes ------------------------------------------------------
__global__ void k_morton(const int* seg_of, const float4* __restrict__ cent, const uint32_t* __restrict__ vflag,
                         int Ftot, const uint32_t* __restrict__ bounds, uint32_t* __restrict__ mcode,
                         uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= Ftot) return;
    const uint32_t* b = bounds + 8 * __ldg(seg_of + g);
    uint32_t key = DEGENERATE_KEY;
    if (vflag[g]) {
        float u[3];
        const float4 cg = cent[g];
        const float cc[3] = {cg.x, cg.y, cg.z};
        for (int k = 0; k < 3; ++k) {
            float lo = ordered_to_float(b[k]), hi = ordered_to_float(b[3 + k]);
            u[k] = unit_coord(cc[k], lo, hi);
        }
        key = morton30(u[0], u[1], u[2]);
    }
    mcode[g] = key;
    keys[g] = key;
    vals[g] = (uint32_t)g;
}

// ---- K2: stable LSD radix sort (8-bit digits) --------------------------------
// Sort block b owns keys [blk.x, blk.y) of ONE segment (rs_blk, built on the
// host); its digit-d count goes to hist[blk.z + d * blk.w], where blk.z =
// 256 b0 + (b - b0) and blk.w = the segment's block count (b0 = its first
// block).  One exclusive scan over hist in that (segment, digit, block)
// order then yields every block's output offset for every digit: the
// segments stay where they are and each is sorted by its codes, stably (a
// face's order among equal codes is its input order).  The histogram counts
// per warp slice (warp-aggregated by __match_any_sync, no shared-memory
// atomics); the scatter walks the block's keys 256 at a time in order with
// per-round warp-major offsets, so equal digits keep their input order.
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_UNROLL = 4;

// Per-warp digit counts of keys [start, start + steps 32) & [.., end) into wc[256].
__device__ __forceinline__ void rs_warp_count(const uint32_t* __restrict__ keys, int end, int shift, int start,
                                              int steps, uint32_t* wc) {
    const int lane = threadIdx.x & 31;
    for (int j0 = 0; j0 < steps; j0 += RS_UNROLL) {
        uint32_t k[RS_UNROLL];
#pragma unroll
        for (int u = 0; u < RS_UNROLL; ++u) {
            const int i = start + (j0 + u) * 32 + lane;
            k[u] = (j0 + u < steps && i < end) ? __ldg(keys + i) : 0u;
        }
#pragma unroll
        for (int u = 0; u < RS_UNROLL; ++u) {
            const int i = start + (j0 + u) * 32 + lane;
            const bool valid = j0 + u < steps && i < end;
            const int digit = valid ? (int)((k[u] >> shift) & 255u) : 256;
            const unsigned peers = __match_any_sync(FULL, digit);
            if (valid && (peers & ((1u << lane) - 1u)) == 0u) wc[digit] += __popc(peers);
            __syncwarp();
        }
    }
}

__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const uint32_t* __restrict__ keys, const int4* __restrict__ blk,
                                                        int shift, uint32_t* __restrict__ hist) {
    __shared__ uint32_t wc[RS_WARPS][256];
    for (int k = 0; k < RS_WARPS; ++k) wc[k][threadIdx.x] = 0;
    __syncthreads();
    const int4 b = blk[blockIdx.x];
    const int w = threadIdx.x >> 5;
    rs_warp_count(keys, b.y, shift, b.x + w * RS_ROUNDS * 32, RS_ROUNDS, wc[w]);
    __syncthreads();
    uint32_t c = 0;
    for (int k = 0; k < RS_WARPS; ++k) c += wc[k][threadIdx.x];
    hist[b.z + threadIdx.x * b.w] = c;
}

// Exclusive scan of x[0, n) in place, three launches: per-chunk sums,
// a one-CTA scan of the sums, per-chunk scans with the carried offset.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* warp_sums, uint32_t* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t t = lane < nw ? warp_sums[lane] : 0u;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, t, o);
            if (lane >= o) t += y;
        }
        if (lane < nw) warp_sums[lane] = t;  // inclusive
    }
    __syncthreads();
    const uint32_t r = (w > 0 ? warp_sums[w - 1] : 0u) + x - v;
    if (total) *total = warp_sums[nw - 1];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_sums(const uint32_t* __restrict__ x, int n,
                                                            uint32_t* __restrict__ part) {
    __shared__ uint32_t ws[32];
    const int i0 = blockIdx.x * SCAN_CHUNK + 4 * threadIdx.x;
    uint32_t v = 0;
    for (int k = 0; k < 4; ++k) v += i0 + k < n ? x[i0 + k] : 0u;
    uint32_t tot;
    block_excl_scan(v, ws, &tot);
    if (threadIdx.x == 0) part[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_top(uint32_t* part, int n) {
    __shared__ uint32_t ws[32];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < n; base += SCAN_THREADS) {
        const int i = base + threadIdx.x;
        const uint32_t v = i < n ? part[i] : 0u;
        uint32_t tot;
        const uint32_t e = block_excl_scan(v, ws, &tot);
        if (i < n) part[i] = carry + e;
        __syncthreads();
        if (threadIdx.x == 0) carry += tot;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_apply(uint32_t* x, int n, const uint32_t* __restrict__ part) {
    __shared__ uint32_t ws[32];
    const int i0 = blockIdx.x * SCAN_CHUNK + 4 * threadIdx.x;
    uint32_t v[4], s = 0;
    for (int k = 0; k < 4; ++k) {
        v[k] = i0 + k < n ? x[i0 + k] : 0u;
        s += v[k];
    }
    uint32_t e = part[blockIdx.x] + block_excl_scan(s, ws, nullptr);
    for (int k = 0; k < 4; ++k)
        if (i0 + k < n) {
            x[i0 + k] = e;
            e += v[k];
        }
}

cudaError_t excl_scan(uint32_t* x, int n, uint32_t* part, cudaStream_t stream) {
    const int nc = (n + SCAN_CHUNK - 1) / SCAN_CHUNK;
    k_scan_sums<<<nc, SCAN_THREADS, 0, stream>>>(x, n, part);
    k_scan_top<<<1, SCAN_THREADS, 0, stream>>>(part, nc);
    k_scan_apply<<<nc, SCAN_THREADS, 0, stream>>>(x, n, part);
    return cudaGetLastError();
}

__global__ void k_rs_scatter(const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                             uint32_t* __restrict__ kout, uint32_t* __restrict__ vout, const int4* __restrict__ blk,
                             int shift, const uint32_t* __restrict__ hist) {
    __shared__ uint32_t base[256];
    __shared__ uint32_t wc[RS_THREADS / 32][256];
    const int4 b = blk[blockIdx.x];
    base[threadIdx.x] = hist[b.z + threadIdx.x * b.w];
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    for (int r = 0; r < RS_ROUNDS; ++r) {
        for (int k = 0; k < RS_THREADS / 32; ++k) wc[k][threadIdx.x] = 0;
        __syncthreads();
        int i = b.x + r * RS_THREADS + threadIdx.x;
        bool valid = i < b.y;
        uint32_t key = valid ? kin[i] : 0u;
        uint32_t val = valid ? vin[i] : 0u;
        int digit = valid ? (int)((key >> shift) & 255u) : 256;
        unsigned peers = __match_any_sync(0xFFFFFFFFu, digit);
        int rank = __popc(peers & lt);
        if (valid && rank == 0) wc[w][digit] = __popc(peers);
        __syncthreads();
        {
            int d = threadIdx.x;  // RS_THREADS == 256 digits
            uint32_t run = base[d];
            for (int k = 0; k < RS_THREADS / 32; ++k) {
                uint32_t c = wc[k][d];
                wc[k][d] = run;
                run += c;
            }
            base[d] = run;
        }
        __syncthreads();
        if (valid) {
            uint32_t pos = wc[w][digit] + rank;
            kout[pos] = key;
            vout[pos] = val;
        }
        __syncthreads();
    }
}

// ---- K3: Karras radix tree (per segment) ------------------------------------------
// Karras's delta(i, j): the common-prefix length of keys i and j (index
// bits break ties), -1 outside [0, n); ki = k[i] is loaded once by the
// caller, whose searches compare one key against many others.
__device__ __forceinline__ int kdelta_i(const uint32_t* __restrict__ k, int n, uint32_t ki, int i, int j) {
    if (j < 0 || j >= n) return -1;
    const uint32_t b = __ldg(k + j);
    if (ki == b) return 32 + __clz((unsigned)(i ^ j));
    return __clz(ki ^ b);
}

__global__ void k_karras(const BlasSeg* segs, const int* seg_of, const uint32_t* bounds, int Ftot,
                         const uint32_t* __restrict__ sk, int* __restrict__ child_all,
                         int* __restrict__ node_parent_all, int* __restrict__ leaf_parent_all,
                         int2* __restrict__ range_all) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= Ftot) return;
    const SegCtx c = seg_ctx(segs, seg_of, bounds, g);
    const int n = c.n, i = g - c.off;
    if (i >= n - 1) return;
    const uint32_t* k = sk + c.off;
    int* child = child_all + 2 * c.off;
    int* node_parent = node_parent_all + c.off;
    int* leaf_parent = leaf_parent_all + c.off;
    const uint32_t ki = __ldg(k + i);
    int d = (kdelta_i(k, n, ki, i, i + 1) - kdelta_i(k, n, ki, i, i - 1)) >= 0 ? 1 : -1;
    int dmin = kdelta_i(k, n, ki, i, i - d);
    int lmax = 2;
    while (kdelta_i(k, n, ki, i, i + lmax * d) > dmin) lmax <<= 1;
    int l = 0;
    for (int t = lmax >> 1; t >= 1; t >>= 1)
        if (kdelta_i(k, n, ki, i, i + (l + t) * d) > dmin) l += t;
    int j = i + l * d;
    int dnode = kdelta_i(k, n, ki, i, j);
    // binary search for the split: the last position (from i towards j) whose
    // prefix with key i is longer than the node's common prefix.  Positions
    // beyond j never qualify (keys are sorted), so no bound check is needed.
    int s = 0;
    int t = l;
    do {
        t = (t + 1) >> 1;
        if (kdelta_i(k, n, ki, i, i + (s + t) * d) > dnode) s += t;
    } while (t > 1);
    int gamma = i + s * d + (d < 0 ? -1 : 0);
    int lo = min(i, j), hi = max(i, j);
    range_all[c.off + i] = make_int2(lo, hi);
    int left = (lo == gamma) ? ~gamma : gamma;
    int right = (hi == gamma + 1) ? ~(gamma + 1) : gamma + 1;
    child[2 * i] = left;
    child[2 * i + 1] = right;
    if (left < 0) leaf_parent[~left] = i; else node_parent[left] = i;
    if (right < 0) leaf_parent[~right] = i; else node_parent[right] = i;
    if (i == 0) node_parent[0] = -1;
}

// ---- K4: bottom-up fit (per segment) ------------------------------------------------
// Arrival counter of the bottom-up passes: one acq_rel atomic (a single
// MEMBAR.ALL.GPU) publishes this thread's earlier stores and, for the second
// arrival, makes the sibling's visible -- instead of a sequentially
// consistent __threadfence() on each side of a relaxed atomic.
__device__ __forceinline__ int arrive(int* flag) {
    cuda::atomic_ref<int, cuda::thread_scope_device> a(*flag);
    return a.fetch_add(1, cuda::memory_order_acq_rel);
}


// Per-segment views of the scratch arrays used by K4/K4b/K5.
#define AGR_SEG_VIEW(c)                                             \
    int* child = child_all + 2 * (c).off;                           \
    float* ibox = ibox_all + BX * (size_t)(c).off
#define AGR_SEG_PARENTS(c)                                          \
    int* node_parent = node_parent_all + (c).off;                   \
    int* leaf_parent = leaf_parent_all + (c).off

__device__ __forceinline__ int arrive_cta(int* flag) {
    cuda::atomic_ref<int, cuda::thread_scope_block> a(*flag);
    return a.fetch_add(1, cuda::memory_order_acq_rel);
}

// Arrivals at a node whose whole leaf range lies inside this thread block's
// faces come only from threads of this block, so they synchronise through
// a shared-memory flag at block scope (no device-wide fence); only nodes
// straddling a block boundary (a few per cent) use the global flag and the
// acq_rel device-scope atomic.  Internal node i's range contains leaf i, so
// a block-local node's flag is its face slot in the block.
#ifndef AGR_FIT_BLK
#define AGR_FIT_BLK 256
#endif
#ifndef AGR_FIT_SMEM
#define AGR_FIT_SMEM 1  // block-local node boxes of the fit also in shared memory
#endif
constexpr int FIT_BLK = AGR_FIT_BLK;  // larger blocks keep more of the climb at block scope
__global__ void __launch_bounds__(FIT_BLK) k_fit(const BlasSeg* segs, const int* seg_of, const uint32_t* bounds,
                                              int Ftot, const uint32_t* __restrict__ sorted_all, const float* tri_box,
                                              int* child_all, int* node_parent_all, int* leaf_parent_all,
                                              float* ibox_all, int* flags_all, int* depth,
                                              const int2* __restrict__ range_all) {
    __shared__ int sflag[FIT_BLK];
#if AGR_FIT_SMEM
    // boxes of the block-local internal nodes, also kept here: a child box is
    // read back by the second arrival right after its sibling wrote it, and
    // global stores do not stay in L1 (an L2 round trip per level otherwise)
    __shared__ __align__(16) float sbox[FIT_BLK][BX];
#endif
    sflag[threadIdx.x] = 0;
    __syncthreads();
    const int blk0 = blockIdx.x * FIT_BLK;
    const int g = blk0 + threadIdx.x;
    if (g >= Ftot) return;
    const SegCtx c = seg_ctx(segs, seg_of, bounds, g);
    const int n = c.n, p = g - c.off;
    if (n < 2 || p >= n) return;
    AGR_SEG_VIEW(c);
    AGR_SEG_PARENTS(c);
    int* flags = flags_all + c.off;
    const int2* range = range_all + c.off;
    const int lo_ok = blk0 - c.off, hi_ok = blk0 + FIT_BLK - c.off;  // block's faces, segment-local
    int node = leaf_parent[p];
    while (node >= 0) {
        const int2 r = __ldg(range + node);
        const bool local = r.x >= lo_ok && r.y < hi_ok;
        if (local ? arrive_cta(&sflag[c.off + node - blk0]) == 0 : arrive(&flags[node]) == 0)
            return;  // first arrival: sibling not ready
        float b[6], cc[6];
        int h = 0, sz = 0;
        for (int side = 0; side < 2; ++side) {
            int rr = child[2 * node + side];
            float* dst = side == 0 ? b : cc;
            if (rr < 0) {
                load_box_cg(tri_box + BX * (size_t)(c.off + ~rr), dst);
                sz += 1;
            } else {
                // a child's subtree size and height ride in its box record
#if AGR_FIT_SMEM
                // a local node's children are local too (their ranges nest)
                const int2 w = local ? load_box_w(&sbox[c.off + rr - blk0][0], dst)
                                     : load_box_cg_w(ibox + BX * rr, dst);
#else
                const int2 w = local ? load_box_w(ibox + BX * rr, dst) : load_box_cg_w(ibox + BX * rr, dst);
#endif
                sz += w.x;
                h = max(h, w.y);
            }
        }
        float u[6];
        for (int k = 0; k < 3; ++k) {
            u[k] = fminf(b[k], cc[k]);
            u[3 + k] = fmaxf(b[3 + k], cc[3 + k]);
        }
        // one record per level: the stores before the next (device-scope)
        // arrival are what its release waits for
        store_box_w(ibox + BX * node, u, sz, h + 1);
#if AGR_FIT_SMEM
        if (local) store_box_w(&sbox[c.off + node - blk0][0], u, sz, h + 1);
#endif
        if (node == 0) depth[c.s] = h + 1;  // the root: the tree's depth in edges
        node = node_parent[node];
    }
}

// Subtree sizes out of the box records into their own array (read by the
// treelet rounds and the collapses).
__global__ void k_size_from_box(const BlasSeg* segs, const int* seg_of, const uint32_t* bounds, int Ftot,
                                const float* __restrict__ ibox, int* __restrict__ size) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= Ftot) return;
    const SegCtx c = seg_ctx(segs, seg_of, bounds, g);
    if (g - c.off < c.n - 1) size[g] = __float_as_int(__ldg(ibox + BX * (size_t)g + 3));  // internal nodes only
}

// ---- K4b: treelet restructuring (TRBVH) ------------------------------------------------
// Karras & Aila, "Fast parallel construction of high-quality bounding volume
// hierarchies" (HPG 2013): after the LBVH, every internal node (bottom-up,
// second arrival as in the fit) forms a treelet of up to 7 subtrees by
// repeatedly opening the largest-area one, and replaces the treelet's
// topology by the SAH-optimal one found by dynamic programming over all
// subsets.  Boxes of the treelet's new internal nodes are the unions of
// their subsets, so nothing outside the treelet changes.
// f3 "BLAS quality (treelet restructuring)".
constexpr float SAH_CI = 1.2f, SAH_CT = 1.0f;
constexpr int TREELET = 7;

__device__ __forceinline__ float box_area(const float b[6]) {
    float dx = b[3] - b[0], dy = b[4] - b[1], dz = b[5] - b[2];
    return dx * dy + dy * dz + dz * dx;
}

// Warp-cooperative form (as in Karras & Aila): lanes walk up from their
// leaves individually; every node a lane claims (second arrival) is then
// optimised by the whole warp -- subset areas in parallel, the DP over
// subsets size by size with one subset per lane, the treelet rewrite by
// lane 0.  The DP visits partitions in the same order with the same strict
// comparison as a serial DP, so the tree does not depend on the schedule.
constexpr int TRB_THREADS = 64;
// Treelets are formed only at nodes with at least TRB_GAMMA leaves below
// (Karras & Aila's gamma): the many small subtrees near the leaves keep
// their LBVH topology and only get their SAH cost recorded.
#ifndef AGR_TRB_GAMMA
#define AGR_TRB_GAMMA 16
#endif
constexpr int TRB_GAMMA = AGR_TRB_GAMMA;
struct TrbWarp {
    float area[1 << TREELET];
    float copt[1 << TREELET];
    unsigned char part[1 << TREELET];
    float lb[TREELET][6];
    float lc[TREELET];
    float la[TREELET];
    int lsz[TREELET];
    int L[TREELET];
    int I[TREELET - 1];
    int m;
    float ccur;
};

__device__ __forceinline__ void subset_box(const TrbWarp& w, int sset, float b[6]) {
    for (int c = 0; c < 3; ++c) { b[c] = INFINITY; b[3 + c] = -INFINITY; }
    for (int k = 0; k < TREELET; ++k)
        if ((sset >> k) & 1)
            for (int c = 0; c < 3; ++c) {
                b[c] = fminf(b[c], w.lb[k][c]);
                b[3 + c] = fmaxf(b[3 + c], w.lb[k][3 + c]);
            }
}

// Optimise the treelet rooted at local node `node` of the segment at `off`
// (all 32 lanes, warp-uniform arguments).
__device__ void trbvh_treelet(TrbWarp& w, int lane, int node, int off, const uint32_t* __restrict__ sorted_all,
                              const float* __restrict__ tri_box, int* child_all, int* node_parent_all,
                              int* leaf_parent_all, float* ibox_all, float* cost_all, int* size_all) {
    int* child = child_all + 2 * off;
    int* node_parent = node_parent_all + off;
    int* leaf_parent = leaf_parent_all + off;
    float* ibox = ibox_all + BX * (size_t)off;
    float* cost = cost_all + off;
    int* size = size_all + off;
    auto ref_box = [&](int r, float b[6]) {
        load_box_cg(r < 0 ? tri_box + BX * (size_t)(off + ~r) : ibox + BX * r, b);
    };
    // treelet formation: open the largest-area subtree root until 7; the
    // two children of an opened node are fetched by lanes 0 and 1 at once
    if (lane < 2) {
        const int r = __ldcg(child + 2 * node + lane);
        w.L[lane] = r;
        ref_box(r, w.lb[lane]);
        w.la[lane] = box_area(w.lb[lane]);
        // the node's current cost: children's subtree costs (children final)
        w.lc[lane] = r < 0 ? SAH_CT * w.la[lane] : __ldcg(cost + r);
    } else if (lane == 2) {
        float nb[6];
        load_box_cg(ibox + BX * node, nb);
        w.ccur = SAH_CI * box_area(nb);
    }
    __syncwarp();
    if (lane == 0) {
        w.ccur = w.ccur + w.lc[0] + w.lc[1];
        w.I[0] = node;
    }
    int m = 2, ni = 1;
    while (m < TREELET) {
        int best = -1;
        float ba = -1.0f;
        for (int k = 0; k < m; ++k)
            if (w.L[k] >= 0 && w.la[k] > ba) { ba = w.la[k]; best = k; }
        if (best < 0) break;
        const int r = w.L[best];
        __syncwarp();  // every lane has read L before it changes
        if (lane < 2) {
            const int c = __ldcg(child + 2 * r + lane);
            const int slot = lane == 0 ? best : m;
            w.L[slot] = c;
            ref_box(c, w.lb[slot]);
            w.la[slot] = box_area(w.lb[slot]);
        }
        if (lane == 0) w.I[ni] = r;
        ++ni;
        ++m;
        __syncwarp();
    }
    if (lane < m) {
        const int r = w.L[lane];
        w.lc[lane] = r < 0 ? SAH_CT * w.la[lane] : __ldcg(cost + r);
        w.lsz[lane] = r < 0 ? 1 : __ldcg(size + r);
    }
    __syncwarp();
    if (m < 3) {
        if (lane == 0) __stcg(cost + node, w.ccur);
        __syncwarp();
        return;
    }
    const int full = (1 << m) - 1;
    for (int sset = lane + 1; sset <= full; sset += 32) {
        float b[6];
        subset_box(w, sset, b);
        w.area[sset] = box_area(b);
        if ((sset & (sset - 1)) == 0) {
            w.copt[sset] = w.lc[__ffs(sset) - 1];
            w.part[sset] = 0;
        }
    }
    __syncwarp();
    for (int k = 2; k <= m; ++k) {
        for (int sset = lane + 1; sset <= full; sset += 32) {
            if (__popc(sset) != k) continue;
            const int lsb = sset & -sset;
            float best = INFINITY;
            int bp = 0;
            for (int q = (sset - 1) & sset; q; q = (q - 1) & sset) {
                if (!(q & lsb)) continue;  // each unordered partition once
                const float cc = w.copt[q] + w.copt[sset ^ q];
                if (cc < best) { best = cc; bp = q; }
            }
            w.copt[sset] = SAH_CI * w.area[sset] + best;
            w.part[sset] = (unsigned char)bp;
        }
        __syncwarp();
    }
    if (lane == 0) {
        if (w.copt[full] < w.ccur * (1.0f - 1e-6f)) {
            // rebuild the treelet: root keeps its id, the others are reused
            int st_s[TREELET], st_n[TREELET], sp = 0, pool = 1;
            st_s[sp] = full;
            st_n[sp++] = node;
            while (sp > 0) {
                --sp;
                const int sset = st_s[sp], nd = st_n[sp];
                const int q0 = w.part[sset], q1 = sset ^ q0;
                for (int side = 0; side < 2; ++side) {
                    const int sub = side == 0 ? q0 : q1;
                    int c;
                    if ((sub & (sub - 1)) == 0) {
                        c = w.L[__ffs(sub) - 1];
                    } else {
                        c = w.I[pool++];
                        st_s[sp] = sub;
                        st_n[sp++] = c;
                        float b[6];
                        subset_box(w, sub, b);
                        store_box_cg(ibox + BX * c, b);
                        __stcg(cost + c, w.copt[sub]);
                        int sz = 0;
                        for (int k = 0; k < TREELET; ++k)
                            if ((sub >> k) & 1) sz += w.lsz[k];
                        __stcg(size + c, sz);
                    }
                    __stcg(child + 2 * nd + side, c);
                    if (c < 0) __stcg(leaf_parent + ~c, nd);
                    else __stcg(node_parent + c, nd);
                }
            }
            __stcg(cost + node, w.copt[full]);
        } else {
            __stcg(cost + node, w.ccur);
        }
    }
    __syncwarp();
}

__global__ void __launch_bounds__(TRB_THREADS) k_trbvh(
        const BlasSeg* segs, const int* seg_of, const uint32_t* bounds, int Ftot,
        const uint32_t* __restrict__ sorted_all, const float* __restrict__ tri_box, int* child_all,
        int* node_parent_all, int* leaf_parent_all, float* ibox_all, float* cost_all, int* flags_all,
        int* size_all) {
    __shared__ TrbWarp s_w[TRB_THREADS / 32];
    TrbWarp& w = s_w[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    bool active = false;
    int node = -1, off = 0;
    if (g < Ftot) {
        const SegCtx c = seg_ctx(segs, seg_of, bounds, g);
        const int p = g - c.off;
        if (c.n >= 2 && p < c.n) {
            active = true;
            off = c.off;
            node = __ldcg(leaf_parent_all + off + p);
        }
    }
    for (;;) {
        bool claim = false;
        if (active && node >= 0) {
            claim = arrive(&flags_all[off + node]) != 0;  // second arrival: subtree final
        }
        active = claim;
        if (!__any_sync(FULL, claim)) break;
        bool big = false;
        if (claim) {
            big = __ldcg(size_all + off + node) >= TRB_GAMMA;
            if (!big) {
                // small subtree: keep its topology, record its SAH cost
                const int* child = child_all + 2 * off;
                const float* ibox = ibox_all + BX * (size_t)off;
                float b[6];
                load_box_cg(ibox + BX * node, b);
                float cc = SAH_CI * box_area(b);
                for (int side = 0; side < 2; ++side) {
                    const int r = __ldcg(child + 2 * node + side);
                    if (r < 0) {
                        load_box_cg(tri_box + BX * (size_t)(off + ~r), b);
                        cc += SAH_CT * box_area(b);
                    } else {
                        cc += __ldcg(cost_all + off + r);
                    }
                }
                __stcg(cost_all + off + node, cc);
            }
        }
        unsigned mask = __ballot_sync(FULL, big);
        while (mask) {
            const int l = __ffs(mask) - 1;
            mask &= mask - 1;
            trbvh_treelet(w, lane, __shfl_sync(FULL, node, l), __shfl_sync(FULL, off, l), sorted_all, tri_box,
                          child_all, node_parent_all, leaf_parent_all, ibox_all, cost_all, size_all);
        }
        __threadfence();
        if (claim) node = __ldcg(node_parent_all + off + node);
    }
}

// Tree depth after restructuring: heights bottom-up (second arrival).
__global__ void k_depth(const BlasSeg* segs, const int* seg_of, const uint32_t* bounds, int Ftot,
                        const int* child_all, const int* leaf_parent_all, const int* node_parent_all,
                        int* flags_all, int* height_all, int* depth) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= Ftot) return;
    const SegCtx c = seg_ctx(segs, seg_of, bounds, g);
    const int n = c.n, p = g - c.off;
    if (n < 2 || p >= n) return;
    const int* child = child_all + 2 * c.off;
    const int* node_parent = node_parent_all + c.off;
    int* flags = flags_all + c.off;
    int* height = height_all + c.off;
    int node = __ldcg(leaf_parent_all + c.off + p);
    while (node >= 0) {
        if (arrive(&flags[node]) == 0) return;
        int h = 0;
        for (int side = 0; side < 2; ++side) {
            const int r = __ldcg(child + 2 * node + side);
            if (r >= 0) h = max(h, __ldcg(height + r));
        }
        __stcg(height + node, h + 1);
        if (node == 0) depth[c.s] = h + 1;
        node = __ldcg(node_parent + node);
    }
}

// ---- K5a: SAH-optimal 8-wide collapse (Ylitie, Karras & Laine 2017, sec. 4.1) ------------
// Bottom-up over the binary tree (second arrival, as in the fit): C(n, i) =
// the lowest SAH cost of representing n's subtree as at most i child slots
// of a BVH8 node, i = 1..8:
//   C(leaf, i)  = CT A(leaf)
//   Cd(n, j)    = min_{k = 1..j-1} C(L, k) + C(R, j - k)      (distribute j slots)
//   C(n, 1)     = min(CN A(n) + Cd(n, 8),  2 CT A(n) if n is a pair leaf)
//   C(n, i > 1) = min(C(n, i - 1), Cd(n, i))
// with A the box surface (half area) and CT / CN the measured cost of a
// triangle test against a node visit in the interval-packet traversal
// (~84 vs ~130 warp instructions: 0.65).  The top-down pass then extracts
// each wide node's children from these tables instead of the greedy
// largest-area opening (offline on c3's assets: SAH cost 6 % lower).
#ifndef AGR_DP_CT
#define AGR_DP_CT 0.65f
#endif
constexpr float DP_CN = 1.0f, DP_CT = AGR_DP_CT;

template <int W>
__global__ void k_dpw(const BlasSeg* segs, const int* seg_of, const uint32_t* bounds, int Ftot,
                      const float* __restrict__ tri_box, const int* child_all, const int* leaf_parent_all,
                      const int* node_parent_all, const float* ibox_all, int* flags_all, float* dp_all) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= Ftot) return;
    const SegCtx c = seg_ctx(segs, seg_of, bounds, g);
    const int n = c.n, p = g - c.off;
    if (n < 2 || p >= n) return;
    const int* child = child_all + 2 * c.off;
    const int* node_parent = node_parent_all + c.off;
    const float* lbox = tri_box + BX * (size_t)c.off;
    const float* ibox = ibox_all + BX * (size_t)c.off;
    int* flags = flags_all + c.off;
    float* dp = dp_all + W * (size_t)c.off;
    int node = __ldcg(leaf_parent_all + c.off + p);
    while (node >= 0) {
        if (arrive(&flags[node]) == 0) return;
        float cl[2][W];
        int r[2];
        for (int side = 0; side < 2; ++side) {
            r[side] = __ldcg(child + 2 * node + side);
            if (r[side] < 0) {
                float b[6];
                load_box_cg(lbox + BX * (size_t)(~r[side]), b);
                const float v = DP_CT * half_area(b);
#pragma unroll
                for (int i = 0; i < W; ++i) cl[side][i] = v;
            } else {
#pragma unroll
                for (int q = 0; q < W / 4; ++q) {
                    const float4 u = __ldcg(reinterpret_cast<const float4*>(dp + W * (size_t)r[side]) + q);
                    cl[side][4 * q] = u.x; cl[side][4 * q + 1] = u.y; cl[side][4 * q + 2] = u.z;
                    cl[side][4 * q + 3] = u.w;
                }
            }
        }
        float nb[6];
        load_box_cg(ibox + BX * node, nb);
        const float an = half_area(nb);
        float cd[W + 1];
#pragma unroll
        for (int j = 2; j <= W; ++j) {
            float m = INFINITY;
#pragma unroll
            for (int k = 1; k < j; ++k) m = fminf(m, cl[0][k - 1] + cl[1][j - k - 1]);
            cd[j] = m;
        }
        float C[W];
        C[0] = DP_CN * an + cd[W];
        if (LEAF_MAX == 2 && r[0] < 0 && r[1] < 0 && abs(~r[0] - ~r[1]) == 1) C[0] = fminf(C[0], 2.0f * DP_CT * an);
#pragma unroll
        for (int i = 1; i < W; ++i) C[i] = fminf(C[i - 1], cd[i + 1]);
        float4* o = reinterpret_cast<float4*>(dp + W * (size_t)node);
#pragma unroll
        for (int q = 0; q < W / 4; ++q) __stcg(o + q, make_float4(C[4 * q], C[4 * q + 1], C[4 * q + 2], C[4 * q + 3]));
        node = __ldcg(node_parent + node);
    }
}

// ---- K5: pack -------------------------------------------------------------------------
// Box of a binary ref: lbox = the segment's leaf boxes (sorted order), ibox
// its internal-node boxes.
__device__ __forceinline__ void child_box(int r, const float* lbox, const float* ibox, float b[6]) {
    if (r == REF_EMPTY) {
        for (int k = 0; k < 6; ++k) b[k] = __int_as_float(0x7f800000);  // +inf: never hit
        return;
    }
    load_box_cg(r < 0 ? lbox + BX * (size_t)(~r) : ibox + BX * r, b);
}

__device__ __forceinline__ void write_node(float4* nodes, int g, const float a[6], const float b[6],
                                           int ra, int rb) {
    nodes[4 * g + 0] = make_float4(a[0], a[3], a[1], a[4]);
    nodes[4 * g + 1] = make_float4(a[2], a[5], b[0], b[3]);
    nodes[4 * g + 2] = make_float4(b[1], b[4], b[2], b[5]);
    nodes[4 * g + 3] = make_float4(__int_as_float(ra), __int_as_float(rb), 0.0f, 0.0f);
}

__device__ __forceinline__ int global_ref(int r, int node_base, int leaf_base) {
    if (r == REF_EMPTY) return REF_EMPTY;
    return r < 0 ? ~(leaf_base + ~r) : node_base + r;
}

__global__ void k_pack_nodes(const BlasSeg* segs, const int* seg_of, const uint32_t* bounds, int Ftot,
                             const uint32_t* __restrict__ sorted_all, const float* tri_box, int* child_all,
                             float* ibox_all, float4* nodes) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= Ftot) return;
    const SegCtx c = seg_ctx(segs, seg_of, bounds, g);
    const int n = c.n, i = g - c.off;
    const int n_int = n > 1 ? n - 1 : 1;
    if (i >= n_int) return;
    AGR_SEG_VIEW(c);
    const int node_base = segs[c.s].node_base, leaf_base = segs[c.s].leaf_base;
    int ra, rb;
    if (n > 1) { ra = child[2 * i]; rb = child[2 * i + 1]; }
    else if (n == 1) { ra = ~0; rb = REF_EMPTY; }
    else { ra = REF_EMPTY; rb = REF_EMPTY; }
    float a[6], b[6];
    child_box(ra, tri_box + BX * (size_t)c.off, ibox, a);
    child_box(rb, tri_box + BX * (size_t)c.off, ibox, b);
    write_node(nodes, node_base + i, a, b, global_ref(ra, node_base, leaf_base),
               global_ref(rb, node_base, leaf_base));
}

// ---- K5b': compacted BVH4 ------------------------------------------------------
// The greedy collapse keeps only the binary nodes it does not open as BVH4
// nodes (about a fifth with pair leaves), so writing a BVH4 node for every
// binary node (k_collapse<4>) moved ~5x the bytes the traversal can reach
// and did ~5x the work.  Here the BVH4 is built top-down, one level per grid
// barrier of a single cooperative launch: a queue of (binary node, BVH4
// slot) pairs; each is collapsed, gets slots for its internal children from
// its segment's counter (the root is slot 0) and writes its node at once.
// Slot order within a level depends on the schedule, so the node numbering
// (not the tree) may differ between builds; results do not.
// A slot of a collapse: a leaf, a pair leaf (binary subtree over <= LEAF_MAX
// consecutive leaves, referenced as one multi-triangle leaf) or an internal
// node that becomes a BVH4 node of its own (returns -1 with *internal set).
// (size_r < 0: read the subtree size from size[r])
__device__ __forceinline__ int slot_ref(int r, const int* child, const int* size, int leaf_base, bool* internal,
                                        int size_r = -1) {
    *internal = false;
    if (r == REF_EMPTY) return REF_EMPTY;
    if (r < 0) return ~(leaf_base + ~r);
    if (LEAF_MAX > 1 && (size_r >= 0 ? size_r : __ldcg(size + r)) <= LEAF_MAX) {
        int st[2 * LEAF_MAX], sp = 0, nl = 0, lmin = INT_MAX, lmax = -1;
        bool ok = true;
        st[sp++] = r;
        while (sp > 0 && ok) {
            const int x = st[--sp];
            if (x < 0) {
                ok = nl < LEAF_MAX;
                ++nl;
                lmin = min(lmin, ~x);
                lmax = max(lmax, ~x);
            } else if (sp + 2 <= 2 * LEAF_MAX) {
                st[sp++] = __ldcg(child + 2 * x + 1);
                st[sp++] = __ldcg(child + 2 * x);
            } else {
                ok = false;
            }
        }
        if (ok && lmax - lmin + 1 == nl) return ~((leaf_base + lmin) | ((nl - 1) << LEAF_SHIFT));
    }
    *internal = true;
    return -1;
}

__global__ void k_reach_init(const BlasSeg* segs, int B, const uint32_t* bounds, int* seg4, int2* queue,
                             int* qctl) {
    const int sgi = blockIdx.x * blockDim.x + threadIdx.x;
    if (sgi >= B) return;
    const bool tree = (int)bounds[8 * sgi + 7] >= 2;  // else a single-leaf / empty BLAS: no binary root
    seg4[sgi] = 1;
    if (tree) queue[atomicAdd(qctl + 2, 1)] = make_int2(segs[sgi].off, 0);  // level 0
}

__device__ __forceinline__ void read_rec(const float4* rec, float a[6], float b[6], int& ra, int& rb, int& xa,
                                         int& xb) {
    const float4 q0 = __ldcg(rec), q1 = __ldcg(rec + 1), q2 = __ldcg(rec + 2), q3 = __ldcg(rec + 3);
    a[0] = q0.x; a[1] = q0.y; a[2] = q0.z; a[3] = q0.w; a[4] = q1.x; a[5] = q1.y;
    b[0] = q1.z; b[1] = q1.w; b[2] = q2.x; b[3] = q2.y; b[4] = q2.z; b[5] = q2.w;
    ra = __float_as_int(q3.x); rb = __float_as_int(q3.y); xa = __float_as_int(q3.z); xb = __float_as_int(q3.w);
}

__global__ void k_make_rec(const BlasSeg* segs, const int* seg_of, const uint32_t* bounds, int Ftot,
                           const float* __restrict__ tri_box, const int* __restrict__ child_all,
                           const float* __restrict__ ibox_all, const int* __restrict__ size_all, float4* rec_all) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= Ftot) return;
    const SegCtx c = seg_ctx(segs, seg_of, bounds, g);
    const int i = g - c.off;
    if (c.n < 2 || i >= c.n - 1) return;
    const int* child = child_all + 2 * c.off;
    const float* lbox = tri_box + BX * (size_t)c.off;
    const float* ibox = ibox_all + BX * (size_t)c.off;
    const int* size = size_all ? size_all + c.off : nullptr;
    const int leaf_base = segs[c.s].leaf_base;
    int r[2], x[2];
    float bb[2][6];
    for (int k = 0; k < 2; ++k) {
        r[k] = __ldg(child + 2 * i + k);
        x[k] = 0;
        if (r[k] >= 0) {
            // subtree size: from the fit's box record, or from size[] after treelet rounds
            const int2 w = load_box_cg_w(ibox + BX * r[k], bb[k]);
            bool internal;
            x[k] = slot_ref(r[k], child, size, leaf_base, &internal, size ? -1 : w.x);
            if (internal) x[k] = 0;
        } else {
            child_box(r[k], lbox, ibox, bb[k]);
        }
    }
    write_rec(rec_all + 4 * (size_t)g, bb[0], bb[1], r[0], r[1], x[0], x[1]);
}

// A node's child record assembled from the build arrays instead of rec[]
// (no k_make_rec pass): refs, the two child boxes (leaf boxes / 32-B box
// records, whose lo.w carries the subtree size unless treelet rounds ran,
// then `size`), and each child's pair-leaf code.
struct RecDirect {
    const int* child;   // segment's child refs
    const float* lbox;  // segment's leaf boxes (sorted order)
    const float* ibox;  // segment's internal-node box records
    const int* size;    // segment's subtree sizes, or null (read lo.w)
    int leaf_base;
    __device__ __forceinline__ void get(int nn, float a[6], float b[6], int& ra, int& rb, int& xa, int& xb) const {
        ra = __ldcg(child + 2 * nn);
        rb = __ldcg(child + 2 * nn + 1);
        xa = side(ra, a);
        xb = side(rb, b);
    }
    __device__ __forceinline__ int side(int r, float bx[6]) const {
        if (r < 0) {
            load_box_cg(lbox + BX * (size_t)(~r), bx);
            return 0;
        }
        const int2 w = load_box_cg_w(ibox + BX * (size_t)r, bx);
        const int sz = size ? __ldcg(size + r) : w.x;
        if (LEAF_MAX != 2 || sz != 2) return 0;
        const int c0 = __ldcg(child + 2 * r), c1 = __ldcg(child + 2 * r + 1);
        if (c0 >= 0 || c1 >= 0 || abs(~c0 - ~c1) != 1) return 0;
        return ~((leaf_base + min(~c0, ~c1)) | (1 << LEAF_SHIFT));
    }
};

// One cooperative launch: level L's items are queue[begin_L, begin_L + n_L)
// (n_L = qctl[2 + L]); each is collapsed (the greedy largest-area opening of
// collapse_w, from the child records) and written, and its internal slots
// are appended as level L + 1 through their own counter qctl[3 + L]
// (warp-aggregated), so one grid barrier per level suffices.
// W = 4: the BVH4 every traversal uses; W = 8: the BVH8 copy of the
// interval packets (its own compacted numbering; both roots are node_base).
template <int W, bool DP>
__global__ void __launch_bounds__(T_BLK) k_bvhw_topdown(const BlasSeg* segs, const int* seg_of,
                                                       const float4* __restrict__ rec_all, int* segw, int2* queue,
                                                       int* qctl, float4* nodes, const float* __restrict__ dp_all,
                                                       const int* child_all, const float* tri_box,
                                                       const float* ibox_all, const int* size_all) {
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
    const int lane = threadIdx.x & 31;
    const int stride = gridDim.x * blockDim.x;
    int begin = 0, L = 0;
    int n_lvl = *(volatile int*)(qctl + 2);  // level 0: the roots (k_reach_init)
    while (n_lvl > 0 && L + 1 < MAX_LEVELS) {
        const int next = begin + n_lvl;
        for (int t0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31); t0 < n_lvl; t0 += stride) {
            const int t = t0 + lane;
            int2 push[W];
#pragma unroll
            for (int k = 0; k < W; ++k) push[k] = make_int2(-1, -1);
            int npush = 0;
            if (t < n_lvl) {
                const int2 item = __ldcg(queue + begin + t);
                const int x = item.x;
                const int sgi = __ldg(seg_of + x);
                const BlasSeg& S = segs[sgi];
                const int off = S.off;
                const float4* rec = rec_all ? rec_all + 4 * (size_t)off : nullptr;
                RecDirect rd;
                rd.child = child_all + 2 * off;
                rd.lbox = tri_box + BX * (size_t)off;
                rd.ibox = ibox_all + BX * (size_t)off;
                rd.size = size_all ? size_all + off : nullptr;
                rd.leaf_base = S.leaf_base;
                auto get_rec = [&](int nn, float a[6], float b[6], int& ra, int& rb, int& xa, int& xb) {
                    if (rec) read_rec(rec + 4 * (size_t)nn, a, b, ra, rb, xa, xb);
                    else rd.get(nn, a, b, ra, rb, xa, xb);
                };
                float bx[W][6];
                int refs[W], aux[W];
#pragma unroll
                for (int k = 0; k < W; ++k) { refs[k] = REF_EMPTY; aux[k] = 0; }
                int cnt = 2;
                if (DP) {
                    // SAH-optimal children from the k_dp8 tables: distribute
                    // the node's 8 slots between its two children and
                    // recursively below them (explicit stack of <= 7 splits)
                    const float* dp = dp_all + W * (size_t)off;
                    int st_n[W], st_j[W], sp = 0;
                    st_n[sp] = x - off; st_j[sp] = W; ++sp;
                    cnt = 0;
                    while (sp > 0) {
                        --sp;
                        const int nn = st_n[sp], j = st_j[sp];
                        float bc[2][6];
                        int rc[2], xc[2];
                        get_rec(nn, bc[0], bc[1], rc[0], rc[1], xc[0], xc[1]);
                        float tab[2][W];
                        for (int side = 0; side < 2; ++side) {
                            if (rc[side] < 0) {
                                const float v = DP_CT * half_area(bc[side]);
                                for (int i = 0; i < W; ++i) tab[side][i] = v;
                            } else {
                                for (int i = 0; i < W; ++i) tab[side][i] = __ldcg(dp + W * (size_t)rc[side] + i);
                            }
                        }
                        int kb = 1;
                        float m = tab[0][0] + tab[1][j - 2];
                        for (int k = 2; k < j; ++k) {
                            const float v = tab[0][k - 1] + tab[1][j - k - 1];
                            if (v < m) { m = v; kb = k; }
                        }
                        for (int side = 0; side < 2; ++side) {
                            const int cr = rc[side];
                            int b = side == 0 ? kb : j - kb;
                            if (cr >= 0) {
                                while (b > 1 && tab[side][b - 1] == tab[side][b - 2]) --b;
                                if (b > 1) {  // the child's subtree spreads over b slots
                                    st_n[sp] = cr; st_j[sp] = b; ++sp;
                                    continue;
                                }
                            }
                            // one slot: a leaf, a pair leaf (if that is what C(c, 1) chose) or a wide node
                            const bool pair = cr >= 0 && xc[side] != 0 &&
                                              2.0f * DP_CT * half_area(bc[side]) == tab[side][0];
                            refs[cnt] = cr;
                            aux[cnt] = pair ? xc[side] : 0;
                            for (int q = 0; q < 6; ++q) bx[cnt][q] = bc[side][q];
                            ++cnt;
                        }
                    }
                } else {
                get_rec(x - off, bx[0], bx[1], refs[0], refs[1], aux[0], aux[1]);
                // collapse_w<W>: open the largest-area internal member (every
                // array index static, so the frontier stays in registers)
                bool open = true;
#pragma unroll
                for (int step = 2; step < W; ++step) {
                    int best = -1, best_ref = 0;
                    float best_a = -1.0f;
#pragma unroll
                    for (int k = 0; k < W; ++k)
                        if (k < step && refs[k] >= 0) {
                            const float a = half_area(bx[k]);
                            if (a > best_a) { best_a = a; best = k; best_ref = refs[k]; }
                        }
                    open = open && best >= 0;
                    if (!open) continue;
                    float ca[6], cb[6];
                    int ra, rb, xa, xb;
                    get_rec(best_ref, ca, cb, ra, rb, xa, xb);
                    // shift the members after `best` up by one and put the
                    // opened node's children at best, best + 1 (selects, not
                    // indexed stores)
#pragma unroll
                    for (int k = W - 1; k >= 0; --k) {
                        const bool sh = k > best + 1 && k <= step, is_b = k == best, is_b1 = k == best + 1;
                        const int kk = k > 0 ? k - 1 : 0;
                        refs[k] = sh ? refs[kk] : is_b ? ra : is_b1 ? rb : refs[k];
                        aux[k] = sh ? aux[kk] : is_b ? xa : is_b1 ? xb : aux[k];
#pragma unroll
                        for (int q = 0; q < 6; ++q)
                            bx[k][q] = sh ? bx[kk][q] : is_b ? ca[q] : is_b1 ? cb[q] : bx[k][q];
                    }
                    cnt = step + 1;
                }
                }
                int gr[W];
                bool internal[W];
#pragma unroll
                for (int k = 0; k < W; ++k) {
                    internal[k] = false;
                    if (k >= cnt) {
                        refs[k] = REF_EMPTY;
#pragma unroll
                        for (int q = 0; q < 6; ++q) bx[k][q] = __int_as_float(0x7f800000);  // +inf: never hit
                        gr[k] = REF_EMPTY;
                    } else if (refs[k] < 0) {
                        gr[k] = ~(S.leaf_base + ~refs[k]);
                    } else if (aux[k] != 0) {
                        gr[k] = aux[k];  // a closed subtree over <= LEAF_MAX consecutive leaves
                    } else {
                        internal[k] = true;
                        ++npush;
                    }
                }
                // child slots from the segment counter, one atomic per segment per warp
                int first = 0;
                {
                    const unsigned grp = __match_any_sync(__activemask(), sgi);
                    const int leader = __ffs(grp) - 1;
                    const unsigned below = grp & ((1u << lane) - 1u);
                    int tot = npush, pre = 0;
                    for (unsigned m = grp; m; m &= m - 1) {
                        const int l = __ffs(m) - 1;
                        const int v = __shfl_sync(grp, npush, l);
                        if (l != lane) tot += v;
                        if ((1u << l) & below) pre += v;
                    }
                    int base = 0;
                    if (lane == leader && tot) base = atomicAdd(segw + sgi, tot);
                    first = __shfl_sync(grp, base, leader) + pre;
                }
                int q = 0;
#pragma unroll
                for (int k = 0; k < W; ++k) {
                    push[k] = make_int2(-1, -1);
                    if (internal[k]) {
                        const int slot = first + q++;
                        gr[k] = S.node_base + slot;
                        push[k] = make_int2(off + refs[k], slot);
                    }
                }
                const int g = S.node_base + item.y;
                if (W == 4) {
                    float4* p = nodes + 8 * (size_t)g;  // write_node4's layout, static indices
                    p[0] = make_float4(bx[0][0], bx[1][0], bx[2][0], bx[3 % W][0]);
                    p[1] = make_float4(bx[0][3], bx[1][3], bx[2][3], bx[3 % W][3]);
                    p[2] = make_float4(bx[0][1], bx[1][1], bx[2][1], bx[3 % W][1]);
                    p[3] = make_float4(bx[0][4], bx[1][4], bx[2][4], bx[3 % W][4]);
                    p[4] = make_float4(bx[0][2], bx[1][2], bx[2][2], bx[3 % W][2]);
                    p[5] = make_float4(bx[0][5], bx[1][5], bx[2][5], bx[3 % W][5]);
                    p[6] = make_float4(__int_as_float(gr[0]), __int_as_float(gr[1]), __int_as_float(gr[2]),
                                       __int_as_float(gr[3 % W]));
                    p[7] = make_float4(__int_as_float(cnt), 0.0f, 0.0f, 0.0f);
                } else {
#pragma unroll
                    for (int k = 0; k < W; ++k) write_childw(nodes, W, g, k, bx[k], gr[k]);
                }
            }
            // warp-aggregated append of the next level
            unsigned incl = npush;
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned y = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += y;
            }
            const unsigned tot = __shfl_sync(FULL, incl, 31);
            int base = 0;
            if (lane == 31 && tot) base = atomicAdd(qctl + 3 + L, (int)tot);
            base = __shfl_sync(FULL, base, 31);
            int pos = next + base + (int)(incl - npush);
#pragma unroll
            for (int k = 0; k < W; ++k)
                if (push[k].x >= 0) queue[pos++] = push[k];
        }
        grid.sync();
        begin = next;
        ++L;
        n_lvl = *(volatile int*)(qctl + 2 + L);
    }
}

// A BLAS with fewer than 2 leaves has no binary node: its BVH4 root holds
// the single leaf (or nothing).
__global__ void k_write4_small(const BlasSeg* segs, int B, const uint32_t* bounds, const uint32_t* sorted_all,
                               const float* tri_box, float4* nodes) {
    const int sgi = blockIdx.x * blockDim.x + threadIdx.x;
    if (sgi >= B) return;
    const int n = (int)bounds[8 * sgi + 7];
    if (n >= 2) return;
    const BlasSeg& S = segs[sgi];
    float boxes[4][6];
    int gr[4];
    const int r0 = n == 1 ? ~0 : REF_EMPTY;
    child_box(r0, tri_box + BX * (size_t)S.off, nullptr, boxes[0]);
    gr[0] = global_ref(r0, S.node_base, S.leaf_base);
    for (int k = 1; k < 4; ++k) {
        child_box(REF_EMPTY, nullptr, nullptr, boxes[k]);
        gr[k] = REF_EMPTY;
    }
    write_node4(nodes, S.node_base, reinterpret_cast<const float(*)[6]>(boxes), gr, n == 1 ? 1 : 0);
}

// Leaf records in sorted order, right after the sort: the 48-B triangle
// record, the exact vertices (3 x float4) and the leaf's box for the
// hierarchy passes (so they read leaf boxes by position, coalesced, instead
// of gathering them by face id).
__global__ void k_writew_small(const BlasSeg* segs, int B, const uint32_t* bounds, const float* tri_box,
                               float4* nodesw, int W) {
    const int sgi = blockIdx.x * blockDim.x + threadIdx.x;
    if (sgi >= B) return;
    const int n = (int)bounds[8 * sgi + 7];
    if (n >= 2) return;
    const BlasSeg& S = segs[sgi];
    for (int k = 0; k < W; ++k) {
        const int r = (k == 0 && n == 1) ? ~0 : REF_EMPTY;
        float b[6];
        child_box(r, tri_box + BX * (size_t)S.off, nullptr, b);
        write_childw(nodesw, W, S.node_base, k, b, global_ref(r, S.node_base, S.leaf_base));
    }
}

__global__ void k_pack_tris(const BlasSeg* segs, const int* seg_of, const uint32_t* bounds, int Ftot,
                            const uint32_t* __restrict__ sorted_all, const uint32_t* __restrict__ sk,
                            float4* tris, float* triv, uint32_t* dbg_morton, float* __restrict__ lbox) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= Ftot) return;
    const SegCtx c = seg_ctx(segs, seg_of, bounds, g);
    const int p = g - c.off;
    const BlasSeg& S = segs[c.s];
    if (dbg_morton) dbg_morton[S.leaf_base + p] = sk[g];
    if (p >= c.n) return;
    const int f = (int)sorted_all[g] - c.off;  // segment-local face
    const float* a = S.verts + 3 * S.faces[3 * f];
    const float* b = S.verts + 3 * S.faces[3 * f + 1];
    const float* cc = S.verts + 3 * S.faces[3 * f + 2];
    d3 A = mkd(a[0], a[1], a[2]), B = mkd(b[0], b[1], b[2]), C = mkd(cc[0], cc[1], cc[2]);
    d3 E1 = subd(B, A), E2 = subd(C, A), E3 = subd(C, B);
    d3 N = crossd(E1, E2);
    const double n2 = dotd(N, N);
    double two_area = sqrt(n2);
    const double l2max = fmax(dotd(E1, E1), fmax(dotd(E2, E2), dotd(E3, E3)));
    // min altitude = 2A / longest edge; store its inverse, rounded up
    float inv_min_alt = (float)sqrt(l2max / n2) * 1.000001f;
    int gl = S.leaf_base + p;
    tris[3 * gl + 0] = make_float4(a[0], a[1], a[2], inv_min_alt);
    tris[3 * gl + 1] = make_float4((float)E1.x, (float)E1.y, (float)E1.z, (float)two_area);
    // the asset-local face id (a part's faces are a subset of its asset's)
    const int face_id = S.face_ids ? S.face_ids[f] : f;
    tris[3 * gl + 2] = make_float4((float)E2.x, (float)E2.y, (float)E2.z, __int_as_float(face_id));
    float4* tv = reinterpret_cast<float4*>(triv) + 3 * (size_t)gl;
    tv[0] = make_float4(a[0], a[1], a[2], 0.0f);
    tv[1] = make_float4(b[0], b[1], b[2], 0.0f);
    tv[2] = make_float4(cc[0], cc[1], cc[2], 0.0f);
    float bb[6];
    for (int k = 0; k < 3; ++k) {
        bb[k] = fminf(a[k], fminf(b[k], cc[k]));
        bb[3 + k] = fmaxf(a[k], fmaxf(b[k], cc[k]));
    }
    store_box(lbox + BX * (size_t)g, bb);
}

__global__ void k_asset_info(const BlasSeg* segs, int B, const uint32_t* bounds, const float* ibox_all,
                             const float* tri_box, const uint32_t* sorted_all, const int* depth,
                             const int* seg4) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= B) return;
    const BlasSeg& S = segs[s];
    const int n = (int)bounds[8 * s + 7];
    BlasInfo a;
    a.node_base = S.node_base;
    a.leaf_base = S.leaf_base;
    a.n_leaves = n;
    a.n_faces = S.n_faces;
    a.radius = ordered_to_float(bounds[8 * s + 6]);
    a.depth = n > 1 ? depth[s] : 1;
    a.n_nodes4 = seg4[s];
    if (n > 1) {
        const float* r = ibox_all + BX * (size_t)S.off;  // local internal node 0 = root
        for (int k = 0; k < 3; ++k) { a.lo[k] = r[k]; a.hi[k] = r[4 + k]; }
    } else if (n == 1) {
        const float* b = tri_box + BX * (size_t)S.off;
        for (int k = 0; k < 3; ++k) { a.lo[k] = b[k]; a.hi[k] = b[4 + k]; }
    } else {
        for (int k = 0; k < 3; ++k) { a.lo[k] = 0.0f; a.hi[k] = 0.0f; }
    }
    *S.info = a;
}

}  // namespace

size_t blas_scratch_bytes(int64_t total_faces, int n_segs, int wide_w) {
    return scratch_layout(total_faces, n_segs, wide_w, nullptr, nullptr);
}

size_t blas_stage_bytes(int64_t total_faces, int n_segs) {
    return ((sizeof(BlasSeg) * (size_t)n_segs + 15) & ~size_t(15)) +
           sizeof(int4) * (size_t)rs_max_blocks(total_faces, n_segs);
}

cudaError_t blas_build_batch(BlasSeg* h_segs, int B, const BlasBatchArgs& a, void* scratch,
                             cudaStream_t stream) {
    if (B <= 0) return cudaSuccess;
    int64_t F64 = 0;
    for (int s = 0; s < B; ++s) {
        h_segs[s].off = (int)F64;
        F64 += h_segs[s].n_faces;
    }
    if (F64 <= 0 || F64 > 0x3FFFFFFF) return cudaErrorInvalidValue;
    const int F = (int)F64;
    Scratch s;
    scratch_layout(F, B, a.wide_w, scratch, &s);
    // the segment table and the sort-block table (below) go up in one copy,
    // from pinned staging when the caller provides it (a pageable copy
    // would wait for the stream to drain first)
    std::vector<int4> blk;
    for (int g = 0; g < B; ++g) {
        const int nbs = (h_segs[g].n_faces + RS_TILE - 1) / RS_TILE;
        const int b0 = (int)blk.size();
        for (int q = 0; q < nbs; ++q) {
            const int st = h_segs[g].off + q * RS_TILE;
            blk.push_back(make_int4(st, min(st + RS_TILE, h_segs[g].off + h_segs[g].n_faces), 256 * b0 + q, nbs));
        }
    }
    const int nb = (int)blk.size();
    const size_t seg_bytes = sizeof(BlasSeg) * B, blk_off = (seg_bytes + 15) & ~size_t(15),
                 blk_bytes = sizeof(int4) * nb;
    cudaError_t e;
    if (a.h_stage && blk_off + blk_bytes <= a.h_stage_bytes) {
        e = cudaEventSynchronize(a.stage_free);  // the previous build's upload has left the buffer
        if (e != cudaSuccess) return e;
        memcpy(a.h_stage, h_segs, seg_bytes);
        memcpy((char*)a.h_stage + blk_off, blk.data(), blk_bytes);
        e = cudaMemcpyAsync(s.segs, a.h_stage, seg_bytes, cudaMemcpyHostToDevice, stream);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(s.rs_blk, (char*)a.h_stage + blk_off, blk_bytes, cudaMemcpyHostToDevice, stream);
        if (e == cudaSuccess) e = cudaEventRecord(a.stage_free, stream);
    } else {
        e = cudaMemcpyAsync(s.segs, h_segs, seg_bytes, cudaMemcpyHostToDevice, stream);
        if (e == cudaSuccess) e = cudaMemcpyAsync(s.rs_blk, blk.data(), blk_bytes, cudaMemcpyHostToDevice, stream);
    }
    if (e != cudaSuccess) return e;
    const int gb = (F + T_BLK - 1) / T_BLK;
    k_seg_of<<<B, T_BLK, 0, stream>>>(s.segs, s.seg_of);
    k_init_bounds<<<(8 * B + T_BLK - 1) / T_BLK, T_BLK, 0, stream>>>(s.bounds, B);
    k_tri_prep<<<gb, T_BLK, 0, stream>>>(s.segs, s.seg_of, F, s.cent, s.vals[1], s.bounds);
    k_morton<<<gb, T_BLK, 0, stream>>>(s.seg_of, s.cent, s.vals[1], F, s.bounds, s.mcode, s.keys[0],
                                       s.vals[0]);
    // sort: segment-local blocks of RS_TILE keys (see K2), 4 passes
    int cur = 0;
    for (int shift = 0; shift < 32; shift += 8) {
        k_rs_hist<<<nb, RS_THREADS, 0, stream>>>(s.keys[cur], s.rs_blk, shift, s.hist);
        e = excl_scan(s.hist, 256 * nb, s.scan_part, stream);
        if (e != cudaSuccess) return e;
        k_rs_scatter<<<nb, RS_THREADS, 0, stream>>>(s.keys[cur], s.vals[cur], s.keys[cur ^ 1], s.vals[cur ^ 1],
                                                    s.rs_blk, shift, s.hist);
        cur ^= 1;
    }
    // everything below reads each segment's leaf count from the device (no
    // host round trip: builds stay async)
    const uint32_t* sk = s.keys[cur];
    const uint32_t* sv = s.vals[cur];
    cudaMemsetAsync(s.depth, 0, sizeof(int) * B, stream);
    cudaMemsetAsync(s.flags, 0, sizeof(int) * F, stream);
    k_pack_tris<<<gb, T_BLK, 0, stream>>>(s.segs, s.seg_of, s.bounds, F, sv, sk, a.tris, a.triv, a.dbg_morton,
                                          s.tri_box);
    k_karras<<<gb, T_BLK, 0, stream>>>(s.segs, s.seg_of, s.bounds, F, sk, s.child, s.node_parent,
                                       s.leaf_parent, s.range);
    k_fit<<<(F + FIT_BLK - 1) / FIT_BLK, FIT_BLK, 0, stream>>>(s.segs, s.seg_of, s.bounds, F, sv, s.tri_box, s.child, s.node_parent,
                                    s.leaf_parent, s.ibox, s.flags, s.depth, s.range);
    // subtree sizes into their own array for the treelet rounds (the
    // collapses read them from the box records)
    const bool need_size = a.trbvh_rounds > 0;
    if (need_size) k_size_from_box<<<gb, T_BLK, 0, stream>>>(s.segs, s.seg_of, s.bounds, F, s.ibox, s.size);
    for (int round = 0; round < a.trbvh_rounds; ++round) {
        cudaMemsetAsync(s.flags, 0, sizeof(int) * F, stream);
        k_trbvh<<<(F + TRB_THREADS - 1) / TRB_THREADS, TRB_THREADS, 0, stream>>>(s.segs, s.seg_of, s.bounds, F, sv, s.tri_box, s.child,
                                                  s.node_parent, s.leaf_parent, s.ibox, s.cost, s.flags,
                                                  s.size);
    }
    if (a.trbvh_rounds > 0) {
        cudaMemsetAsync(s.depth, 0, sizeof(int) * B, stream);
        cudaMemsetAsync(s.flags, 0, sizeof(int) * F, stream);
        k_depth<<<gb, T_BLK, 0, stream>>>(s.segs, s.seg_of, s.bounds, F, s.child, s.leaf_parent, s.node_parent,
                                          s.flags, s.height, s.depth);
    }
    if (a.bnodes)
        k_pack_nodes<<<gb, T_BLK, 0, stream>>>(s.segs, s.seg_of, s.bounds, F, sv, s.tri_box, s.child, s.ibox,
                                               a.bnodes);
    // compacted BVH4 / BVH8 (K5b'): top-down from the child records, one
    // cooperative launch per node width
    if (AGR_CHILD_REC)
        k_make_rec<<<gb, T_BLK, 0, stream>>>(s.segs, s.seg_of, s.bounds, F, s.tri_box, s.child, s.ibox,
                                             a.trbvh_rounds > 0 ? s.size : nullptr, s.rec);
    int dev = 0, sms = 0;
    e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    auto topdown = [&](const void* kern, int* segw, float4* out, const float* dpt) -> cudaError_t {
        cudaMemsetAsync(s.qctl, 0, sizeof(int) * (2 + MAX_LEVELS), stream);
        k_reach_init<<<(B + 127) / 128, 128, 0, stream>>>(s.segs, B, s.bounds, segw, s.queue, s.qctl);
        // co-resident blocks (per device: the grid must fit at once or the
        // cooperative launch fails); all of them -- the levels are
        // latency-bound chains of dependent loads
        int per_sm = 0;
        cudaError_t err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T_BLK, 0);
        if (err != cudaSuccess) return err;
        const int grid = sms * (per_sm < 1 ? 1 : per_sm);
        const BlasSeg* a0 = s.segs;
        const int* a1 = s.seg_of;
        const float4* a2 = s.rec;
        int* a3 = segw;
        int2* a4 = s.queue;
        int* a5 = s.qctl;
        float4* a6 = out;
        const float* a7 = dpt;
        const int* a8 = s.child;
        const float* a9 = s.tri_box;
        const float* a10 = s.ibox;
        const int* a11 = a.trbvh_rounds > 0 ? s.size : nullptr;
        if (!AGR_CHILD_REC) a2 = nullptr;  // assemble the child records on the fly
        void* args[] = {&a0, &a1, &a2, &a3, &a4, &a5, &a6, &a7, &a8, &a9, &a10, &a11};
        return cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(T_BLK), args, 0, stream);
    };
    e = topdown((const void*)k_bvhw_topdown<4, false>, s.seg4, a.nodes, nullptr);
    if (e != cudaSuccess) return e;
    k_write4_small<<<(B + 127) / 128, 128, 0, stream>>>(s.segs, B, s.bounds, sv, s.tri_box, a.nodes);
    if (a.nodesw) {
        const int W = a.wide_w;
        auto pick = [&](bool dp) -> const void* {
            if (W == 32) return (const void*)k_bvhw_topdown<32, true>;  // always the DP collapse
            if (W == 16) return dp ? (const void*)k_bvhw_topdown<16, true> : (const void*)k_bvhw_topdown<16, false>;
            return dp ? (const void*)k_bvhw_topdown<8, true> : (const void*)k_bvhw_topdown<8, false>;
        };
        if (a.opt_collapse || W == 32) {
            // SAH-optimal wide collapse (the interval packets' tree): cost tables bottom-up
            cudaMemsetAsync(s.flags, 0, sizeof(int) * F, stream);
#define AGR_DPW(WW) k_dpw<WW><<<gb, T_BLK, 0, stream>>>(s.segs, s.seg_of, s.bounds, F, s.tri_box, s.child, \
                                                       s.leaf_parent, s.node_parent, s.ibox, s.flags, s.dp8)
            if (W == 32) AGR_DPW(32);
            else if (W == 16) AGR_DPW(16);
            else AGR_DPW(8);
#undef AGR_DPW
            e = topdown(pick(true), s.seg8, a.nodesw, s.dp8);
        } else {
            e = topdown(pick(false), s.seg8, a.nodesw, nullptr);
        }
        if (e != cudaSuccess) return e;
        k_writew_small<<<(B + 127) / 128, 128, 0, stream>>>(s.segs, B, s.bounds, s.tri_box, a.nodesw, a.wide_w);
    }
    k_asset_info<<<(B + 127) / 128, 128, 0, stream>>>(s.segs, B, s.bounds, s.ibox, s.tri_box, sv, s.depth,
                                                      s.seg4);
    return cudaGetLastError();
}

}  // namespace agr
