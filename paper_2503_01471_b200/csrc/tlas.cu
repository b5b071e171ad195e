// tlas.cu -- per-instance ray transforms and the per-env top-level BVH.
//
// PAPER.md:226 (§III.D.1): transformations T_{j,t} are kept for each
// sub-mesh, "the vertices of the mesh are transformed to match the obstacles
// in the simulator at time t" and a BVH is computed over M_{i,t}.  Here the
// vertices are not rewritten: each instance stores the inverse transform so
// rays are moved into object space instead, and each env
// gets a TLAS over its instance boxes (north_star: "a per-env TLAS over
// instances, refit in place when obstacles are re-posed").
//   K6 k_items       per TLAS item (instance, part): inverse affine (FP64 ->
//                    FP32), conservative world box of the part
//   K7 k_tlas        (rebuild) per-env Morton sort + Karras + fit, one CTA/env
//   K8 k_tlas        (refit)   same CTA shape, stored topology, boxes only
#include <algorithm>
#include "agr_internal.cuh"

#include <cfloat>

namespace agr {
namespace {

constexpr int TLAS_THREADS = 256;

__device__ __forceinline__ float inf_f() { return __int_as_float(0x7f800000); }

// ---- K6: per-item record and world box -----------------------------------------
// Item i = part item_part[i] of instance item_inst[i]: the instance's inverse
// transform (recomputed per part: a few FP64 flops) and the world box of the
// part's BLAS.
__global__ void k_items(TlasArgs a, int n_items) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_items) return;
    const int inst = a.item_inst[i];
    const float* T = a.inst_T + 12 * inst;
    const BlasInfo& as = a.parts[a.item_part[i]];
    double A[3][3], b[3];
    for (int r = 0; r < 3; ++r) {
        for (int c = 0; c < 3; ++c) A[r][c] = T[4 * r + c];
        b[r] = T[4 * r + 3];
    }
    double c00 = A[1][1] * A[2][2] - A[1][2] * A[2][1];
    double c01 = A[1][2] * A[2][0] - A[1][0] * A[2][2];
    double c02 = A[1][0] * A[2][1] - A[1][1] * A[2][0];
    double det = A[0][0] * c00 + A[0][1] * c01 + A[0][2] * c02;
    float4* rec = a.irec + 4 * i;
    float* box = a.item_box + 6 * i;
    bool ok = det != 0.0 && isfinite(det) && as.n_leaves > 0;
    if (!ok) {
        // singular transform or an all-degenerate asset: the instance is never
        // hit.  Its box is the empty box (lo = +inf, hi = -inf), the identity
        // of the fit's union, so its TLAS ancestors keep their tight boxes;
        // BVH4 child slots turn it into the never-hit sentinel (slot_box)
        for (int k = 0; k < 3; ++k) { box[k] = inf_f(); box[3 + k] = -inf_f(); }
        for (int k = 0; k < 4; ++k) rec[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        return;
    }
    double inv[3][3];
    double id = 1.0 / det;
    inv[0][0] = c00 * id;
    inv[1][0] = c01 * id;
    inv[2][0] = c02 * id;
    inv[0][1] = (A[0][2] * A[2][1] - A[0][1] * A[2][2]) * id;
    inv[1][1] = (A[0][0] * A[2][2] - A[0][2] * A[2][0]) * id;
    inv[2][1] = (A[0][1] * A[2][0] - A[0][0] * A[2][1]) * id;
    inv[0][2] = (A[0][1] * A[1][2] - A[0][2] * A[1][1]) * id;
    inv[1][2] = (A[0][2] * A[1][0] - A[0][0] * A[1][2]) * id;
    inv[2][2] = (A[0][0] * A[1][1] - A[0][1] * A[1][0]) * id;
    double nrm2 = 0.0, b1 = fabs(b[0]) + fabs(b[1]) + fabs(b[2]);
    for (int r = 0; r < 3; ++r) {
        double binv = -(inv[r][0] * b[0] + inv[r][1] * b[1] + inv[r][2] * b[2]);
        rec[r] = make_float4((float)inv[r][0], (float)inv[r][1], (float)inv[r][2], (float)binv);
        for (int c = 0; c < 3; ++c) nrm2 += inv[r][c] * inv[r][c];
    }
    double nAinv = sqrt(nrm2) * (1.0 + 1e-6);
    double err_off = nAinv * b1 + (double)as.radius;
    rec[3] = make_float4(__int_as_float(as.node_base), (float)nAinv, (float)(err_off * (1.0 + 1e-6)),
                         __int_as_float(inst));
    // conservative world box: the union of the transformed boxes of the
    // BLAS's second BVH4 level (up to 16 boxes; much tighter than the
    // transformed root box under rotation), each in centre/extent form and
    // rounded outward
    double wlo[3] = {INFINITY, INFINITY, INFINITY}, whi[3] = {-INFINITY, -INFINITY, -INFINITY};
    auto add_box = [&](const float* lo, const float* hi) {
        for (int r = 0; r < 3; ++r) {
            double c = b[r], e = 0.0;
            for (int k = 0; k < 3; ++k) {
                double ck = 0.5 * ((double)lo[k] + (double)hi[k]);
                double ek = 0.5 * ((double)hi[k] - (double)lo[k]);
                c += A[r][k] * ck;
                e += fabs(A[r][k]) * ek;
            }
            wlo[r] = fmin(wlo[r], c - e);
            whi[r] = fmax(whi[r], c + e);
        }
    };
    auto node_box = [&](int node, int k, float* lo, float* hi) {
        const float* f = reinterpret_cast<const float*>(a.nodes + 8 * (size_t)node);
        for (int c = 0; c < 3; ++c) {
            lo[c] = f[4 * (2 * c) + k];
            hi[c] = f[4 * (2 * c + 1) + k];
        }
    };
    const int root = as.node_base;
    const int* rrefs = reinterpret_cast<const int*>(a.nodes + 8 * (size_t)root + 6);
    for (int k = 0; k < 4; ++k) {
        const int ref = rrefs[k];
        if (ref == REF_EMPTY) continue;
        float lo[3], hi[3];
        if (ref < 0) {  // a leaf under the root: its own box
            node_box(root, k, lo, hi);
            add_box(lo, hi);
            continue;
        }
        const int* crefs = reinterpret_cast<const int*>(a.nodes + 8 * (size_t)ref + 6);
        for (int j = 0; j < 4; ++j) {
            if (crefs[j] == REF_EMPTY) continue;
            node_box(ref, j, lo, hi);
            add_box(lo, hi);
        }
    }
    for (int r = 0; r < 3; ++r) {
        double lo = wlo[r], hi = whi[r];
        double pad = (fabs(lo) + fabs(hi)) * 1e-12 + 1e-30;
        box[r] = __double2float_rd(lo - pad);
        box[3 + r] = __double2float_ru(hi + pad);
    }
}

// BVH4 child-slot box of a fitted box: an empty box (lo > hi, an instance
// that is never hit or a subtree of them) becomes the +inf sentinel, which
// every slab test misses (an inverted box would pass the min/max slab test).
__device__ __forceinline__ void slot_box(const float* src, float* dst) {
    const bool empty = !(src[0] <= src[3]);
    for (int k = 0; k < 6; ++k) dst[k] = empty ? inf_f() : src[k];
}

// ---- SAH-optimal BVH8 collapse of a TLAS (Ylitie, Karras & Laine 2017) -----------
// As for the BLAS (blas.cu k_dp8): C(n, i) = the lowest SAH cost of n's
// subtree as <= i BVH8 child slots; here a leaf is an instance entry and
// there are no pair leaves, so every leaf's term is the same in every
// collapse and only the node terms decide (TDP_CT 1.5, 3 and 5 give the
// same trees).
// Tables are computed by a fixed-point iteration over all internal nodes
// (each := its formula over the children's current tables, from +inf, until
// nothing changes -- min and + of decreasing values converge in height
// steps), so both the warp and the CTA builders get the same tables.  Envs
// of at most TDP_MAX items use it; larger ones keep the greedy collapse.
#ifndef AGR_TDP_CT
#define AGR_TDP_CT 1.5f
#endif
constexpr float TDP_CN = 1.0f, TDP_CT = AGR_TDP_CT;
constexpr int TDP_MAX = 128;
__device__ __forceinline__ float box_cost_area(const float* b) { return b[0] <= b[3] ? half_area(b) : 0.0f; }

// New table of internal node j from its children's current tables.
constexpr int TDP_STRIDE = 32;  // floats per table row (W <= 32)
template <int W, class CH, class LB, class NB, class TB>
__device__ __forceinline__ void tdp_node(int j, const CH& child, const LB& lbox, const NB& nbox, const TB& tab,
                                         float C[W]) {
    float cl[2][W];
    for (int side = 0; side < 2; ++side) {
        const int r = child(j, side);
        if (r < 0) {
            const float v = TDP_CT * box_cost_area(lbox(~r));
            for (int i = 0; i < W; ++i) cl[side][i] = v;
        } else {
            for (int i = 0; i < W; ++i) cl[side][i] = tab(r)[i];
        }
    }
    float cd[W + 1];
    for (int jj = 2; jj <= W; ++jj) {
        float m = INFINITY;
        for (int k = 1; k < jj; ++k) m = fminf(m, cl[0][k - 1] + cl[1][jj - k - 1]);
        cd[jj] = m;
    }
    C[0] = TDP_CN * box_cost_area(nbox(j)) + cd[W];
    for (int i = 1; i < W; ++i) C[i] = fminf(C[i - 1], cd[i + 1]);
}

// The W-wide children (binary refs, REF_EMPTY padded) of internal node j.
template <int W, class CH, class LB, class TB>
__device__ __forceinline__ void tdp_children(int j, const CH& child, const LB& lbox, const TB& tab, int refs[W]) {
    for (int k = 0; k < W; ++k) refs[k] = REF_EMPTY;
    int st_n[W], st_j[W], sp = 0, cnt = 0;
    st_n[sp] = j; st_j[sp] = W; ++sp;
    while (sp > 0) {
        --sp;
        const int nn = st_n[sp], jj = st_j[sp];
        int rc[2];
        float t[2][W];
        for (int side = 0; side < 2; ++side) {
            rc[side] = child(nn, side);
            if (rc[side] < 0) {
                const float v = TDP_CT * box_cost_area(lbox(~rc[side]));
                for (int i = 0; i < W; ++i) t[side][i] = v;
            } else {
                for (int i = 0; i < W; ++i) t[side][i] = tab(rc[side])[i];
            }
        }
        int kb = 1;
        float m = t[0][0] + t[1][jj - 2];
        for (int k = 2; k < jj; ++k) {
            const float v = t[0][k - 1] + t[1][jj - k - 1];
            if (v < m) { m = v; kb = k; }
        }
        for (int side = 0; side < 2; ++side) {
            int b = side == 0 ? kb : jj - kb;
            if (rc[side] >= 0) {
                while (b > 1 && t[side][b - 1] == t[side][b - 2]) --b;
                if (b > 1) { st_n[sp] = rc[side]; st_j[sp] = b; ++sp; continue; }
            }
            refs[cnt++] = rc[side];
        }
    }
}

// An env of n <= W items fits one wide node: the SAH-optimal collapse is the
// root holding every item (a wide child node would only add its own term),
// so no DP tables are needed.  The items in the DP extraction's order (the
// same stack walk with every internal child expanded).
template <int W, class CH>
__device__ __forceinline__ void all_items(const CH& child, int refs[W]) {
    for (int k = 0; k < W; ++k) refs[k] = REF_EMPTY;
    int st[W], sp = 0, cnt = 0;
    st[sp++] = 0;
    while (sp > 0) {
        const int nn = st[--sp];
        for (int side = 0; side < 2; ++side) {
            const int r = child(nn, side);
            if (r >= 0) st[sp++] = r;
            else refs[cnt++] = r;
        }
    }
}

// Writes the wide node j (W children) from its binary refs.
template <int W, class SRC>
__device__ __forceinline__ void write_wide(const TlasArgs& a, int j, const int refs[W], const SRC& src_of, int i0,
                                           int nodebase) {
    const float EMPTY[6] = {inf_f(), inf_f(), inf_f(), inf_f(), inf_f(), inf_f()};
    for (int c = 0; c < W; ++c) {
        const int r = refs[c];
        float b[6];
        slot_box(r == REF_EMPTY ? EMPTY : src_of(r), b);
        write_childw(a.nodesw, W, nodebase + j, c, b, r == REF_EMPTY ? REF_EMPTY : (r < 0 ? ~(i0 + ~r) : nodebase + r));
    }
}

// ---- K7/K8: per-env TLAS build / refit -----------------------------------------
struct TlasSmem {
    int* task;       // [4 (n-1)] SAH build tasks (start, end, ready, -) by node id
    float* box;      // [n][6] instance boxes (local index)
    float* ibox;     // [n-1][6] internal boxes
    uint64_t* keys;  // [P] Morton<<32 | local index
    int* child;      // [2(n-1)]
    int* nparent;    // [n-1]
    int* lparent;    // [n]
    int* flags;      // [n-1]
};

__device__ __forceinline__ int kdelta64(const uint64_t* k, int n, int i, int j) {
    if (j < 0 || j >= n) return -1;
    return __clzll(k[i] ^ k[j]);  // keys are distinct (local index in the low bits)
}

// ---- K7 (default): binned-SAH top-down build of one env's TLAS in one CTA --------
// Each internal node is one task; warps claim tasks in node-id order from a
// shared-memory queue (a child's id is always larger than its parent's, so a
// waiting warp always waits on a warp that is running).  A task bins the
// centroids of its items into 16 bins per axis, takes the split with the
// lowest SAH cost A_L N_L + A_R N_R, and partitions the items stably.  The
// result is the same binary form as the Karras build (child refs + parents),
// so the fit, the BVH4 collapse and the refit are shared.
#ifndef AGR_SAH_BINS
#define AGR_SAH_BINS 48  // 16 / 32 / 48: c3 9.53 / 9.57 / 9.58 Grays/s (64 exceeds the static shared memory)
#endif
constexpr int SAH_BINS = AGR_SAH_BINS;

__device__ void sah_build_cta(const TlasSmem& s, int n) {
    __shared__ int q_head, next_node;
    __shared__ float bins[TLAS_THREADS / 32][3 * SAH_BINS][7];  // count + box per (axis, bin)
    int* perm = (int*)s.keys;          // [n] item order
    int* tmp = perm + n;               // [n] partition scratch
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const unsigned FULL = 0xFFFFFFFFu;
    for (int i = tid; i < n; i += blockDim.x) perm[i] = i;
    for (int j = tid; j < n - 1; j += blockDim.x) s.task[4 * j + 2] = 0;
    __syncthreads();
    if (tid == 0) {
        q_head = 0;
        next_node = 1;
        s.task[0] = 0;
        s.task[1] = n;
        __threadfence_block();
        ((volatile int*)s.task)[2] = 1;
        s.nparent[0] = -1;
    }
    __syncthreads();
    volatile int* vtask = s.task;
    for (;;) {
        int k = 0;
        if (lane == 0) k = atomicAdd(&q_head, 1);
        k = __shfl_sync(FULL, k, 0);
        if (k >= n - 1) break;
        if (lane == 0)
            while (vtask[4 * k + 2] == 0) __nanosleep(64);  // leave the issue slots to the producer
        __syncwarp();
        __threadfence_block();
        const int start = vtask[4 * k], end = vtask[4 * k + 1];
        const int m = end - start;
        // centroid bounds of the task's items
        float clo[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, chi[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
        for (int i = start + lane; i < end; i += 32) {
            const float* b = s.box + 6 * perm[i];
            for (int c = 0; c < 3; ++c) {
                float x = 0.5f * b[c] + 0.5f * b[3 + c];
                if (isfinite(x)) { clo[c] = fminf(clo[c], x); chi[c] = fmaxf(chi[c], x); }
            }
        }
        for (int o = 16; o > 0; o >>= 1)
            for (int c = 0; c < 3; ++c) {
                clo[c] = fminf(clo[c], __shfl_xor_sync(FULL, clo[c], o));
                chi[c] = fmaxf(chi[c], __shfl_xor_sync(FULL, chi[c], o));
            }
        float scale[3];
        for (int c = 0; c < 3; ++c) {
            const float ext = chi[c] - clo[c];
            scale[c] = ext > 0.0f ? (float)SAH_BINS / ext : 0.0f;
        }
        auto bin_of = [&](int item, int axis) {
            const float* b = s.box + 6 * item;
            const float x = 0.5f * b[axis] + 0.5f * b[3 + axis];
            if (!isfinite(x)) return SAH_BINS - 1;
            const int bi = (int)((x - clo[axis]) * scale[axis]);
            return bi < 0 ? 0 : (bi >= SAH_BINS ? SAH_BINS - 1 : bi);
        };
        // per (axis, bin) count and box: each lane bins its items with
        // shared-memory atomics (boxes as order-preserving integers)
        unsigned* ub = reinterpret_cast<unsigned*>(&bins[w][0][0]);
        for (int pp = lane; pp < 3 * SAH_BINS; pp += 32) {
            ub[7 * pp] = 0u;
            for (int c = 0; c < 3; ++c) {
                ub[7 * pp + 1 + c] = float_to_ordered(FLT_MAX);
                ub[7 * pp + 4 + c] = float_to_ordered(-FLT_MAX);
            }
        }
        __syncwarp();
        for (int i = start + lane; i < end; i += 32) {
            const int it = perm[i];
            const float* b = s.box + 6 * it;
            unsigned lo_o[3], hi_o[3];
            for (int c = 0; c < 3; ++c) {
                lo_o[c] = float_to_ordered(b[c]);
                hi_o[c] = float_to_ordered(b[3 + c]);
            }
            for (int axis = 0; axis < 3; ++axis) {
                unsigned* bb = ub + 7 * (axis * SAH_BINS + bin_of(it, axis));
                atomicAdd(bb, 1u);
                for (int c = 0; c < 3; ++c) {
                    atomicMin(bb + 1 + c, lo_o[c]);
                    atomicMax(bb + 4 + c, hi_o[c]);
                }
            }
        }
        __syncwarp();
        for (int pp = lane; pp < 3 * SAH_BINS; pp += 32) {
            bins[w][pp][0] = (float)ub[7 * pp];
            for (int c = 0; c < 6; ++c) bins[w][pp][1 + c] = ordered_to_float(ub[7 * pp + 1 + c]);
        }
        __syncwarp();
        // SAH sweep per axis (lanes 0..2): split after bin p, p = 0..SAH_BINS-2
        float best_cost = INFINITY;
        int best_split = -1;
        if (lane < 3) {
            const int axis = lane;
            float rcnt[SAH_BINS], rarea[SAH_BINS];
            float l[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, h[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX}, c = 0.0f;
            for (int bi = SAH_BINS - 1; bi >= 1; --bi) {
                const float* bb = bins[w][axis * SAH_BINS + bi];
                c += bb[0];
                for (int q = 0; q < 3; ++q) { l[q] = fminf(l[q], bb[1 + q]); h[q] = fmaxf(h[q], bb[4 + q]); }
                const float bx[6] = {l[0], l[1], l[2], h[0], h[1], h[2]};
                rcnt[bi] = c;
                rarea[bi] = c > 0.0f ? half_area(bx) : 0.0f;
            }
            for (int q = 0; q < 3; ++q) { l[q] = FLT_MAX; h[q] = -FLT_MAX; }
            c = 0.0f;
            for (int bi = 0; bi < SAH_BINS - 1; ++bi) {
                const float* bb = bins[w][axis * SAH_BINS + bi];
                c += bb[0];
                for (int q = 0; q < 3; ++q) { l[q] = fminf(l[q], bb[1 + q]); h[q] = fmaxf(h[q], bb[4 + q]); }
                if (c <= 0.0f || rcnt[bi + 1] <= 0.0f) continue;
                const float bx[6] = {l[0], l[1], l[2], h[0], h[1], h[2]};
                const float cost = half_area(bx) * c + rarea[bi + 1] * rcnt[bi + 1];
                if (cost < best_cost) { best_cost = cost; best_split = axis * SAH_BINS + bi; }
            }
        }
        for (int o = 1; o < 4; o <<= 1) {
            const float oc = __shfl_xor_sync(FULL, best_cost, o);
            const int os = __shfl_xor_sync(FULL, best_split, o);
            if (oc < best_cost || (oc == best_cost && os >= 0 && (best_split < 0 || os < best_split))) {
                best_cost = oc;
                best_split = os;
            }
        }
        best_split = __shfl_sync(FULL, best_split, 0);
        // stable partition of perm[start, end) into tmp
        int mid;
        if (best_split >= 0) {
            const int axis = best_split / SAH_BINS, sb = best_split % SAH_BINS;
            int nl = 0, nr = 0;
            // left side first, then the right side, both in the current order
            for (int base = start; base < end; base += 32) {
                const int i = base + lane;
                const bool valid = i < end;
                const int it = valid ? perm[i] : 0;
                const bool left = valid && bin_of(it, axis) <= sb;
                const unsigned ml = __ballot_sync(FULL, left);
                if (left) tmp[start + nl + __popc(ml & ((1u << lane) - 1u))] = it;
                nl += __popc(ml);
            }
            mid = start + nl;
            for (int base = start; base < end; base += 32) {
                const int i = base + lane;
                const bool valid = i < end;
                const int it = valid ? perm[i] : 0;
                const bool right = valid && bin_of(it, axis) > sb;
                const unsigned mr = __ballot_sync(FULL, right);
                if (right) tmp[mid + nr + __popc(mr & ((1u << lane) - 1u))] = it;
                nr += __popc(mr);
            }
            __syncwarp();
            for (int i = start + lane; i < end; i += 32) perm[i] = tmp[i];
            __syncwarp();
        } else {
            mid = start + m / 2;  // no useful split (coincident centroids): halve
        }
        // children: single items are leaves, ranges are new tasks
        for (int side = 0; side < 2; ++side) {
            const int cs = side == 0 ? start : mid, ce = side == 0 ? mid : end;
            int ref;
            if (ce - cs == 1) {
                ref = ~perm[cs];
                if (lane == 0) s.lparent[perm[cs]] = k;
            } else {
                int id = 0;
                if (lane == 0) {
                    id = atomicAdd(&next_node, 1);
                    s.task[4 * id] = cs;
                    s.task[4 * id + 1] = ce;
                    s.nparent[id] = k;
                    __threadfence_block();
                    vtask[4 * id + 2] = 1;
                }
                ref = __shfl_sync(FULL, id, 0);
            }
            if (lane == 0) s.child[2 * k + side] = ref;
        }
        __syncwarp();
    }
    __syncthreads();
}

template <int W, class CH, class BXF>
__device__ __forceinline__ void cta_wide(const TlasArgs& a, const TlasSmem& s, int n, int i0, int nodebase, int toff,
                                         int tid, int rebuild, float (*dpt)[TDP_STRIDE], const CH& ch, const BXF& bx) {
    if (n <= W) {  // one wide node (the other binary nodes are unreachable and not written)
        if (tid == 0) {
            int refs[W];
            int* keep = a.tlas_refsw + W * (size_t)toff;
            if (rebuild) {
                all_items<W>(ch, refs);
                for (int c = 0; c < W; ++c) keep[c] = refs[c];
            } else {
                for (int c = 0; c < W; ++c) refs[c] = keep[c];
            }
            auto src = [&](int r) { return r < 0 ? s.box + 6 * ~r : s.ibox + 6 * r; };
            write_wide<W>(a, 0, refs, src, i0, nodebase);
        }
        return;
    }
    const bool opt = rebuild && n <= TDP_MAX;
    auto lbf = [&](int i) { return s.box + 6 * i; };
    auto nbf = [&](int r) { return s.ibox + 6 * r; };
    auto tbf = [&](int r) { return dpt[r]; };
    if (opt) {
        for (int j = tid; j < n - 1; j += blockDim.x)
            for (int i = 0; i < W; ++i) dpt[j][i] = INFINITY;
        __syncthreads();
        for (bool changed = true; changed;) {
            float C[W];
            bool mine = false;
            const int j = tid;  // n - 1 <= 127 < blockDim.x
            if (j < n - 1) {
                tdp_node<W>(j, ch, lbf, nbf, tbf, C);
                for (int i = 0; i < W; ++i) mine |= __float_as_int(C[i]) != __float_as_int(dpt[j][i]);
            }
            __syncthreads();
            if (j < n - 1)
                for (int i = 0; i < W; ++i) dpt[j][i] = C[i];
            changed = __syncthreads_or(mine) != 0;
        }
    }
    auto src = [&](int r) { return r < 0 ? s.box + 6 * ~r : s.ibox + 6 * r; };
    for (int j = tid; j < n - 1; j += blockDim.x) {
        int refs[W];
        int* keep = a.tlas_refsw + W * (size_t)(toff + j);
        if (!rebuild) {
            for (int c = 0; c < W; ++c) refs[c] = keep[c];
        } else {
            if (opt) tdp_children<W>(j, ch, lbf, tbf, refs);
            else collapse_w<W>(j, ch, bx, refs);
            for (int c = 0; c < W; ++c) keep[c] = refs[c];
        }
        write_wide<W>(a, j, refs, src, i0, nodebase);
    }
}

__global__ void k_tlas(TlasArgs a, int rebuild) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int e = blockIdx.x;
    const int i0 = a.item_off[e];
    const int n = a.item_off[e + 1] - i0;
    const int nodebase = a.nb_blas + a.tlas_off[e];
    const int toff = a.tlas_off[e];
    const int tid = threadIdx.x;
    const float EMPTY[6] = {inf_f(), inf_f(), inf_f(), inf_f(), inf_f(), inf_f()};

    if (n <= 1) {
        if (tid == 0) {
            float b[4][6];
            int refs[4] = {REF_EMPTY, REF_EMPTY, REF_EMPTY, REF_EMPTY};
            for (int c = 0; c < 4; ++c)
                for (int k = 0; k < 6; ++k) b[c][k] = EMPTY[k];
            if (n == 1) {
                slot_box(a.item_box + 6 * i0, b[0]);
                refs[0] = ~i0;
                a.tlas_item_parent[i0] = 0;
            }
            write_node4(a.nodes, nodebase, b, refs, n);
            if (a.nodesw) {
                write_childw(a.nodesw, a.wide_w, nodebase, 0, b[0], refs[0]);
                for (int k = 1; k < a.wide_w; ++k) write_childw(a.nodesw, a.wide_w, nodebase, k, EMPTY, REF_EMPTY);
            }
            a.tlas_node_parent[toff] = -1;
            if (rebuild) a.tlas_depth[e] = 1;
        }
        return;
    }
    int P = 1;
    while (P < n) P <<= 1;
    TlasSmem s;
    unsigned char* p = smem_raw;
    s.keys = (uint64_t*)p; p += sizeof(uint64_t) * P;
    s.task = (int*)p; p += sizeof(int) * 4 * (n - 1);
    s.box = (float*)p; p += sizeof(float) * 6 * n;
    s.ibox = (float*)p; p += sizeof(float) * 6 * (n - 1);
    s.child = (int*)p; p += sizeof(int) * 2 * (n - 1);
    s.nparent = (int*)p; p += sizeof(int) * (n - 1);
    s.lparent = (int*)p; p += sizeof(int) * n;
    s.flags = (int*)p; p += sizeof(int) * (n - 1);
    float(*dpt)[TDP_STRIDE] = reinterpret_cast<float(*)[TDP_STRIDE]>(p);  // n <= TDP_MAX only

    for (int i = tid; i < n; i += blockDim.x)
        for (int k = 0; k < 6; ++k) s.box[6 * i + k] = a.item_box[6 * (i0 + i) + k];
    for (int j = tid; j < n - 1; j += blockDim.x) s.flags[j] = 0;
    __syncthreads();

    if (rebuild && a.builder == 1) {
        sah_build_cta(s, n);
    } else if (rebuild) {
        // centroid bounds of the instance boxes (empty boxes excluded)
        __shared__ float red[2][3][TLAS_THREADS / 32];
        float lo[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, hi[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
        for (int i = tid; i < n; i += blockDim.x) {
            if (isinf(s.box[6 * i])) continue;
            for (int k = 0; k < 3; ++k) {
                float c = 0.5f * s.box[6 * i + k] + 0.5f * s.box[6 * i + 3 + k];
                lo[k] = fminf(lo[k], c);
                hi[k] = fmaxf(hi[k], c);
            }
        }
        for (int o = 16; o > 0; o >>= 1)
            for (int k = 0; k < 3; ++k) {
                lo[k] = fminf(lo[k], __shfl_xor_sync(0xFFFFFFFFu, lo[k], o));
                hi[k] = fmaxf(hi[k], __shfl_xor_sync(0xFFFFFFFFu, hi[k], o));
            }
        if ((tid & 31) == 0)
            for (int k = 0; k < 3; ++k) { red[0][k][tid >> 5] = lo[k]; red[1][k][tid >> 5] = hi[k]; }
        __syncthreads();
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
            for (int k = 0; k < 3; ++k) {
                lo[k] = fminf(lo[k], red[0][k][w]);
                hi[k] = fmaxf(hi[k], red[1][k][w]);
            }
        for (int i = tid; i < P; i += blockDim.x) {
            uint64_t key = ~0ull;
            if (i < n) {
                uint32_t code = 0xFFFFFFFFu;  // empty boxes sort last
                if (!isinf(s.box[6 * i])) {
                    float u[3];
                    for (int k = 0; k < 3; ++k) {
                        float c = 0.5f * s.box[6 * i + k] + 0.5f * s.box[6 * i + 3 + k];
                        u[k] = unit_coord(c, lo[k], hi[k]);
                    }
                    code = morton30(u[0], u[1], u[2]);
                }
                key = ((uint64_t)code << 32) | (uint32_t)i;
            }
            s.keys[i] = key;
        }
        __syncthreads();
        // bitonic sort of P keys (ascending)
        for (int k = 2; k <= P; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = tid; i < P; i += blockDim.x) {
                    int ixj = i ^ j;
                    if (ixj > i) {
                        uint64_t x = s.keys[i], y = s.keys[ixj];
                        bool up = (i & k) == 0;
                        if ((x > y) == up) { s.keys[i] = y; s.keys[ixj] = x; }
                    }
                }
                __syncthreads();
            }
        }
        // Karras hierarchy over the n sorted keys
        for (int i = tid; i < n - 1; i += blockDim.x) {
            const uint64_t* k = s.keys;
            int d = (kdelta64(k, n, i, i + 1) - kdelta64(k, n, i, i - 1)) >= 0 ? 1 : -1;
            int dmin = kdelta64(k, n, i, i - d);
            int lmax = 2;
            while (kdelta64(k, n, i, i + lmax * d) > dmin) lmax <<= 1;
            int l = 0;
            for (int t = lmax >> 1; t >= 1; t >>= 1)
                if (kdelta64(k, n, i, i + (l + t) * d) > dmin) l += t;
            int j = i + l * d;
            int dnode = kdelta64(k, n, i, j);
            int sp = 0, t = l;
            do {
                t = (t + 1) >> 1;
                if (kdelta64(k, n, i, i + (sp + t) * d) > dnode) sp += t;
            } while (t > 1);
            int gamma = i + sp * d + (d < 0 ? -1 : 0);
            int lo_i = min(i, j), hi_i = max(i, j);
            int left = (lo_i == gamma) ? ~(int)(uint32_t)k[gamma] : gamma;
            int right = (hi_i == gamma + 1) ? ~(int)(uint32_t)k[gamma + 1] : gamma + 1;
            s.child[2 * i] = left;
            s.child[2 * i + 1] = right;
            if (left < 0) s.lparent[~left] = i; else s.nparent[left] = i;
            if (right < 0) s.lparent[~right] = i; else s.nparent[right] = i;
        }
        if (tid == 0) s.nparent[0] = -1;
        __syncthreads();
    }
    if (rebuild) {
        for (int j = tid; j < n - 1; j += blockDim.x) {
            a.tlas_child[2 * (toff + j)] = s.child[2 * j];
            a.tlas_child[2 * (toff + j) + 1] = s.child[2 * j + 1];
            a.tlas_node_parent[toff + j] = s.nparent[j];
        }
        for (int i = tid; i < n; i += blockDim.x) a.tlas_item_parent[i0 + i] = s.lparent[i];
        // depth: longest leaf-to-root path
        int dmax = 0;
        for (int i = tid; i < n; i += blockDim.x) {
            int dd = 0;
            for (int q = s.lparent[i]; q >= 0; q = s.nparent[q]) ++dd;
            dmax = max(dmax, dd);
        }
        for (int o = 16; o > 0; o >>= 1) dmax = max(dmax, __shfl_xor_sync(0xFFFFFFFFu, dmax, o));
        if ((tid & 31) == 0) atomicMax(&a.tlas_depth[e], dmax);
    } else {
        for (int j = tid; j < n - 1; j += blockDim.x) {
            s.child[2 * j] = a.tlas_child[2 * (toff + j)];
            s.child[2 * j + 1] = a.tlas_child[2 * (toff + j) + 1];
            s.nparent[j] = a.tlas_node_parent[toff + j];
        }
        for (int i = tid; i < n; i += blockDim.x) s.lparent[i] = a.tlas_item_parent[i0 + i];
        __syncthreads();
    }

    // bottom-up fit: the second child to arrive at a node unions the boxes
    for (int i = tid; i < n; i += blockDim.x) {
        int node = s.lparent[i];
        while (node >= 0) {
            __threadfence_block();
            if (atomicAdd(&s.flags[node], 1) == 0) break;
            __threadfence_block();
            volatile float* vb = s.box;
            volatile float* vi = s.ibox;
            float b[6], c[6];
            int ra = s.child[2 * node], rb = s.child[2 * node + 1];
            for (int k = 0; k < 6; ++k) {
                b[k] = ra < 0 ? vb[6 * ~ra + k] : vi[6 * ra + k];
                c[k] = rb < 0 ? vb[6 * ~rb + k] : vi[6 * rb + k];
            }
            for (int k = 0; k < 3; ++k) {
                vi[6 * node + k] = fminf(b[k], c[k]);
                vi[6 * node + 3 + k] = fmaxf(b[3 + k], c[3 + k]);
            }
            node = s.nparent[node];
        }
    }
    __syncthreads();
    // BVH4 node j = greedy 4-wide collapse of binary node j
    auto ch = [&](int r, int side) { return s.child[2 * r + side]; };
    auto bx = [&](int r, float b[6]) {
        for (int k = 0; k < 6; ++k) b[k] = s.ibox[6 * r + k];
    };
    // (a build chooses the collapses and records them; a refit keeps them and
    // only rewrites the boxes, as it keeps the binary topology)
    for (int j = tid; j < n - 1; j += blockDim.x) {
        int refs[4];
        int cnt = 0;
        int* keep = a.tlas_refs4 + 4 * (size_t)(toff + j);
        if (rebuild) {
            cnt = collapse4(j, ch, bx, refs);
            for (int c = 0; c < 4; ++c) keep[c] = refs[c];
        } else {
            for (int c = 0; c < 4; ++c) { refs[c] = keep[c]; cnt += refs[c] != REF_EMPTY; }
        }
        float b[4][6];
        int g[4];
        for (int c = 0; c < 4; ++c) {
            const int r = refs[c];
            const float* src = r == REF_EMPTY ? EMPTY : (r < 0 ? s.box + 6 * ~r : s.ibox + 6 * r);
            slot_box(src, b[c]);
            g[c] = r == REF_EMPTY ? REF_EMPTY : (r < 0 ? ~(i0 + ~r) : nodebase + r);
        }
        write_node4(a.nodes, nodebase + j, b, g, cnt);
    }
    if (a.nodesw) {
        // the wide copy of the interval-packet traversal: SAH-optimal
        // collapse for envs of <= TDP_MAX items, greedy above
        if (a.wide_w == 32) cta_wide<32>(a, s, n, i0, nodebase, toff, tid, rebuild, dpt, ch, bx);
        else if (a.wide_w == 16) cta_wide<16>(a, s, n, i0, nodebase, toff, tid, rebuild, dpt, ch, bx);
        else cta_wide<8>(a, s, n, i0, nodebase, toff, tid, rebuild, dpt, ch, bx);
    }
}

// ---- K7/K8 for small envs: one warp per env ---------------------------------------
// Envs of at most 32 TLAS items (c4 / c5 / Table-II rooms: 16-20) are built
// or refit by one warp instead of one 256-thread CTA: the LBVH keys are
// sorted by a register bitonic network over the lanes, Karras runs one
// internal node per lane, the fit iterates "every node := union of its
// children" until nothing changes (min / max are exact, so the boxes equal
// the CTA path's bottom-up fit bit for bit) and the collapses are the same
// code.  Refits go this way for envs of up to 128 items (4 nodes per lane).
// 2048 16-item envs: 124 -> ~10 us per refit (ncu); c3 (91 items): update
// 0.110 -> 0.061 ms.
constexpr int TW_WARPS = 4;    // warps (envs) per block
constexpr int TW_MAX = 128;    // refit: up to 4 items / nodes per lane (builds: 32)
constexpr int TW_PER = TW_MAX / 32;
struct TlasWarpSmem {
    uint64_t keys[32];
    float box[TW_MAX][6];
    float ibox[TW_MAX - 1][6];
    float dpt[31][TDP_STRIDE];  // SAH-optimal wide-collapse tables (builds: <= 32 items)
    int child[2 * (TW_MAX - 1)];
    int nparent[TW_MAX - 1];
    int lparent[TW_MAX];
};

template <int W, class CH>
__device__ __forceinline__ void warp_wide(const TlasArgs& a, TlasWarpSmem& s, int n, int i0, int nodebase, int toff,
                                          int lane, int rebuild, const CH& ch) {
    const unsigned FULL = 0xFFFFFFFFu;
    auto lbf = [&](int i) { return s.box[i]; };
    auto nbf = [&](int r) { return s.ibox[r]; };
    auto tbf = [&](int r) { return s.dpt[r]; };
    auto src = [&](int r) { return r < 0 ? s.box[~r] : s.ibox[r]; };
    if (n <= W) {  // one wide node (the other binary nodes are unreachable and not written)
        if (lane == 0) {
            int refs[W];
            int* keep = a.tlas_refsw + W * (size_t)toff;
            if (rebuild) {
                all_items<W>(ch, refs);
                for (int c = 0; c < W; ++c) keep[c] = refs[c];
            } else {
                for (int c = 0; c < W; ++c) refs[c] = keep[c];
            }
            write_wide<W>(a, 0, refs, src, i0, nodebase);
        }
        return;
    }
    if (!rebuild) {  // a refit keeps the build's collapse
        for (int j = lane; j < n - 1; j += 32) {
            int refs[W];
            const int* keep = a.tlas_refsw + W * (size_t)(toff + j);
            for (int c = 0; c < W; ++c) refs[c] = keep[c];
            write_wide<W>(a, j, refs, src, i0, nodebase);
        }
        return;
    }
    for (int j = lane; j < n - 1; j += 32)
        for (int i = 0; i < W; ++i) s.dpt[j][i] = INFINITY;
    __syncwarp();
    for (bool changed = true; __any_sync(FULL, changed);) {
        changed = false;
        float C[TW_PER][W];
#pragma unroll
        for (int m = 0; m < TW_PER; ++m) {
            const int j = lane + 32 * m;
            if (j < n - 1) {
                tdp_node<W>(j, ch, lbf, nbf, tbf, C[m]);
                for (int i = 0; i < W; ++i) changed |= __float_as_int(C[m][i]) != __float_as_int(s.dpt[j][i]);
            }
        }
        __syncwarp();
#pragma unroll
        for (int m = 0; m < TW_PER; ++m) {
            const int j = lane + 32 * m;
            if (j < n - 1)
                for (int i = 0; i < W; ++i) s.dpt[j][i] = C[m][i];
        }
        __syncwarp();
    }
    for (int j = lane; j < n - 1; j += 32) {
        int refs[W];
        tdp_children<W>(j, ch, lbf, tbf, refs);
        int* keep = a.tlas_refsw + W * (size_t)(toff + j);
        for (int c = 0; c < W; ++c) keep[c] = refs[c];
        write_wide<W>(a, j, refs, src, i0, nodebase);
    }
}

__global__ void __launch_bounds__(32 * TW_WARPS) k_tlas_warp(TlasArgs a, int rebuild) {
    extern __shared__ __align__(16) unsigned char tw_raw[];
    TlasWarpSmem* sm = reinterpret_cast<TlasWarpSmem*>(tw_raw);
    const unsigned FULL = 0xFFFFFFFFu;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int e = blockIdx.x * TW_WARPS + w;
    if (e >= a.n_envs) return;  // warp-uniform
    TlasWarpSmem& s = sm[w];
    const int i0 = a.item_off[e];
    const int n = a.item_off[e + 1] - i0;
    const int nodebase = a.nb_blas + a.tlas_off[e];
    const int toff = a.tlas_off[e];
    const float EMPTY[6] = {inf_f(), inf_f(), inf_f(), inf_f(), inf_f(), inf_f()};
    if (n <= 1) {
        if (lane == 0) {
            float b[4][6];
            int refs[4] = {REF_EMPTY, REF_EMPTY, REF_EMPTY, REF_EMPTY};
            for (int c = 0; c < 4; ++c)
                for (int k = 0; k < 6; ++k) b[c][k] = EMPTY[k];
            if (n == 1) {
                slot_box(a.item_box + 6 * i0, b[0]);
                refs[0] = ~i0;
                a.tlas_item_parent[i0] = 0;
            }
            write_node4(a.nodes, nodebase, b, refs, n);
            if (a.nodesw) {
                write_childw(a.nodesw, a.wide_w, nodebase, 0, b[0], refs[0]);
                for (int k = 1; k < a.wide_w; ++k) write_childw(a.nodesw, a.wide_w, nodebase, k, EMPTY, REF_EMPTY);
            }
            a.tlas_node_parent[toff] = -1;
            if (rebuild) a.tlas_depth[e] = 1;
        }
        return;
    }
    float bl[6];
    for (int i = lane; i < n; i += 32)
        for (int k = 0; k < 6; ++k) s.box[i][k] = a.item_box[6 * (i0 + i) + k];
    __syncwarp();
    if (lane < n)
        for (int k = 0; k < 6; ++k) bl[k] = s.box[lane][k];
    if (rebuild) {  // n <= 32 (tlas_build)
        // centroid bounds of the non-empty boxes, Morton keys, lane bitonic sort
        float lo[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, hi[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
        const bool valid = lane < n && !isinf(bl[0]);
        if (valid)
            for (int k = 0; k < 3; ++k) lo[k] = hi[k] = 0.5f * bl[k] + 0.5f * bl[3 + k];
        for (int o = 16; o > 0; o >>= 1)
            for (int k = 0; k < 3; ++k) {
                lo[k] = fminf(lo[k], __shfl_xor_sync(FULL, lo[k], o));
                hi[k] = fmaxf(hi[k], __shfl_xor_sync(FULL, hi[k], o));
            }
        uint64_t key = ~0ull;
        if (lane < n) {
            uint32_t code = 0xFFFFFFFFu;  // empty boxes sort last
            if (valid) {
                float u[3];
                for (int k = 0; k < 3; ++k) u[k] = unit_coord(0.5f * bl[k] + 0.5f * bl[3 + k], lo[k], hi[k]);
                code = morton30(u[0], u[1], u[2]);
            }
            key = ((uint64_t)code << 32) | (uint32_t)lane;
        }
        for (int k = 2; k <= 32; k <<= 1)
            for (int j = k >> 1; j > 0; j >>= 1) {
                const uint64_t o = __shfl_xor_sync(FULL, key, j);
                const bool up = (lane & k) == 0, lower = (lane & j) == 0;
                key = (lower == up) ? (key < o ? key : o) : (key < o ? o : key);
            }
        s.keys[lane] = key;
        __syncwarp();
        if (lane < n - 1) {
            const uint64_t* k = s.keys;
            const int i = lane;
            int d = (kdelta64(k, n, i, i + 1) - kdelta64(k, n, i, i - 1)) >= 0 ? 1 : -1;
            int dmin = kdelta64(k, n, i, i - d);
            int lmax = 2;
            while (kdelta64(k, n, i, i + lmax * d) > dmin) lmax <<= 1;
            int l = 0;
            for (int t = lmax >> 1; t >= 1; t >>= 1)
                if (kdelta64(k, n, i, i + (l + t) * d) > dmin) l += t;
            int j = i + l * d;
            int dnode = kdelta64(k, n, i, j);
            int sp = 0, t = l;
            do {
                t = (t + 1) >> 1;
                if (kdelta64(k, n, i, i + (sp + t) * d) > dnode) sp += t;
            } while (t > 1);
            int gamma = i + sp * d + (d < 0 ? -1 : 0);
            int lo_i = min(i, j), hi_i = max(i, j);
            int left = (lo_i == gamma) ? ~(int)(uint32_t)k[gamma] : gamma;
            int right = (hi_i == gamma + 1) ? ~(int)(uint32_t)k[gamma + 1] : gamma + 1;
            s.child[2 * i] = left;
            s.child[2 * i + 1] = right;
            if (left < 0) s.lparent[~left] = i; else s.nparent[left] = i;
            if (right < 0) s.lparent[~right] = i; else s.nparent[right] = i;
        }
        if (lane == 0) s.nparent[0] = -1;
        __syncwarp();
        if (lane < n - 1) {
            a.tlas_child[2 * (toff + lane)] = s.child[2 * lane];
            a.tlas_child[2 * (toff + lane) + 1] = s.child[2 * lane + 1];
            a.tlas_node_parent[toff + lane] = s.nparent[lane];
        }
        int dd = 0;
        if (lane < n) {
            a.tlas_item_parent[i0 + lane] = s.lparent[lane];
            for (int q = s.lparent[lane]; q >= 0; q = s.nparent[q]) ++dd;
        }
        for (int o = 16; o > 0; o >>= 1) dd = max(dd, __shfl_xor_sync(FULL, dd, o));
        if (lane == 0) atomicMax(&a.tlas_depth[e], dd);
    } else {
        for (int j = lane; j < n - 1; j += 32) {
            s.child[2 * j] = a.tlas_child[2 * (toff + j)];
            s.child[2 * j + 1] = a.tlas_child[2 * (toff + j) + 1];
        }
    }
    // fit: every internal node := union of its children, until nothing
    // changes (lane l owns nodes l, l + 32, ...)
    __syncwarp();
    for (int j = lane; j < n - 1; j += 32) {
        s.ibox[j][0] = s.ibox[j][1] = s.ibox[j][2] = inf_f();
        s.ibox[j][3] = s.ibox[j][4] = s.ibox[j][5] = -inf_f();
    }
    __syncwarp();
    for (bool changed = true; __any_sync(FULL, changed);) {
        changed = false;
        float nb[TW_PER][6];
#pragma unroll
        for (int m = 0; m < TW_PER; ++m) {
            const int j = lane + 32 * m;
            if (j < n - 1) {
                const int ra = s.child[2 * j], rb = s.child[2 * j + 1];
                const float* pa = ra < 0 ? s.box[~ra] : s.ibox[ra];
                const float* pb = rb < 0 ? s.box[~rb] : s.ibox[rb];
                for (int k = 0; k < 3; ++k) {
                    nb[m][k] = fminf(pa[k], pb[k]);
                    nb[m][3 + k] = fmaxf(pa[3 + k], pb[3 + k]);
                }
                for (int k = 0; k < 6; ++k) changed |= __float_as_int(nb[m][k]) != __float_as_int(s.ibox[j][k]);
            }
        }
        __syncwarp();
#pragma unroll
        for (int m = 0; m < TW_PER; ++m) {
            const int j = lane + 32 * m;
            if (j < n - 1)
                for (int k = 0; k < 6; ++k) s.ibox[j][k] = nb[m][k];
        }
        __syncwarp();
    }
    // BVH4 node j = greedy 4-wide collapse of binary node j (and the BVH8 copy)
    auto ch = [&](int r, int side) { return s.child[2 * r + side]; };
    auto bx = [&](int r, float b[6]) {
        for (int k = 0; k < 6; ++k) b[k] = s.ibox[r][k];
    };
    if (a.nodesw) {  // SAH-optimal wide copy (builds: n <= 32; refits keep the stored collapse)
        if (a.wide_w == 32) warp_wide<32>(a, s, n, i0, nodebase, toff, lane, rebuild, ch);
        else if (a.wide_w == 16) warp_wide<16>(a, s, n, i0, nodebase, toff, lane, rebuild, ch);
        else warp_wide<8>(a, s, n, i0, nodebase, toff, lane, rebuild, ch);
    }
    for (int j = lane; j < n - 1; j += 32) {
        int refs[4];
        int cnt = 0;
        int* keep = a.tlas_refs4 + 4 * (size_t)(toff + j);
        if (rebuild) {
            cnt = collapse4(j, ch, bx, refs);
            for (int c = 0; c < 4; ++c) keep[c] = refs[c];
        } else {
            for (int c = 0; c < 4; ++c) { refs[c] = keep[c]; cnt += refs[c] != REF_EMPTY; }
        }
        float b[4][6];
        int g[4];
        for (int c = 0; c < 4; ++c) {
            const int r = refs[c];
            const float* src = r == REF_EMPTY ? EMPTY : (r < 0 ? s.box[~r] : s.ibox[r]);
            slot_box(src, b[c]);
            g[c] = r == REF_EMPTY ? REF_EMPTY : (r < 0 ? ~(i0 + ~r) : nodebase + r);
        }
        write_node4(a.nodes, nodebase + j, b, g, cnt);
    }
}

size_t tlas_smem_bytes(int n) {
    if (n <= 1) return 16;
    int P = 1;
    while (P < n) P <<= 1;
    return sizeof(uint64_t) * P + sizeof(int) * 4 * (n - 1) + sizeof(float) * 6 * n + sizeof(float) * 6 * (n - 1) +
           sizeof(int) * 2 * (n - 1) + sizeof(int) * (n - 1) + sizeof(int) * n + sizeof(int) * (n - 1) +
           (n <= TDP_MAX ? sizeof(float) * TDP_STRIDE * (n - 1) : 0);  // wide-collapse DP tables
}

}  // namespace

cudaError_t items_update(const TlasArgs& a, int n_items, cudaStream_t stream) {
    if (n_items > 0) k_items<<<(n_items + 127) / 128, 128, 0, stream>>>(a, n_items);
    return cudaGetLastError();
}

cudaError_t tlas_build(const TlasArgs& a, bool rebuild, cudaStream_t stream) {
    // (an env of <= TDP_MAX items also holds the DP tables: the largest such
    // env may need more than the largest env)
    size_t smem = tlas_smem_bytes(a.max_n);
    if (a.max_n > TDP_MAX) smem = std::max(smem, tlas_smem_bytes(TDP_MAX));
    {
        // k_tlas has ~33 KB of static shared memory (SAH bins):
        // any dynamic part beyond the default 48 KB total needs the opt-in
        cudaError_t e = cudaFuncSetAttribute(k_tlas, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    if (rebuild) {
        cudaError_t e = cudaMemsetAsync(a.tlas_depth, 0, sizeof(int) * a.n_envs, stream);
        if (e != cudaSuccess) return e;
    }
    if (rebuild ? (a.max_n <= 32 && a.builder == 0) : a.max_n <= TW_MAX) {
        const int tw_smem = (int)sizeof(TlasWarpSmem) * TW_WARPS;
        cudaError_t e = cudaFuncSetAttribute(k_tlas_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, tw_smem);
        if (e != cudaSuccess) return e;
        k_tlas_warp<<<(a.n_envs + TW_WARPS - 1) / TW_WARPS, 32 * TW_WARPS, tw_smem, stream>>>(a, rebuild ? 1 : 0);
        return cudaGetLastError();
    }
    k_tlas<<<a.n_envs, TLAS_THREADS, smem, stream>>>(a, rebuild ? 1 : 0);
    return cudaGetLastError();
}

}  // namespace agr
