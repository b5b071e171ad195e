// blas.cu -- per-asset bottom-level BVH (BLAS) build on the GPU.
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
//   K5 pack         64-B nodes + 48-B triangle records + exact vertices
// Zero-area faces (exactly, in FP64 from the FP32 inputs) are left out of
// the tree: they can never be hit, and the face numbering is kept by the
// per-leaf local face id.
#include "agr_internal.cuh"

#include <cfloat>

namespace agr {
namespace {

constexpr int T_BLK = 256;
constexpr int RS_THREADS = 256;
constexpr int RS_ROUNDS = 4;
constexpr int RS_TILE = RS_THREADS * RS_ROUNDS;
constexpr uint32_t DEGENERATE_KEY = 0xFFFFFFFFu;

struct Scratch {
    float* tri_box;      // [F][6] (lo xyz, hi xyz)
    uint32_t* bounds;    // [8]: ordered-int centroid lo xyz, hi xyz, radius, n_valid
    uint32_t* keys[2];   // [F]
    uint32_t* vals[2];   // [F]
    uint32_t* hist;      // [256 * nblocks]
    int* child;          // [2 * (F-1)] local refs
    int* node_parent;    // [F-1]
    int* leaf_parent;    // [F]
    float* ibox;         // [F-1][6]
    int* flags;          // [F-1]
    int* depth;          // [1]
    float* cost;         // [F-1] SAH cost of each internal node's subtree (TRBVH)
};

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

Scratch carve(void* base, int F) {
    char* p = (char*)base;
    size_t nb = (F + RS_TILE - 1) / RS_TILE;
    int Fi = F > 1 ? F - 1 : 1;
    Scratch s;
    s.tri_box = (float*)p; p += align_up(sizeof(float) * 6 * F);
    s.bounds = (uint32_t*)p; p += align_up(sizeof(uint32_t) * 8);
    for (int i = 0; i < 2; ++i) { s.keys[i] = (uint32_t*)p; p += align_up(sizeof(uint32_t) * F); }
    for (int i = 0; i < 2; ++i) { s.vals[i] = (uint32_t*)p; p += align_up(sizeof(uint32_t) * F); }
    s.hist = (uint32_t*)p; p += align_up(sizeof(uint32_t) * 256 * nb);
    s.child = (int*)p; p += align_up(sizeof(int) * 2 * Fi);
    s.node_parent = (int*)p; p += align_up(sizeof(int) * Fi);
    s.leaf_parent = (int*)p; p += align_up(sizeof(int) * F);
    s.ibox = (float*)p; p += align_up(sizeof(float) * 6 * Fi);
    s.flags = (int*)p; p += align_up(sizeof(int) * Fi);
    s.depth = (int*)p; p += align_up(sizeof(int));
    s.cost = (float*)p; p += align_up(sizeof(float) * Fi);
    return s;
}

// ---- K1: triangle prep ------------------------------------------------------
__global__ void k_init_bounds(uint32_t* b) {
    int i = threadIdx.x;
    if (i < 3) b[i] = float_to_ordered(FLT_MAX);
    else if (i < 6) b[i] = float_to_ordered(-FLT_MAX);
    else if (i == 6) b[i] = float_to_ordered(0.0f);
    else if (i == 7) b[i] = 0u;
}

__global__ void k_tri_prep(const float* __restrict__ verts, const int* __restrict__ faces, int F,
                           int V, float* __restrict__ tri_box, uint32_t* __restrict__ vflag,
                           uint32_t* bounds) {
    int f = blockIdx.x * blockDim.x + threadIdx.x;
    // asset radius over vertices
    float r = 0.0f;
    for (int v = f; v < V; v += gridDim.x * blockDim.x) {
        float x = verts[3 * v], y = verts[3 * v + 1], z = verts[3 * v + 2];
        r = fmaxf(r, sqrtf(x * x + y * y + z * z) * 1.000001f);
    }
    float clo[3] = {FLT_MAX, FLT_MAX, FLT_MAX}, chi[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
    bool valid = false;
    if (f < F) {
        const float* a = verts + 3 * faces[3 * f];
        const float* b = verts + 3 * faces[3 * f + 1];
        const float* c = verts + 3 * faces[3 * f + 2];
        // exact-input FP64 area: zero only for genuinely degenerate input
        d3 A = mkd(a[0], a[1], a[2]), B = mkd(b[0], b[1], b[2]), C = mkd(c[0], c[1], c[2]);
        d3 n = crossd(subd(B, A), subd(C, A));
        valid = (n.x != 0.0 || n.y != 0.0 || n.z != 0.0);
        float lo[3], hi[3];
        for (int k = 0; k < 3; ++k) {
            lo[k] = fminf(a[k], fminf(b[k], c[k]));
            hi[k] = fmaxf(a[k], fmaxf(b[k], c[k]));
            tri_box[6 * f + k] = lo[k];
            tri_box[6 * f + 3 + k] = hi[k];
            if (valid) {
                float cc = 0.5f * lo[k] + 0.5f * hi[k];
                clo[k] = cc;
                chi[k] = cc;
            }
        }
        vflag[f] = valid ? 1u : 0u;
    }
    // block reduce bounds, radius and valid count
    __shared__ float s_lo[3][T_BLK / 32], s_hi[3][T_BLK / 32], s_r[T_BLK / 32];
    __shared__ unsigned s_cnt[T_BLK / 32];
    unsigned cnt = __popc(__ballot_sync(0xFFFFFFFFu, valid));
    for (int o = 16; o > 0; o >>= 1) {
        for (int k = 0; k < 3; ++k) {
            clo[k] = fminf(clo[k], __shfl_xor_sync(0xFFFFFFFFu, clo[k], o));
            chi[k] = fmaxf(chi[k], __shfl_xor_sync(0xFFFFFFFFu, chi[k], o));
        }
        r = fmaxf(r, __shfl_xor_sync(0xFFFFFFFFu, r, o));
    }
    int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        for (int k = 0; k < 3; ++k) { s_lo[k][w] = clo[k]; s_hi[k][w] = chi[k]; }
        s_r[w] = r;
        s_cnt[w] = cnt;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned tot = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
            for (int k = 0; k < 3; ++k) {
                clo[k] = fminf(clo[k], s_lo[k][i]);
                chi[k] = fmaxf(chi[k], s_hi[k][i]);
            }
            r = fmaxf(r, s_r[i]);
            tot += s_cnt[i];
        }
        for (int k = 0; k < 3; ++k) {
            atomicMin(&bounds[k], float_to_ordered(clo[k]));
            atomicMax(&bounds[3 + k], float_to_ordered(chi[k]));
        }
        atomicMax(&bounds[6], float_to_ordered(r));
        atomicAdd(&bounds[7], tot);
    }
}

// ---- K1b: Morton codes ------------------------------------------------------
__global__ void k_morton(const float* __restrict__ tri_box, const uint32_t* __restrict__ vflag,
                         int F, const uint32_t* __restrict__ bounds, uint32_t* __restrict__ keys,
                         uint32_t* __restrict__ vals) {
    int f = blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= F) return;
    uint32_t key = DEGENERATE_KEY;
    if (vflag[f]) {
        float u[3];
        for (int k = 0; k < 3; ++k) {
            float lo = ordered_to_float(bounds[k]), hi = ordered_to_float(bounds[3 + k]);
            float c = 0.5f * tri_box[6 * f + k] + 0.5f * tri_box[6 * f + 3 + k];
            u[k] = unit_coord(c, lo, hi);
        }
        key = morton30(u[0], u[1], u[2]);
    }
    keys[f] = key;
    vals[f] = (uint32_t)f;
}

// ---- K2: stable LSD radix sort (8-bit digits) --------------------------------
__global__ void k_rs_hist(const uint32_t* __restrict__ keys, int n, int shift,
                          uint32_t* __restrict__ hist, int nblocks) {
    __shared__ uint32_t cnt[256];
    cnt[threadIdx.x] = 0;
    __syncthreads();
    int base = blockIdx.x * RS_TILE;
    for (int r = 0; r < RS_ROUNDS; ++r) {
        int i = base + r * RS_THREADS + threadIdx.x;
        if (i < n) atomicAdd(&cnt[(keys[i] >> shift) & 255u], 1u);
    }
    __syncthreads();
    hist[threadIdx.x * nblocks + blockIdx.x] = cnt[threadIdx.x];
}

// single-CTA exclusive scan of hist[total] in place
__global__ void k_rs_scan(uint32_t* hist, int total) {
    __shared__ uint32_t warp_sums[32];
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int base = 0; base < total; base += blockDim.x) {
        int i = base + threadIdx.x;
        uint32_t v = i < total ? hist[i] : 0u;
        uint32_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_sums[w] = x;
        __syncthreads();
        if (w == 0) {
            uint32_t s = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0u;
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t y = __shfl_up_sync(0xFFFFFFFFu, s, o);
                if (lane >= o) s += y;
            }
            if (lane < (int)(blockDim.x >> 5)) warp_sums[lane] = s;  // inclusive
        }
        __syncthreads();
        uint32_t excl = carry + (w > 0 ? warp_sums[w - 1] : 0u) + x - v;
        if (i < total) hist[i] = excl;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = excl + v;
        __syncthreads();
    }
}

__global__ void k_rs_scatter(const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                             uint32_t* __restrict__ kout, uint32_t* __restrict__ vout, int n,
                             int shift, const uint32_t* __restrict__ hist, int nblocks) {
    __shared__ uint32_t base[256];
    __shared__ uint32_t wc[RS_THREADS / 32][256];
    base[threadIdx.x] = hist[threadIdx.x * nblocks + blockIdx.x];
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    for (int r = 0; r < RS_ROUNDS; ++r) {
        for (int k = 0; k < RS_THREADS / 32; ++k) wc[k][threadIdx.x] = 0;
        __syncthreads();
        int i = blockIdx.x * RS_TILE + r * RS_THREADS + threadIdx.x;
        bool valid = i < n;
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

// ---- K3: Karras radix tree ------------------------------------------------------
__device__ __forceinline__ int kdelta(const uint32_t* k, int n, int i, int j) {
    if (j < 0 || j >= n) return -1;
    uint32_t a = k[i], b = k[j];
    if (a == b) return 32 + __clz((unsigned)(i ^ j));
    return __clz(a ^ b);
}

__global__ void k_karras(const uint32_t* __restrict__ k, const uint32_t* n_dev, int* __restrict__ child,
                         int* __restrict__ node_parent, int* __restrict__ leaf_parent) {
    const int n = (int)*n_dev;
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n - 1) return;
    int d = (kdelta(k, n, i, i + 1) - kdelta(k, n, i, i - 1)) >= 0 ? 1 : -1;
    int dmin = kdelta(k, n, i, i - d);
    int lmax = 2;
    while (kdelta(k, n, i, i + lmax * d) > dmin) lmax <<= 1;
    int l = 0;
    for (int t = lmax >> 1; t >= 1; t >>= 1)
        if (kdelta(k, n, i, i + (l + t) * d) > dmin) l += t;
    int j = i + l * d;
    int dnode = kdelta(k, n, i, j);
    // binary search for the split: the last position (from i towards j) whose
    // prefix with key i is longer than the node's common prefix.  Positions
    // beyond j never qualify (keys are sorted), so no bound check is needed.
    int s = 0;
    int t = l;
    do {
        t = (t + 1) >> 1;
        if (kdelta(k, n, i, i + (s + t) * d) > dnode) s += t;
    } while (t > 1);
    int gamma = i + s * d + (d < 0 ? -1 : 0);
    int lo = min(i, j), hi = max(i, j);
    int left = (lo == gamma) ? ~gamma : gamma;
    int right = (hi == gamma + 1) ? ~(gamma + 1) : gamma + 1;
    child[2 * i] = left;
    child[2 * i + 1] = right;
    if (left < 0) leaf_parent[~left] = i; else node_parent[left] = i;
    if (right < 0) leaf_parent[~right] = i; else node_parent[right] = i;
    if (i == 0) node_parent[0] = -1;
}

// ---- K4: bottom-up fit ------------------------------------------------------------
__device__ __forceinline__ void load_box_cg(const float* p, float b[6]) {
    for (int k = 0; k < 6; ++k) b[k] = __ldcg(p + k);
}

__global__ void k_fit(const uint32_t* n_dev, const uint32_t* __restrict__ sorted_prim, const float* tri_box,
                      const int* __restrict__ child, const int* __restrict__ node_parent,
                      const int* __restrict__ leaf_parent, float* ibox, int* flags, int* depth) {
    const int n = (int)*n_dev;
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (n < 2 || p >= n) return;
    // depth of this leaf
    int dd = 0;
    for (int q = leaf_parent[p]; q >= 0; q = node_parent[q]) ++dd;
    atomicMax(depth, dd);
    int node = leaf_parent[p];
    while (node >= 0) {
        __threadfence();
        if (atomicAdd(&flags[node], 1) == 0) return;  // first arrival: sibling not ready
        __threadfence();
        float b[6], c[6];
        for (int side = 0; side < 2; ++side) {
            int r = child[2 * node + side];
            float* dst = side == 0 ? b : c;
            if (r < 0) load_box_cg(tri_box + 6 * sorted_prim[~r], dst);
            else load_box_cg(ibox + 6 * r, dst);
        }
        for (int k = 0; k < 3; ++k) {
            __stcg(ibox + 6 * node + k, fminf(b[k], c[k]));
            __stcg(ibox + 6 * node + 3 + k, fmaxf(b[3 + k], c[3 + k]));
        }
        node = node_parent[node];
    }
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

__global__ void k_trbvh(const uint32_t* n_dev, const uint32_t* __restrict__ sorted_prim,
                        const float* __restrict__ tri_box, int* child, int* node_parent,
                        int* leaf_parent, float* ibox, float* cost, int* flags) {
    const int n = (int)*n_dev;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (n < 2 || p >= n) return;
    int node = __ldcg(leaf_parent + p);
    while (node >= 0) {
        __threadfence();
        if (atomicAdd(&flags[node], 1) == 0) return;  // the sibling subtree is not final yet
        __threadfence();
        // treelet leaves (subtree roots) and internal nodes
        int L[TREELET], I[TREELET - 1];
        int m = 2, ni = 1;
        L[0] = __ldcg(child + 2 * node);
        L[1] = __ldcg(child + 2 * node + 1);
        I[0] = node;
        while (m < TREELET) {
            int best = -1;
            float ba = -1.0f;
            for (int k = 0; k < m; ++k) {
                if (L[k] < 0) continue;
                float b[6];
                for (int c = 0; c < 6; ++c) b[c] = __ldcg(ibox + 6 * L[k] + c);
                const float a = box_area(b);
                if (a > ba) { ba = a; best = k; }
            }
            if (best < 0) break;
            const int r = L[best];
            I[ni++] = r;
            L[best] = __ldcg(child + 2 * r);
            L[m++] = __ldcg(child + 2 * r + 1);
        }
        // leaf boxes / costs
        float lb[TREELET][6], lc[TREELET];
        for (int k = 0; k < m; ++k) {
            const float* src = L[k] < 0 ? tri_box + 6 * sorted_prim[~L[k]] : ibox + 6 * L[k];
            for (int c = 0; c < 6; ++c) lb[k][c] = __ldcg(src + c);
            lc[k] = L[k] < 0 ? SAH_CT * box_area(lb[k]) : __ldcg(cost + L[k]);
        }
        // the node's current cost (children final)
        float nb[6];
        for (int c = 0; c < 6; ++c) nb[c] = __ldcg(ibox + 6 * node + c);
        float ccur;
        {
            const int c0 = __ldcg(child + 2 * node), c1 = __ldcg(child + 2 * node + 1);
            auto sub_cost = [&](int r) {
                if (r < 0) {
                    float b[6];
                    for (int c = 0; c < 6; ++c) b[c] = __ldcg(tri_box + 6 * sorted_prim[~r] + c);
                    return SAH_CT * box_area(b);
                }
                return __ldcg(cost + r);
            };
            ccur = SAH_CI * box_area(nb) + sub_cost(c0) + sub_cost(c1);
        }
        if (m >= 3) {
            const int full = (1 << m) - 1;
            float sb[1 << TREELET][6];
            float copt[1 << TREELET];
            unsigned char part[1 << TREELET];
            for (int sset = 1; sset <= full; ++sset) {
                const int low = __ffs(sset) - 1;
                const int rest = sset & (sset - 1);
                if (rest == 0) {
                    for (int c = 0; c < 6; ++c) sb[sset][c] = lb[low][c];
                    copt[sset] = lc[low];
                    part[sset] = 0;
                    continue;
                }
                for (int c = 0; c < 3; ++c) {
                    sb[sset][c] = fminf(sb[rest][c], lb[low][c]);
                    sb[sset][3 + c] = fmaxf(sb[rest][3 + c], lb[low][3 + c]);
                }
                const int lsb = sset & -sset;
                float best = INFINITY;
                int bp = 0;
                for (int q = (sset - 1) & sset; q; q = (q - 1) & sset) {
                    if (!(q & lsb)) continue;  // each unordered partition once
                    const float cc = copt[q] + copt[sset ^ q];
                    if (cc < best) { best = cc; bp = q; }
                }
                copt[sset] = SAH_CI * box_area(sb[sset]) + best;
                part[sset] = (unsigned char)bp;
            }
            if (copt[full] < ccur * (1.0f - 1e-6f)) {
                // rebuild the treelet: root keeps its id, the others are reused
                int st_s[TREELET], st_n[TREELET], sp = 0, pool = 1;
                st_s[sp] = full;
                st_n[sp++] = node;
                while (sp > 0) {
                    --sp;
                    const int sset = st_s[sp], nd = st_n[sp];
                    const int q0 = part[sset], q1 = sset ^ q0;
                    for (int side = 0; side < 2; ++side) {
                        const int sub = side == 0 ? q0 : q1;
                        int c;
                        if ((sub & (sub - 1)) == 0) {
                            c = L[__ffs(sub) - 1];
                        } else {
                            c = I[pool++];
                            st_s[sp] = sub;
                            st_n[sp++] = c;
                            for (int k = 0; k < 6; ++k) __stcg(ibox + 6 * c + k, sb[sub][k]);
                            __stcg(cost + c, copt[sub]);
                        }
                        __stcg(child + 2 * nd + side, c);
                        if (c < 0) __stcg(leaf_parent + ~c, nd);
                        else __stcg(node_parent + c, nd);
                    }
                }
                __stcg(cost + node, copt[full]);
            } else {
                __stcg(cost + node, ccur);
            }
        } else {
            __stcg(cost + node, ccur);
        }
        __threadfence();
        node = __ldcg(node_parent + node);
    }
}

__global__ void k_depth(const uint32_t* n_dev, const int* leaf_parent, const int* node_parent, int* depth) {
    const int n = (int)*n_dev;
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (n < 2 || p >= n) return;
    int dd = 0;
    for (int q = leaf_parent[p]; q >= 0; q = node_parent[q]) ++dd;
    atomicMax(depth, dd);
}

// ---- K5: pack -------------------------------------------------------------------------
__device__ __forceinline__ void child_box(int r, const uint32_t* sorted_prim, const float* tri_box,
                                          const float* ibox, float b[6]) {
    if (r == REF_EMPTY) {
        for (int k = 0; k < 6; ++k) b[k] = __int_as_float(0x7f800000);  // +inf: never hit
        return;
    }
    const float* src = r < 0 ? tri_box + 6 * sorted_prim[~r] : ibox + 6 * r;
    for (int k = 0; k < 6; ++k) b[k] = __ldcg(src + k);
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

__global__ void k_pack_nodes(const uint32_t* n_dev, const uint32_t* __restrict__ sorted_prim,
                             const float* tri_box, const int* __restrict__ child,
                             const float* ibox, float4* nodes, int node_base, int leaf_base) {
    const int n = (int)*n_dev;
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    int n_int = n > 1 ? n - 1 : 1;
    if (i >= n_int) return;
    int ra, rb;
    if (n > 1) { ra = child[2 * i]; rb = child[2 * i + 1]; }
    else if (n == 1) { ra = ~0; rb = REF_EMPTY; }
    else { ra = REF_EMPTY; rb = REF_EMPTY; }
    float a[6], b[6];
    child_box(ra, sorted_prim, tri_box, ibox, a);
    child_box(rb, sorted_prim, tri_box, ibox, b);
    write_node(nodes, node_base + i, a, b, global_ref(ra, node_base, leaf_base),
               global_ref(rb, node_base, leaf_base));
}

// K5b: BVH4 node j = greedy 4-wide collapse of binary node j.
__global__ void k_collapse4(const uint32_t* n_dev, const uint32_t* __restrict__ sorted_prim, const float* tri_box,
                            const int* __restrict__ child, const float* ibox, float4* nodes,
                            int node_base, int leaf_base) {
    const int n = (int)*n_dev;
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    int n_int = n > 1 ? n - 1 : 1;
    if (j >= n_int) return;
    int refs[4];
    int cnt;
    if (n > 1) {
        auto ch = [&](int r, int side) { return __ldg(child + 2 * r + side); };
        auto bx = [&](int r, float bb[6]) {
            for (int k = 0; k < 6; ++k) bb[k] = __ldcg(ibox + 6 * r + k);
        };
        cnt = collapse4(j, ch, bx, refs);
    } else {
        refs[0] = n == 1 ? ~0 : REF_EMPTY;
        refs[1] = refs[2] = refs[3] = REF_EMPTY;
        cnt = n == 1 ? 1 : 0;
    }
    float boxes[4][6];
    int g[4];
    for (int k = 0; k < 4; ++k) {
        child_box(refs[k], sorted_prim, tri_box, ibox, boxes[k]);
        g[k] = global_ref(refs[k], node_base, leaf_base);
    }
    write_node4(nodes, node_base + j, boxes, g, cnt);
}

__global__ void k_pack_tris(const uint32_t* n_dev, const uint32_t* __restrict__ sorted_prim,
                            const float* __restrict__ verts, const int* __restrict__ faces,
                            float4* tris, float* triv, int leaf_base) {
    const int n = (int)*n_dev;
    int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    int f = (int)sorted_prim[p];
    const float* a = verts + 3 * faces[3 * f];
    const float* b = verts + 3 * faces[3 * f + 1];
    const float* c = verts + 3 * faces[3 * f + 2];
    d3 A = mkd(a[0], a[1], a[2]), B = mkd(b[0], b[1], b[2]), C = mkd(c[0], c[1], c[2]);
    d3 E1 = subd(B, A), E2 = subd(C, A), E3 = subd(C, B);
    d3 N = crossd(E1, E2);
    double two_area = sqrt(dotd(N, N));
    double lmax = fmax(sqrt(dotd(E1, E1)), fmax(sqrt(dotd(E2, E2)), sqrt(dotd(E3, E3))));
    // min altitude = 2A / longest edge; store its inverse, rounded up
    float inv_min_alt = (float)(lmax / two_area) * 1.000001f;
    int g = leaf_base + p;
    tris[3 * g + 0] = make_float4(a[0], a[1], a[2], inv_min_alt);
    tris[3 * g + 1] = make_float4((float)E1.x, (float)E1.y, (float)E1.z, (float)two_area);
    tris[3 * g + 2] = make_float4((float)E2.x, (float)E2.y, (float)E2.z, __int_as_float(f));
    for (int k = 0; k < 3; ++k) {
        triv[9 * g + k] = a[k];
        triv[9 * g + 3 + k] = b[k];
        triv[9 * g + 6 + k] = c[k];
    }
}

__global__ void k_asset_info(const uint32_t* n_dev, int F, const uint32_t* bounds, const float* ibox,
                             const float* tri_box, const uint32_t* sorted_prim, const int* depth,
                             int node_base, int leaf_base, AssetInfo* info) {
    const int n = (int)*n_dev;
    AssetInfo a;
    a.node_base = node_base;
    a.leaf_base = leaf_base;
    a.n_leaves = n;
    a.n_faces = F;
    a.radius = ordered_to_float(bounds[6]);
    a.depth = n > 1 ? *depth + 0 : 1;
    if (n > 1) {
        for (int k = 0; k < 3; ++k) { a.lo[k] = ibox[k]; a.hi[k] = ibox[3 + k]; }
    } else if (n == 1) {
        const float* b = tri_box + 6 * sorted_prim[0];
        for (int k = 0; k < 3; ++k) { a.lo[k] = b[k]; a.hi[k] = b[3 + k]; }
    } else {
        for (int k = 0; k < 3; ++k) { a.lo[k] = 0.0f; a.hi[k] = 0.0f; }
    }
    *info = a;
}

}  // namespace

size_t blas_scratch_bytes(int F) {
    size_t nb = (F + RS_TILE - 1) / RS_TILE;
    int Fi = F > 1 ? F - 1 : 1;
    return align_up(sizeof(float) * 6 * F) + align_up(32) + 4 * align_up(sizeof(uint32_t) * F) +
           align_up(sizeof(uint32_t) * 256 * nb) + align_up(sizeof(int) * 2 * Fi) +
           align_up(sizeof(int) * Fi) + align_up(sizeof(int) * F) + align_up(sizeof(float) * 6 * Fi) +
           align_up(sizeof(int) * Fi) + align_up(sizeof(int)) + align_up(sizeof(float) * Fi) + 256;
}

cudaError_t blas_build(const BlasBuildArgs& a, void* scratch, int* n_leaves_out,
                       cudaStream_t stream) {
    const int F = a.n_faces;
    Scratch s = carve(scratch, F);
    int gb = (F + T_BLK - 1) / T_BLK;
    int gv = (a.n_verts + T_BLK - 1) / T_BLK;
    k_init_bounds<<<1, 32, 0, stream>>>(s.bounds);
    k_tri_prep<<<max(gb, gv), T_BLK, 0, stream>>>(a.verts, a.faces, F, a.n_verts, s.tri_box,
                                                 s.vals[1], s.bounds);
    k_morton<<<gb, T_BLK, 0, stream>>>(s.tri_box, s.vals[1], F, s.bounds, s.keys[0], s.vals[0]);
    int nb = (F + RS_TILE - 1) / RS_TILE;
    int cur = 0;
    for (int shift = 0; shift < 32; shift += 8) {
        k_rs_hist<<<nb, RS_THREADS, 0, stream>>>(s.keys[cur], F, shift, s.hist, nb);
        k_rs_scan<<<1, 1024, 0, stream>>>(s.hist, 256 * nb);
        k_rs_scatter<<<nb, RS_THREADS, 0, stream>>>(s.keys[cur], s.vals[cur], s.keys[cur ^ 1],
                                                    s.vals[cur ^ 1], F, shift, s.hist, nb);
        cur ^= 1;
    }
    // everything below is sized by F and reads the number of non-degenerate
    // leaves n from the device (no host round trip: updates stay async)
    const uint32_t* n_dev = s.bounds + 7;
    if (a.dbg_morton)
        cudaMemcpyAsync(a.dbg_morton, s.keys[cur], sizeof(uint32_t) * F, cudaMemcpyDeviceToDevice, stream);
    const uint32_t* sk = s.keys[cur];
    const uint32_t* sv = s.vals[cur];
    cudaMemsetAsync(s.depth, 0, sizeof(int), stream);
    const int Fi = F > 1 ? F - 1 : 1;
    cudaMemsetAsync(s.flags, 0, sizeof(int) * Fi, stream);
    k_karras<<<(Fi + T_BLK - 1) / T_BLK, T_BLK, 0, stream>>>(sk, n_dev, s.child, s.node_parent, s.leaf_parent);
    k_fit<<<(F + T_BLK - 1) / T_BLK, T_BLK, 0, stream>>>(n_dev, sv, s.tri_box, s.child, s.node_parent,
                                                        s.leaf_parent, s.ibox, s.flags, s.depth);
    for (int round = 0; round < a.trbvh_rounds; ++round) {
        cudaMemsetAsync(s.flags, 0, sizeof(int) * Fi, stream);
        k_trbvh<<<(F + 63) / 64, 64, 0, stream>>>(n_dev, sv, s.tri_box, s.child, s.node_parent, s.leaf_parent,
                                                  s.ibox, s.cost, s.flags);
    }
    if (a.trbvh_rounds > 0) {
        cudaMemsetAsync(s.depth, 0, sizeof(int), stream);
        k_depth<<<(F + T_BLK - 1) / T_BLK, T_BLK, 0, stream>>>(n_dev, s.leaf_parent, s.node_parent, s.depth);
    }
    k_pack_nodes<<<(Fi + T_BLK - 1) / T_BLK, T_BLK, 0, stream>>>(n_dev, sv, s.tri_box, s.child, s.ibox,
                                                                a.bnodes, a.node_base, a.leaf_base);
    k_collapse4<<<(Fi + T_BLK - 1) / T_BLK, T_BLK, 0, stream>>>(n_dev, sv, s.tri_box, s.child, s.ibox,
                                                               a.nodes, a.node_base, a.leaf_base);
    k_pack_tris<<<(F + T_BLK - 1) / T_BLK, T_BLK, 0, stream>>>(n_dev, sv, a.verts, a.faces, a.tris,
                                                              a.triv, a.leaf_base);
    k_asset_info<<<1, 1, 0, stream>>>(n_dev, F, s.bounds, s.ibox, s.tri_box, sv, s.depth, a.node_base,
                                      a.leaf_base, a.info_dev);
    if (n_leaves_out) *n_leaves_out = -1;  // known on the device only
    return cudaGetLastError();
}


}  // namespace agr
