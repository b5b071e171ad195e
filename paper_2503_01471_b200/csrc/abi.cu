// abi.cu -- the C ABI of libagr.so (include/agr.h) and the scene runtime
// behind it: argument validation, device memory ownership, BLAS build at
// create, TLAS build/refit, cast dispatch, the host-buffer end-to-end path
// and debug/introspection hooks.  SURVEY.md §8(b) is the contract.
#include "../../include/agr.h"
#include "agr_internal.cuh"

#include <nvtx3/nvToolsExt.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

using namespace agr;

namespace {

thread_local std::string g_err;

agr_status fail(agr_status s, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
agr_status fail(agr_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

agr_status cuda_fail(cudaError_t e, const char* where) {
    return fail(e == cudaErrorMemoryAllocation ? AGR_ENOMEM : AGR_ECUDA, "%s: %s", where,
                cudaGetErrorString(e));
}

#define CK(call)                                            \
    do {                                                    \
        cudaError_t _e = (call);                            \
        if (_e != cudaSuccess) return cuda_fail(_e, #call); \
    } while (0)

// Restores the caller's current device on scope exit.
struct DeviceGuard {
    int prev = -1;
    bool ok = false;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        ok = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// NVTX range over one ABI call (visible in nsys / ncu --nvtx timelines;
// header-only NVTX3, a no-op without a tool attached).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

}  // namespace

struct agr_scene_s {
    int device = 0;
    int n_assets = 0, n_envs = 0, n_parts = 0;
    int64_t n_inst = 0, n_items = 0;
    int nb_blas = 0, nt_tlas = 0, n_leaves_cap = 0, max_n = 0;
    std::vector<BlasInfo> h_parts;    // per part (BLAS), refreshed after mesh updates
    std::vector<int> h_part_off;      // [n_assets + 1] parts of each asset
    std::vector<int> h_part_nfaces;   // [n_parts]
    std::vector<int64_t> h_part_foff; // [n_parts] first face of the part in part_faces (-1: the asset's
                                      // own face array, single-part assets)
    std::vector<int> h_env_off;
    std::vector<int> h_item_off;      // [n_envs + 1] TLAS items (instance, part) of each env
    std::vector<int> h_tlas_off;
    std::vector<void*> allocs;
    size_t device_bytes = 0;
    // device arrays
    float4* nodes = nullptr;   // BVH4 (BLAS then TLAS), 8 float4 per node
    float4* nodesw = nullptr;  // BVH8 / BVH16 copy (BLAS compacted, roots / TLAS at the BVH4's indices), or null
    int wide_w = 0;            // its width (2 wide_w float4 per node)
    float4* bnodes = nullptr;  // binary BLAS nodes, 4 float4 per node (debug export)
    float4* tris = nullptr;
    float* triv = nullptr;
    float4* irec = nullptr;    // per item
    float* inst_T = nullptr;
    float* item_box = nullptr;
    int* item_inst = nullptr;
    int* item_part = nullptr;
    int* item_off = nullptr;
    int* inst_asset = nullptr;
    int* inst_label = nullptr;
    int* inst_face_off = nullptr;
    int* env_off = nullptr;
    int* tlas_off = nullptr;
    int* tlas_root = nullptr;
    int* tlas_child = nullptr;
    int* tlas_item_parent = nullptr;
    int* tlas_node_parent = nullptr;
    int* tlas_refs4 = nullptr;  // collapses chosen by the last agr_build, kept by agr_refit
    int* tlas_refsw = nullptr;
    int* tlas_depth = nullptr;
    BlasInfo* parts = nullptr;      // [n_parts]
    int* part_off = nullptr;        // [n_assets + 1]
    int* part_faces = nullptr;      // gathered face triples of the multi-part assets, by part
    int* part_face_ids = nullptr;   // their asset-local face ids
    uint32_t* morton = nullptr;  // sorted BLAS Morton codes (debug export)
    // asset meshes kept on the device for BLAS rebuilds (agr_update_mesh)
    float* mesh_verts = nullptr;
    int* mesh_faces = nullptr;
    int* asset_voff = nullptr;  // [n_assets] first vertex / face of each asset (device)
    int* asset_foff = nullptr;
    float* annot = nullptr;     // [sum V][annot_k] vertex annotations, NaN = none
    int annot_k = 0;
    void* blas_scratch = nullptr;
    void* blas_stage = nullptr;          // pinned upload staging of the BLAS batch tables
    size_t blas_stage_bytes = 0;
    cudaEvent_t blas_stage_free = nullptr;
    std::vector<int64_t> h_mvert_off, h_mface_off;
    std::vector<int> h_node_base, h_leaf_base, h_nverts, h_nfaces;
    std::vector<char> h_bin_stale;  // binary LBVH export out of date (mesh updated)
    bool parts_stale = false;       // h_parts out of date (mesh updated)
    int trbvh_rounds = 3;
    unsigned long long* counters = nullptr;
    bool built = false, dirty = false;
    int exact = 0;
    float stereo[3] = {0.0f, -0.095f, 0.0f};
    float stereo_eps = 1e-4f;
    int traversal = 0;  // 0 auto (interval packets for pinhole / beams, on the BVH8 if built;
                        //   per-lane for wide-tile pinholes, set_schedule),
                        // 1 per-lane, 2 interval packets on the BVH4
    int tlas_builder = 0;  // 0 LBVH (default), 1 binned SAH
    bool counting = false;
    // end-to-end staging (lazily allocated)
    // recorded on the caller's stream after every call that changes scene
    // data (transforms, meshes, annotations, build, refit): the host-buffer
    // casts run on internal streams and wait on it first
    cudaEvent_t ready = nullptr;
    cudaStream_t e2e_stream[2] = {nullptr, nullptr};
    cudaEvent_t e2e_event[4] = {nullptr, nullptr, nullptr, nullptr};
    float* e2e_poses = nullptr;
    size_t e2e_poses_bytes = 0;
    void* e2e_out[2] = {nullptr, nullptr};
    size_t e2e_out_bytes = 0;
    void* e2e_host[2] = {nullptr, nullptr};
    size_t e2e_host_bytes = 0;
    float* e2e_beams = nullptr;
    size_t e2e_beams_bytes = 0;

    template <class T>
    cudaError_t alloc(T** p, size_t n) {
        size_t bytes = sizeof(T) * (n > 0 ? n : 1);
        cudaError_t e = cudaMalloc((void**)p, bytes);
        if (e == cudaSuccess) {
            allocs.push_back(*p);
            device_bytes += bytes;
        }
        return e;
    }

    SceneView view() const {
        SceneView v;
        v.nodes = nodes;
        v.nodesw = nodesw;
        v.wide_w = wide_w;
        v.tris = tris;
        v.triv = triv;
        v.irec = irec;
        v.inst_T = inst_T;
        v.inst_face_off = inst_face_off;
        v.inst_label = inst_label;
        v.env_off = env_off;
        v.tlas_root = tlas_root;
        v.inst_asset = inst_asset;
        v.parts = parts;
        v.part_off = part_off;
        v.n_envs = n_envs;
        v.annot = annot;
        v.annot_k = annot_k;
        v.mesh_faces = mesh_faces;
        v.asset_voff = asset_voff;
        v.asset_foff = asset_foff;
        return v;
    }

    TlasArgs tlas_args() const {
        TlasArgs a;
        a.nodes = nodes;
        a.nodesw = nodesw;
        a.wide_w = wide_w;
        a.irec = irec;
        a.item_box = item_box;
        a.inst_T = inst_T;
        a.item_inst = item_inst;
        a.item_part = item_part;
        a.parts = parts;
        a.item_off = item_off;
        a.tlas_off = tlas_off;
        a.nb_blas = nb_blas;
        a.tlas_child = tlas_child;
        a.tlas_item_parent = tlas_item_parent;
        a.tlas_node_parent = tlas_node_parent;
        a.tlas_refs4 = tlas_refs4;
        a.tlas_refsw = tlas_refsw;
        a.tlas_depth = tlas_depth;
        a.n_envs = n_envs;
        a.max_n = max_n;
        a.builder = tlas_builder;
        return a;
    }

    void release() {
        for (void* p : allocs) cudaFree(p);
        allocs.clear();
        for (auto& s : e2e_stream)
            if (s) cudaStreamDestroy(s);
        for (auto& e : e2e_event)
            if (e) cudaEventDestroy(e);
        if (ready) cudaEventDestroy(ready);
        if (blas_stage) cudaFreeHost(blas_stage);
        if (blas_stage_free) cudaEventDestroy(blas_stage_free);
        for (auto& h : e2e_host)
            if (h) cudaFreeHost(h);
        if (e2e_poses) cudaFree(e2e_poses);
        if (e2e_beams) cudaFree(e2e_beams);
        for (auto& o : e2e_out)
            if (o) cudaFree(o);
    }
};

// (Re)build the BLAS of every part of the assets `assets[0, n)` from the
// device copy of their meshes, in one batch (async on st).  `binary`: also
// pack the binary LBVH nodes for agr_debug_export_blas (the create-time build
// only; mesh updates skip it and mark the asset's binary export stale).
static cudaError_t build_assets(agr_scene_s* s, const int* assets, int n, cudaStream_t st, bool binary) {
    std::vector<BlasSeg> segs;
    for (int k = 0; k < n; ++k) {
        const int a = assets[k];
        for (int p = s->h_part_off[a]; p < s->h_part_off[a + 1]; ++p) {
            BlasSeg g;
            g.verts = s->mesh_verts + 3 * s->h_mvert_off[a];
            g.n_verts = s->h_nverts[a];
            if (s->h_part_foff[p] < 0) {  // the whole asset
                g.faces = s->mesh_faces + 3 * s->h_mface_off[a];
                g.face_ids = nullptr;
            } else {
                g.faces = s->part_faces + 3 * s->h_part_foff[p];
                g.face_ids = s->part_face_ids + s->h_part_foff[p];
            }
            g.n_faces = s->h_part_nfaces[p];
            g.off = 0;
            g.node_base = s->h_node_base[p];
            g.leaf_base = s->h_leaf_base[p];
            g.info = s->parts + p;
            segs.push_back(g);
        }
    }
    BlasBatchArgs ba;
    ba.nodes = s->nodes;
    ba.nodesw = s->nodesw;
    ba.wide_w = s->wide_w;
    ba.bnodes = binary ? s->bnodes : nullptr;
    ba.tris = s->tris;
    ba.triv = s->triv;
    ba.dbg_morton = s->morton;
    ba.trbvh_rounds = s->trbvh_rounds;
    // the SAH-optimal BVH8 collapse costs a bottom-up pass more (+1.5 ms per
    // 8.4 M triangles): static assets get it at create, mesh updates keep the
    // greedy collapse
    ba.opt_collapse = binary ? 1 : 0;
    ba.h_stage = s->blas_stage;
    ba.h_stage_bytes = s->blas_stage_bytes;
    ba.stage_free = s->blas_stage_free;
    return blas_build_batch(segs.data(), (int)segs.size(), ba, s->blas_scratch, st);
}

static agr_status refresh_parts(agr_scene_s* s) {
    if (!s->parts_stale) return AGR_OK;
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(s->h_parts.data(), s->parts, sizeof(BlasInfo) * s->n_parts, cudaMemcpyDeviceToHost));
    s->parts_stale = false;
    return AGR_OK;
}

// Partition of an asset's faces into BLAS parts (DESIGN.md §8 "instance
// parts"): connected components of the face-vertex graph (union-find),
// merged greedily -- the pair whose union box grows the summed box surface
// area least -- down to MAX_PARTS; kept only if the parts' boxes have less
// than PART_SA_RATIO of the whole asset's box surface area (a random ray
// crosses a box with probability ~ its area, so that many fewer entries).
// Returns the part of every face (0 .. n_parts - 1, numbered by first face).
constexpr double PART_SA_RATIO = 0.85;
constexpr int PART_MAX_COMPONENTS = 64;

static std::vector<int> asset_parts(const agr_mesh& m, int* n_parts) {
    const int F = m.n_faces, V = m.n_verts;
    std::vector<int> part(F, 0);
    *n_parts = 1;
    std::vector<int> up(V);
    for (int v = 0; v < V; ++v) up[v] = v;
    auto find = [&](int x) {
        while (up[x] != x) x = up[x] = up[up[x]];
        return x;
    };
    for (int f = 0; f < F; ++f)
        for (int c = 1; c < 3; ++c) {
            const int a = find(m.faces[3 * f]), b = find(m.faces[3 * f + c]);
            if (a != b) up[a] = b;
        }
    std::vector<int> comp_of_root(V, -1), comp(F);
    int k = 0;
    for (int f = 0; f < F; ++f) {
        const int r = find(m.faces[3 * f]);
        if (comp_of_root[r] < 0) {
            if (k == PART_MAX_COMPONENTS) return part;  // a triangle soup: one part
            comp_of_root[r] = k++;
        }
        comp[f] = comp_of_root[r];
    }
    if (k < 2) return part;
    struct Box { double lo[3], hi[3]; };
    auto area = [](const Box& b) {
        const double dx = b.hi[0] - b.lo[0], dy = b.hi[1] - b.lo[1], dz = b.hi[2] - b.lo[2];
        return dx * dy + dy * dz + dz * dx;
    };
    auto join = [](const Box& a, const Box& b) {
        Box r;
        for (int c = 0; c < 3; ++c) { r.lo[c] = std::min(a.lo[c], b.lo[c]); r.hi[c] = std::max(a.hi[c], b.hi[c]); }
        return r;
    };
    std::vector<Box> box(k, Box{{1e300, 1e300, 1e300}, {-1e300, -1e300, -1e300}});
    Box all{{1e300, 1e300, 1e300}, {-1e300, -1e300, -1e300}};
    for (int f = 0; f < F; ++f)
        for (int c = 0; c < 3; ++c) {
            const float* v = m.verts + 3 * m.faces[3 * f + c];
            for (int q = 0; q < 3; ++q) {
                box[comp[f]].lo[q] = std::min(box[comp[f]].lo[q], (double)v[q]);
                box[comp[f]].hi[q] = std::max(box[comp[f]].hi[q], (double)v[q]);
            }
        }
    for (auto& b : box) all = join(all, b);
    std::vector<int> group(k);  // component -> group (merged components)
    for (int c = 0; c < k; ++c) group[c] = c;
    int live = k;
    std::vector<char> alive(k, 1);
    while (live > MAX_PARTS) {
        int bi = -1, bj = -1;
        double best = 1e300;
        for (int i = 0; i < k; ++i)
            for (int j = i + 1; j < k; ++j)
                if (alive[i] && alive[j]) {
                    const double g = area(join(box[i], box[j])) - area(box[i]) - area(box[j]);
                    if (g < best) { best = g; bi = i; bj = j; }
                }
        box[bi] = join(box[bi], box[bj]);
        alive[bj] = 0;
        for (int c = 0; c < k; ++c) if (group[c] == bj) group[c] = bi;
        --live;
    }
    double sum = 0.0;
    for (int i = 0; i < k; ++i) if (alive[i]) sum += area(box[i]);
    if (!(sum < PART_SA_RATIO * area(all))) return part;
    // number the parts by their first face
    std::vector<int> id(k, -1);
    int np = 0;
    for (int f = 0; f < F; ++f) {
        const int g = group[comp[f]];
        if (id[g] < 0) id[g] = np++;
        part[f] = id[g];
    }
    *n_parts = np;
    return part;
}

// Marks the end of the scene-changing work just queued on `st` (see `ready`).
// Inside a CUDA-graph capture the record becomes an external event-record
// node, so every replay of the graph re-records `ready`.
static agr_status mark_ready(agr_scene_s* s, cudaStream_t st) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(st, &cap));
    if (cap == cudaStreamCaptureStatusActive)
        CK(cudaEventRecordWithFlags(s->ready, st, cudaEventRecordExternal));
    else
        CK(cudaEventRecord(s->ready, st));
    return AGR_OK;
}

// agr_last_error for the other translation units (sim.cu).
namespace agr {
agr_status set_error(agr_status st, const char* msg) {
    g_err = msg;
    return st;
}
}  // namespace agr

extern "C" {

int32_t agr_abi_version(void) { return AGR_ABI_VERSION; }

const char* agr_last_error(void) { return g_err.c_str(); }

agr_status agr_scene_create(int32_t device, const agr_mesh* meshes, int32_t n_meshes, int32_t n_envs,
                            const int64_t* env_offsets, const agr_instance* inst, agr_scene* out) {
    return agr_scene_create_ex(device, meshes, n_meshes, n_envs, env_offsets, inst, nullptr, out);
}

agr_status agr_scene_create_ex(int32_t device, const agr_mesh* meshes, int32_t n_meshes, int32_t n_envs,
                               const int64_t* env_offsets, const agr_instance* inst,
                               const agr_create_options* opts, agr_scene* out) {
    NvtxRange nvtx_range("agr_scene_create_ex");
    g_err.clear();
    if (!out) return fail(AGR_EINVAL, "out is NULL");
    *out = nullptr;
    if (!meshes || n_meshes < 1) return fail(AGR_EINVAL, "need at least one mesh");
    if (n_envs < 1 || !env_offsets) return fail(AGR_EINVAL, "need n_envs >= 1 and env_offsets");
    if (env_offsets[0] != 0) return fail(AGR_EINVAL, "env_offsets[0] must be 0");
    for (int e = 0; e < n_envs; ++e) {
        if (env_offsets[e + 1] < env_offsets[e]) return fail(AGR_EINVAL, "env_offsets not monotone at %d", e);
        if (env_offsets[e + 1] - env_offsets[e] > AGR_MAX_INSTANCES_PER_ENV)
            return fail(AGR_EUNSUPPORTED, "env %d has %lld instances (limit %d)", e,
                        (long long)(env_offsets[e + 1] - env_offsets[e]), AGR_MAX_INSTANCES_PER_ENV);
    }
    const int64_t n_inst = env_offsets[n_envs];
    if (n_inst > 0x3FFFFFFF) return fail(AGR_EUNSUPPORTED, "too many instances");
    if (n_inst > 0 && !inst) return fail(AGR_EINVAL, "inst is NULL");
    int64_t faces_total = 0, verts_total = 0;
    for (int a = 0; a < n_meshes; ++a) {
        const agr_mesh& m = meshes[a];
        if (!m.verts || !m.faces || m.n_verts < 3 || m.n_faces < 1)
            return fail(AGR_EINVAL, "mesh %d: need verts, faces, n_verts >= 3, n_faces >= 1", a);
        for (int64_t k = 0; k < 3LL * m.n_verts; ++k)
            if (!std::isfinite(m.verts[k])) return fail(AGR_EINVAL, "mesh %d: non-finite vertex", a);
        for (int64_t k = 0; k < 3LL * m.n_faces; ++k)
            if (m.faces[k] < 0 || m.faces[k] >= m.n_verts)
                return fail(AGR_EINVAL, "mesh %d: face index %d out of range", a, m.faces[k]);
        faces_total += m.n_faces;
        verts_total += m.n_verts;
    }
    if (faces_total > LEAF_MASK - 4) return fail(AGR_EUNSUPPORTED, "too many faces");
    for (int64_t j = 0; j < n_inst; ++j) {
        if (inst[j].asset < 0 || inst[j].asset >= n_meshes)
            return fail(AGR_EINVAL, "instance %lld: asset %d out of range", (long long)j, inst[j].asset);
        if (inst[j].label < 0) return fail(AGR_EINVAL, "instance %lld: negative label", (long long)j);
    }
    int dev_count = 0;
    if (cudaGetDeviceCount(&dev_count) != cudaSuccess || device < 0 || device >= dev_count)
        return fail(AGR_EINVAL, "device %d not available (%d CUDA devices)", device, dev_count);
    DeviceGuard guard(device);
    if (!guard.ok) return fail(AGR_ECUDA, "cudaSetDevice(%d) failed", device);

    if (opts && (opts->trbvh_rounds < 0 || opts->trbvh_rounds > 16))
        return fail(AGR_EINVAL, "trbvh_rounds must be in [0, 16]");
    if (opts && (opts->part_policy < 0 || opts->part_policy > 1))
        return fail(AGR_EINVAL, "part_policy must be 0 (auto) or 1 (one BLAS per asset)");
    if (opts && opts->node_width != 0 && opts->node_width != 4 && opts->node_width != 8 && opts->node_width != 16 &&
        opts->node_width != 32)
        return fail(AGR_EINVAL, "node_width must be 0 (default), 4, 8, 16 or 32");
    agr_scene_s* s = new agr_scene_s();
    s->device = device;
    if (opts) s->trbvh_rounds = opts->trbvh_rounds;
    s->n_assets = n_meshes;
    s->n_envs = n_envs;
    s->n_inst = n_inst;
    // ---- asset parts (one BLAS each) and the TLAS items (instance, part) ----
    std::vector<std::vector<int>> part_of(n_meshes);
    std::vector<int> np_asset(n_meshes, 1);
    if (!opts || opts->part_policy == 0)
        for (int a = 0; a < n_meshes; ++a) part_of[a] = asset_parts(meshes[a], &np_asset[a]);
    // a split that would push an env past the one-CTA TLAS limit is dropped
    for (int e = 0; e < n_envs; ++e) {
        int64_t items = 0;
        for (int64_t j = env_offsets[e]; j < env_offsets[e + 1]; ++j) items += np_asset[inst[j].asset];
        if (items > MAX_TLAS_N) {
            for (int a = 0; a < n_meshes; ++a) np_asset[a] = 1;
            break;
        }
    }
    s->h_part_off.assign(n_meshes + 1, 0);
    for (int a = 0; a < n_meshes; ++a) s->h_part_off[a + 1] = s->h_part_off[a] + np_asset[a];
    const int n_parts = s->h_part_off[n_meshes];
    s->n_parts = n_parts;
    // gathered faces of the multi-part assets, part by part, faces ascending
    std::vector<int> h_pfaces, h_pface_ids;
    s->h_part_nfaces.assign(n_parts, 0);
    s->h_part_foff.assign(n_parts, -1);
    for (int a = 0; a < n_meshes; ++a) {
        const int p0 = s->h_part_off[a];
        if (np_asset[a] == 1) {
            s->h_part_nfaces[p0] = meshes[a].n_faces;
            continue;
        }
        for (int p = 0; p < np_asset[a]; ++p) {
            s->h_part_foff[p0 + p] = (int64_t)h_pface_ids.size();
            for (int f = 0; f < meshes[a].n_faces; ++f)
                if (part_of[a][f] == p) {
                    for (int c = 0; c < 3; ++c) h_pfaces.push_back(meshes[a].faces[3 * f + c]);
                    h_pface_ids.push_back(f);
                    ++s->h_part_nfaces[p0 + p];
                }
        }
    }
    std::vector<int> node_base(n_parts), leaf_base(n_parts);
    int nb = 0, nl = 0;
    for (int p = 0; p < n_parts; ++p) {
        node_base[p] = nb;
        leaf_base[p] = nl;
        nb += s->h_part_nfaces[p] > 1 ? s->h_part_nfaces[p] - 1 : 1;
        nl += s->h_part_nfaces[p];
    }
    s->nb_blas = nb;
    s->n_leaves_cap = nl;
    s->h_env_off.resize(n_envs + 1);
    s->h_item_off.resize(n_envs + 1);
    s->h_tlas_off.resize(n_envs);
    std::vector<int> h_item_inst, h_item_part;
    int nt = 0, max_n = 0;
    for (int e = 0; e < n_envs; ++e) {
        s->h_env_off[e] = (int)env_offsets[e];
        s->h_item_off[e] = (int)h_item_inst.size();
        for (int64_t j = env_offsets[e]; j < env_offsets[e + 1]; ++j)
            for (int p = s->h_part_off[inst[j].asset]; p < s->h_part_off[inst[j].asset + 1]; ++p) {
                h_item_inst.push_back((int)j);
                h_item_part.push_back(p);
            }
        const int n = (int)h_item_inst.size() - s->h_item_off[e];
        s->h_tlas_off[e] = nt;
        nt += n > 1 ? n - 1 : 1;
        max_n = n > max_n ? n : max_n;
    }
    s->h_env_off[n_envs] = (int)n_inst;
    const int64_t n_items = (int64_t)h_item_inst.size();
    s->h_item_off[n_envs] = (int)n_items;
    s->n_items = n_items;
    s->nt_tlas = nt;
    s->max_n = max_n;
    std::vector<int> h_asset(n_inst), h_label(n_inst), h_face_off(n_inst), h_root(n_envs);
    for (int e = 0; e < n_envs; ++e) {
        int off = 0;
        for (int64_t j = env_offsets[e]; j < env_offsets[e + 1]; ++j) {
            h_asset[j] = inst[j].asset;
            h_label[j] = inst[j].label;
            h_face_off[j] = off;
            off += meshes[inst[j].asset].n_faces;
        }
        h_root[e] = nb + s->h_tlas_off[e];
    }

    auto bail = [&](agr_status st) {
        s->release();
        delete s;
        return st;
    };
#define CKB(call)                                                    \
    do {                                                             \
        cudaError_t _e = (call);                                     \
        if (_e != cudaSuccess) return bail(cuda_fail(_e, #call));    \
    } while (0)

    CKB(s->alloc(&s->nodes, 8 * (size_t)(nb + nt)));
    // node_width 0: BVH32 (c3's 91-item envs: BVH16 +3.5 % over BVH8,
    // BVH32 +1.3 % over BVH16; c4 / c5's 16-20-item envs: one 32-wide TLAS
    // node, built without DP tables: c4 +1.8 %, c5 +3.6 % over BVH8)
    s->wide_w = !opts || opts->node_width == 0 ? 32 : opts->node_width == 4 ? 0 : opts->node_width;
    if (s->wide_w) CKB(s->alloc(&s->nodesw, (size_t)2 * s->wide_w * (nb + nt)));
    CKB(s->alloc(&s->bnodes, 4 * (size_t)nb));
    CKB(s->alloc(&s->tris, 3 * (size_t)nl));
    CKB(s->alloc(&s->triv, 12 * (size_t)nl));  // 3 x float4 (v.xyz, 0) per leaf
    CKB(s->alloc(&s->irec, 4 * (size_t)n_items));
    CKB(s->alloc(&s->inst_T, 12 * (size_t)n_inst));
    CKB(s->alloc(&s->item_box, 6 * (size_t)n_items));
    CKB(s->alloc(&s->item_inst, (size_t)n_items));
    CKB(s->alloc(&s->item_part, (size_t)n_items));
    CKB(s->alloc(&s->item_off, (size_t)n_envs + 1));
    CKB(s->alloc(&s->inst_asset, (size_t)n_inst));
    CKB(s->alloc(&s->inst_label, (size_t)n_inst));
    CKB(s->alloc(&s->inst_face_off, (size_t)n_inst));
    CKB(s->alloc(&s->env_off, (size_t)n_envs + 1));
    CKB(s->alloc(&s->tlas_off, (size_t)n_envs));
    CKB(s->alloc(&s->tlas_root, (size_t)n_envs));
    CKB(s->alloc(&s->tlas_child, 2 * (size_t)nt));
    CKB(s->alloc(&s->tlas_item_parent, (size_t)n_items));
    CKB(s->alloc(&s->tlas_node_parent, (size_t)nt));
    CKB(s->alloc(&s->tlas_refs4, 4 * (size_t)nt));
    if (s->wide_w) CKB(s->alloc(&s->tlas_refsw, (size_t)s->wide_w * nt));
    CKB(s->alloc(&s->tlas_depth, (size_t)n_envs));
    CKB(s->alloc(&s->parts, (size_t)n_parts));
    CKB(s->alloc(&s->part_off, (size_t)n_meshes + 1));
    CKB(s->alloc(&s->part_faces, h_pfaces.size()));
    CKB(s->alloc(&s->part_face_ids, h_pface_ids.size()));
    CKB(s->alloc(&s->morton, (size_t)nl));
    CKB(s->alloc(&s->counters, 8));
    CKB(cudaMemset(s->morton, 0xFF, sizeof(uint32_t) * (size_t)nl));
    CKB(cudaMemset(s->tris, 0, sizeof(float4) * 3 * (size_t)nl));
    CKB(cudaMemcpy(s->inst_asset, h_asset.data(), sizeof(int) * n_inst, cudaMemcpyHostToDevice));
    CKB(cudaMemcpy(s->inst_label, h_label.data(), sizeof(int) * n_inst, cudaMemcpyHostToDevice));
    CKB(cudaMemcpy(s->inst_face_off, h_face_off.data(), sizeof(int) * n_inst, cudaMemcpyHostToDevice));
    CKB(cudaMemcpy(s->env_off, s->h_env_off.data(), sizeof(int) * (n_envs + 1), cudaMemcpyHostToDevice));
    CKB(cudaMemcpy(s->tlas_off, s->h_tlas_off.data(), sizeof(int) * n_envs, cudaMemcpyHostToDevice));
    CKB(cudaMemcpy(s->tlas_root, h_root.data(), sizeof(int) * n_envs, cudaMemcpyHostToDevice));
    CKB(cudaMemcpy(s->item_inst, h_item_inst.data(), sizeof(int) * n_items, cudaMemcpyHostToDevice));
    CKB(cudaMemcpy(s->item_part, h_item_part.data(), sizeof(int) * n_items, cudaMemcpyHostToDevice));
    CKB(cudaMemcpy(s->item_off, s->h_item_off.data(), sizeof(int) * (n_envs + 1), cudaMemcpyHostToDevice));
    CKB(cudaMemcpy(s->part_off, s->h_part_off.data(), sizeof(int) * (n_meshes + 1), cudaMemcpyHostToDevice));
    if (!h_pfaces.empty()) {
        CKB(cudaMemcpy(s->part_faces, h_pfaces.data(), sizeof(int) * h_pfaces.size(), cudaMemcpyHostToDevice));
        CKB(cudaMemcpy(s->part_face_ids, h_pface_ids.data(), sizeof(int) * h_pface_ids.size(),
                       cudaMemcpyHostToDevice));
    }

    // BLAS build: all asset meshes stay on the device (for agr_update_mesh),
    // and every asset is built in one batch (one set of launches)
    cudaStream_t st;
    CKB(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    s->h_mvert_off.assign(n_meshes + 1, 0);
    s->h_mface_off.assign(n_meshes + 1, 0);
    for (int a = 0; a < n_meshes; ++a) {
        s->h_mvert_off[a + 1] = s->h_mvert_off[a] + meshes[a].n_verts;
        s->h_mface_off[a + 1] = s->h_mface_off[a] + meshes[a].n_faces;
        s->h_nverts.push_back(meshes[a].n_verts);
        s->h_nfaces.push_back(meshes[a].n_faces);
        s->h_bin_stale.push_back(0);
    }
    s->h_node_base = node_base;
    s->h_leaf_base = leaf_base;
    if (s->h_mvert_off[n_meshes] > 0x3FFFFFFF) return bail(fail(AGR_EUNSUPPORTED, "too many vertices"));
    CKB(s->alloc(&s->mesh_verts, 3 * (size_t)s->h_mvert_off[n_meshes]));
    CKB(s->alloc(&s->mesh_faces, 3 * (size_t)s->h_mface_off[n_meshes]));
    {
        std::vector<int> vo(n_meshes), fo(n_meshes);
        for (int a = 0; a < n_meshes; ++a) {
            vo[a] = (int)s->h_mvert_off[a];
            fo[a] = (int)s->h_mface_off[a];
        }
        CKB(s->alloc(&s->asset_voff, n_meshes));
        CKB(s->alloc(&s->asset_foff, n_meshes));
        CKB(cudaMemcpy(s->asset_voff, vo.data(), sizeof(int) * n_meshes, cudaMemcpyHostToDevice));
        CKB(cudaMemcpy(s->asset_foff, fo.data(), sizeof(int) * n_meshes, cudaMemcpyHostToDevice));
    }
    // scratch for a batch of every asset (any update batch fits in it)
    CKB(s->alloc((char**)&s->blas_scratch, blas_scratch_bytes(s->h_mface_off[n_meshes], n_parts, s->wide_w)));
    s->blas_stage_bytes = blas_stage_bytes(s->h_mface_off[n_meshes], n_parts);
    CKB(cudaMallocHost(&s->blas_stage, s->blas_stage_bytes));
    CKB(cudaEventCreateWithFlags(&s->blas_stage_free, cudaEventDisableTiming));
    cudaError_t err = cudaSuccess;
    for (int a = 0; a < n_meshes && err == cudaSuccess; ++a) {
        err = cudaMemcpyAsync(s->mesh_verts + 3 * s->h_mvert_off[a], meshes[a].verts,
                              sizeof(float) * 3 * meshes[a].n_verts, cudaMemcpyHostToDevice, st);
        if (err != cudaSuccess) break;
        err = cudaMemcpyAsync(s->mesh_faces + 3 * s->h_mface_off[a], meshes[a].faces,
                              sizeof(int) * 3 * meshes[a].n_faces, cudaMemcpyHostToDevice, st);
    }
    if (err == cudaSuccess) err = cudaStreamSynchronize(st);  // the host arrays are the caller's
    if (err == cudaSuccess) {
        std::vector<int> all(n_meshes);
        for (int a = 0; a < n_meshes; ++a) all[a] = a;
        err = build_assets(s, all.data(), n_meshes, st, true);
    }
    if (err == cudaSuccess) err = cudaStreamSynchronize(st);
    if (err != cudaSuccess) {
        cudaStreamDestroy(st);
        return bail(cuda_fail(err, "BLAS build"));
    }
    s->h_parts.resize(n_parts);
    CKB(cudaMemcpy(s->h_parts.data(), s->parts, sizeof(BlasInfo) * n_parts, cudaMemcpyDeviceToHost));
    int max_depth = 0;
    for (auto& a : s->h_parts) max_depth = a.depth > max_depth ? a.depth : max_depth;
    // identity transforms until the caller sets them
    {
        std::vector<float> I(12 * (size_t)n_inst, 0.0f);
        for (int64_t j = 0; j < n_inst; ++j) I[12 * j + 0] = I[12 * j + 5] = I[12 * j + 10] = 1.0f;
        CKB(cudaMemcpy(s->inst_T, I.data(), sizeof(float) * I.size(), cudaMemcpyHostToDevice));
    }
    err = items_update(s->tlas_args(), (int)n_items, st);
    if (err == cudaSuccess) err = cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    if (err != cudaSuccess) return bail(cuda_fail(err, "items_update"));
    if (max_depth > AGR_MAX_BVH_DEPTH)
        return bail(fail(AGR_EUNSUPPORTED, "BLAS depth %d exceeds AGR_MAX_BVH_DEPTH (%d)", max_depth,
                         AGR_MAX_BVH_DEPTH));
    CKB(cudaEventCreateWithFlags(&s->ready, cudaEventDisableTiming));
    CKB(cudaEventRecord(s->ready, 0));
#undef CKB
    *out = s;
    return AGR_OK;
}

agr_status agr_scene_destroy(agr_scene s) {
    g_err.clear();
    if (!s) return AGR_OK;
    DeviceGuard guard(s->device);
    cudaDeviceSynchronize();
    s->release();
    delete s;
    return AGR_OK;
}

agr_status agr_scene_get_info(agr_scene s, agr_scene_info* info) {
    g_err.clear();
    if (!s || !info) return fail(AGR_EINVAL, "NULL argument");
    DeviceGuard guard(s->device);
    info->n_assets = s->n_assets;
    info->n_envs = s->n_envs;
    info->n_instances = s->n_inst;
    info->n_blas_nodes = s->nb_blas;
    agr_status rs = refresh_parts(s);
    if (rs != AGR_OK) return rs;
    int64_t leaves = 0;
    int bd = 0;
    for (auto& a : s->h_parts) {
        leaves += a.n_leaves;
        bd = a.depth > bd ? a.depth : bd;
    }
    info->n_blas_tris = leaves;
    info->n_tlas_nodes = s->nt_tlas;
    info->blas_max_depth = bd;
    info->tlas_max_depth = 0;
    if (s->built) {
        std::vector<int> d(s->n_envs);
        CK(cudaMemcpy(d.data(), s->tlas_depth, sizeof(int) * s->n_envs, cudaMemcpyDeviceToHost));
        for (int x : d) info->tlas_max_depth = x > info->tlas_max_depth ? x : info->tlas_max_depth;
    }
    info->device_bytes = (int64_t)s->device_bytes;
    info->built = s->built ? 1 : 0;
    info->n_parts = s->n_parts;
    info->n_items = s->n_items;
    return AGR_OK;
}

agr_status agr_set_instance_transforms(agr_scene s, const float* T, void* stream) {
    NvtxRange nvtx_range("agr_set_instance_transforms");
    g_err.clear();
    if (!s) return fail(AGR_EINVAL, "scene is NULL");
    if (s->n_inst == 0) return AGR_OK;
    if (!T) return fail(AGR_EINVAL, "T is NULL");
    DeviceGuard guard(s->device);
    cudaStream_t st = (cudaStream_t)stream;
    CK(cudaMemcpyAsync(s->inst_T, T, sizeof(float) * 12 * s->n_inst, cudaMemcpyDeviceToDevice, st));
    CK(items_update(s->tlas_args(), (int)s->n_items, st));
    s->dirty = true;
    return mark_ready(s, st);
}

agr_status agr_update_mesh(agr_scene s, int32_t asset, const float* verts, int32_t n_verts, void* stream) {
    g_err.clear();
    if (!s) return fail(AGR_EINVAL, "scene is NULL");
    if (asset < 0 || asset >= s->n_assets) return fail(AGR_EINVAL, "asset %d out of range", asset);
    if (!verts || n_verts != s->h_nverts[asset])
        return fail(AGR_EINVAL, "asset %d has %d vertices (got %d)", asset, s->h_nverts[asset], n_verts);
    return agr_update_meshes(s, 1, &asset, verts, stream);
}

agr_status agr_update_meshes(agr_scene s, int32_t n, const int32_t* assets, const float* verts, void* stream) {
    NvtxRange nvtx_range("agr_update_meshes");
    g_err.clear();
    if (!s) return fail(AGR_EINVAL, "scene is NULL");
    if (n == 0) return AGR_OK;
    if (n < 0 || !assets || !verts) return fail(AGR_EINVAL, "need n > 0, assets and verts");
    std::vector<char> seen(s->n_assets, 0);
    for (int k = 0; k < n; ++k) {
        if (assets[k] < 0 || assets[k] >= s->n_assets) return fail(AGR_EINVAL, "asset %d out of range", assets[k]);
        if (seen[assets[k]]) return fail(AGR_EINVAL, "asset %d listed twice", assets[k]);
        seen[assets[k]] = 1;
    }
    DeviceGuard guard(s->device);
    cudaStream_t st = (cudaStream_t)stream;
    // one copy per run of consecutive asset ids (their vertex arrays are
    // contiguous on both sides): a whole-scene reset is a single copy
    int64_t v = 0;
    for (int k = 0; k < n;) {
        const int a0 = assets[k];
        int64_t nv = s->h_nverts[a0];
        int k1 = k + 1;
        while (k1 < n && assets[k1] == assets[k1 - 1] + 1) nv += s->h_nverts[assets[k1++]];
        CK(cudaMemcpyAsync(s->mesh_verts + 3 * s->h_mvert_off[a0], verts + 3 * v, sizeof(float) * 3 * nv,
                           cudaMemcpyDeviceToDevice, st));
        v += nv;
        k = k1;
    }
    CK(build_assets(s, assets, n, st, false));
    for (int k = 0; k < n; ++k) s->h_bin_stale[assets[k]] = 1;
    CK(items_update(s->tlas_args(), (int)s->n_items, st));  // item boxes from the new BLAS
    s->parts_stale = true;
    s->dirty = true;
    return mark_ready(s, st);
}

agr_status agr_set_vertex_annotations(agr_scene s, int32_t asset, const float* values, int32_t n_verts,
                                      int32_t k, void* stream) {
    g_err.clear();
    if (!s) return fail(AGR_EINVAL, "scene is NULL");
    if (asset < 0 || asset >= s->n_assets) return fail(AGR_EINVAL, "asset %d out of range", asset);
    if (!values || n_verts != s->h_nverts[asset])
        return fail(AGR_EINVAL, "asset %d has %d vertices (got %d)", asset, s->h_nverts[asset], n_verts);
    if (k < 1 || k > AGR_MAX_ANNOT) return fail(AGR_EINVAL, "k must be in [1, %d]", AGR_MAX_ANNOT);
    if (s->annot_k != 0 && k != s->annot_k)
        return fail(AGR_EINVAL, "the scene's annotations have k = %d (got %d)", s->annot_k, k);
    DeviceGuard guard(s->device);
    cudaStream_t st = (cudaStream_t)stream;
    if (!s->annot) {
        const size_t n = (size_t)k * s->h_mvert_off[s->n_assets];
        CK(s->alloc(&s->annot, n));
        CK(cudaMemsetAsync(s->annot, 0xFF, sizeof(float) * n, st));  // all-ones bits: NaN
        s->annot_k = k;
    }
    CK(cudaMemcpyAsync(s->annot + (size_t)k * s->h_mvert_off[asset], values, sizeof(float) * k * (size_t)n_verts,
                       cudaMemcpyDeviceToDevice, st));
    return mark_ready(s, st);
}

agr_status agr_build(agr_scene s, void* stream) {
    NvtxRange nvtx_range("agr_build");
    g_err.clear();
    if (!s) return fail(AGR_EINVAL, "scene is NULL");
    DeviceGuard guard(s->device);
    CK(tlas_build(s->tlas_args(), true, (cudaStream_t)stream));
    s->built = true;
    s->dirty = false;
    return mark_ready(s, (cudaStream_t)stream);
}

agr_status agr_refit(agr_scene s, void* stream) {
    NvtxRange nvtx_range("agr_refit");
    g_err.clear();
    if (!s) return fail(AGR_EINVAL, "scene is NULL");
    if (!s->built) return fail(AGR_ESTATE, "agr_refit before the first agr_build");
    DeviceGuard guard(s->device);
    CK(tlas_build(s->tlas_args(), false, (cudaStream_t)stream));
    s->dirty = false;
    return mark_ready(s, (cudaStream_t)stream);
}

static agr_status check_cast_state(agr_scene s, float max_range, const agr_outputs& out) {
    if (!s) return fail(AGR_EINVAL, "scene is NULL");
    if (out.annot && s->annot_k == 0) return fail(AGR_EINVAL, "annot requested but no vertex annotations set");
    if (!s->built) return fail(AGR_ESTATE, "cast before the first agr_build");
    if (s->dirty) return fail(AGR_ESTATE, "transforms changed since the last agr_build/agr_refit");
    if (!(max_range > 0.0f) || !std::isfinite(max_range)) return fail(AGR_EINVAL, "max_range must be > 0");
    return AGR_OK;
}

// Interval packets pay when a 4x8 tile's rays are nearly parallel: with the
// tile spanning more than ~0.12 rad (a pinhole with fx, fy below ~67 px:
// 8x8 .. 64x64 images at 87 deg hfov) the direction interval culls little
// and the warp walks most of the env, one slow packet per tile, while
// independent lanes finish 1.4-5x sooner (bench.py --table2).
// Mode 0 (auto) therefore casts such cameras one ray per lane.
constexpr float PACKET_MAX_TILE_RAD = 0.12f;

static void set_schedule(const agr_scene_s* s, CastArgs& a) {
    bool packet = s->traversal != 1;
    if (s->traversal == 0 && a.model == 1 &&
        (4.0f / a.fx > PACKET_MAX_TILE_RAD || 8.0f / a.fy > PACKET_MAX_TILE_RAD))
        packet = false;
    a.packet = packet ? 1 : 0;
    a.wide = packet && (s->traversal == 0 || s->traversal == 3) && s->nodesw ? 1 : 0;
}

static agr_status run_cast(agr_scene s, CastArgs& a, cudaStream_t st) {
    a.sv = s->view();
    a.exact = s->exact;
    set_schedule(s, a);
    a.counters = nullptr;
    if (s->counting) {
        CK(cudaMemsetAsync(s->counters, 0, sizeof(unsigned long long) * 8, st));
        a.counters = s->counters;
    }
    CK(cast_launch(a, st));
    return AGR_OK;
}

static CastArgs base_args(agr_scene s, float max_range, agr_outputs out) {
    CastArgs a;
    memset(&a, 0, sizeof a);
    a.max_range = max_range;
    a.out_dist = out.dist;
    a.out_seg = out.seg;
    a.out_face = out.face;
    a.out_normal = out.normal;
    a.out_bary = out.bary;
    a.out_point = out.point;
    a.out_valid = out.valid;
    a.out_annot = out.annot;
    for (int k = 0; k < 3; ++k) a.stereo[k] = s->stereo[k];
    a.stereo_eps = s->stereo_eps;
    a.env_begin = 0;
    a.env_end = s->n_envs;
    a.S = 1;
    return a;
}

agr_status agr_cast_pinhole(agr_scene s, const agr_pinhole* cam, agr_distance kind, const float* poses,
                            int32_t n_sensors, float max_range, agr_outputs out, void* stream) {
    NvtxRange nvtx_range("agr_cast_pinhole");
    g_err.clear();
    agr_status st = check_cast_state(s, max_range, out);
    if (st != AGR_OK) return st;
    if (!cam || !poses || n_sensors < 1) return fail(AGR_EINVAL, "need cam, poses and n_sensors >= 1");
    if (cam->width < 1 || cam->height < 1 || !(cam->fx > 0.0f) || !(cam->fy > 0.0f))
        return fail(AGR_EINVAL, "bad pinhole intrinsics");
    if (kind != AGR_DEPTH && kind != AGR_RANGE) return fail(AGR_EINVAL, "bad distance kind");
    DeviceGuard guard(s->device);
    CastArgs a = base_args(s, max_range, out);
    a.model = 1;
    a.kind = (int)kind;
    a.W = cam->width;
    a.H = cam->height;
    a.fx = cam->fx;
    a.fy = cam->fy;
    a.cx = cam->cx;
    a.cy = cam->cy;
    a.inv_fx64 = 1.0 / (double)cam->fx;
    a.inv_fy64 = 1.0 / (double)cam->fy;
    a.poses = poses;
    a.S = n_sensors;
    return run_cast(s, a, (cudaStream_t)stream);
}

agr_status agr_cast_beams(agr_scene s, const float* dirs, int32_t C, int32_t K, const float* poses,
                          int32_t n_sensors, float max_range, agr_outputs out, void* stream) {
    NvtxRange nvtx_range("agr_cast_beams");
    g_err.clear();
    agr_status st = check_cast_state(s, max_range, out);
    if (st != AGR_OK) return st;
    if (!dirs || !poses || C < 1 || K < 1 || n_sensors < 1)
        return fail(AGR_EINVAL, "need dirs, poses, C, K, n_sensors >= 1");
    DeviceGuard guard(s->device);
    CastArgs a = base_args(s, max_range, out);
    a.model = 2;
    a.W = K;
    a.H = C;
    a.beams = dirs;
    a.poses = poses;
    a.S = n_sensors;
    return run_cast(s, a, (cudaStream_t)stream);
}

agr_status agr_cast_rays(agr_scene s, const float* orig, const float* dir, int32_t R, float max_range,
                         agr_outputs out, void* stream) {
    NvtxRange nvtx_range("agr_cast_rays");
    g_err.clear();
    agr_status st = check_cast_state(s, max_range, out);
    if (st != AGR_OK) return st;
    if (!orig || !dir || R < 1) return fail(AGR_EINVAL, "need orig, dir and R >= 1");
    DeviceGuard guard(s->device);
    CastArgs a = base_args(s, max_range, out);
    a.model = 0;
    a.orig = orig;
    a.dir = dir;
    a.R = R;
    return run_cast(s, a, (cudaStream_t)stream);
}

// ---- end-to-end casts through host buffers ---------------------------------------
static agr_status e2e_prepare(agr_scene s, size_t pose_bytes, size_t chunk_out_bytes) {
    if (!s->e2e_stream[0]) {
        for (auto& x : s->e2e_stream) CK(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
        for (auto& x : s->e2e_event) CK(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    }
    // order the internal streams after the scene work queued on the
    // caller's stream (agr.h: the host casts need no caller-side sync)
    CK(cudaStreamWaitEvent(s->e2e_stream[0], s->ready, 0));
    if (pose_bytes > s->e2e_poses_bytes) {
        if (s->e2e_poses) cudaFree(s->e2e_poses);
        s->e2e_poses = nullptr;
        CK(cudaMalloc(&s->e2e_poses, pose_bytes));
        s->e2e_poses_bytes = pose_bytes;
    }
    if (chunk_out_bytes > s->e2e_out_bytes) {
        for (auto& o : s->e2e_out) {
            if (o) cudaFree(o);
            o = nullptr;
            CK(cudaMalloc(&o, chunk_out_bytes));
        }
        s->e2e_out_bytes = chunk_out_bytes;
    }
    return AGR_OK;
}

static bool is_pinned(const void* p) {
    if (!p) return true;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

// Casts env chunks into a double-buffered device area and streams each chunk
// back to the host while the next one is traced.
#ifndef AGR_E2E_CHUNKS
#define AGR_E2E_CHUNKS 32  // env chunks of a host cast: chunk k + 1 is cast while chunk k is copied back
#endif
#ifndef AGR_E2E_MIN_ELEMS
#define AGR_E2E_MIN_ELEMS (1 << 20)  // rays per chunk at least (so each chunk's cast fills the GPU)
#endif
struct E2EChannel {
    void* host;   // caller's host pointer (whole output)
    int bytes;    // bytes per element
};

static agr_status e2e_run(agr_scene s, CastArgs& a, int64_t elems_per_env, agr_outputs out_host) {
    const int E = s->n_envs;
    constexpr int NCH = 8;
    E2EChannel ch[NCH] = {{out_host.dist, 4}, {out_host.seg, 4}, {out_host.face, 4},
                          {out_host.normal, 12}, {out_host.bary, 8}, {out_host.point, 12},
                          {out_host.valid, 4}, {out_host.annot, 4 * s->annot_k}};
    int64_t bytes_per_elem = 0;
    bool direct = true;
    for (auto& c : ch)
        if (c.host) {
            bytes_per_elem += c.bytes;
            direct = direct && is_pinned(c.host);
        }
    // up to AGR_E2E_CHUNKS chunks of at least AGR_E2E_MIN_ELEMS rays (a
    // smaller cast leaves the GPU in its launch tail: c6's 8-env chunks of
    // 32 ran at 0.87 Grays/s end to end, 8 chunks at 1.19), >= 1 env each
    int64_t n_chunks = (int64_t)E * elems_per_env / AGR_E2E_MIN_ELEMS;
    if (n_chunks > AGR_E2E_CHUNKS) n_chunks = AGR_E2E_CHUNKS;
    if (n_chunks < 1) n_chunks = 1;
    int chunk = (int)((E + n_chunks - 1) / n_chunks);
    if (chunk < 1) chunk = 1;
    size_t chunk_bytes = (size_t)(chunk * elems_per_env * bytes_per_elem);
    agr_status st = e2e_prepare(s, a.S * 12 * sizeof(float) * (size_t)E, chunk_bytes);
    if (st != AGR_OK) return st;
    if (!direct && chunk_bytes > s->e2e_host_bytes) {
        for (auto& h : s->e2e_host) {
            if (h) cudaFreeHost(h);
            h = nullptr;
            CK(cudaMallocHost(&h, chunk_bytes));
        }
        s->e2e_host_bytes = chunk_bytes;
    }
    cudaStream_t cs = s->e2e_stream[0], xs = s->e2e_stream[1];
    int k = 0;
    for (int e0 = 0; e0 < E; e0 += chunk, ++k) {
        int e1 = e0 + chunk < E ? e0 + chunk : E;
        int slot = k & 1;
        if (k >= 2) CK(cudaStreamWaitEvent(cs, s->e2e_event[2 + slot], 0));  // slot drained
        char* base = (char*)s->e2e_out[slot];
        const int64_t n = (int64_t)(e1 - e0) * elems_per_env;
        CastArgs c = a;
        c.env_begin = e0;
        c.env_end = e1;
        c.out_env_base = e0;  // the chunk's outputs start at env e0 of the chunk buffer
        char* dev[NCH];
        char* p = base;
        for (int q = 0; q < NCH; ++q) {
            dev[q] = ch[q].host ? p : nullptr;
            if (ch[q].host) p += ch[q].bytes * n;
        }
        c.out_dist = (float*)dev[0];
        c.out_seg = (int*)dev[1];
        c.out_face = (int*)dev[2];
        c.out_normal = (float*)dev[3];
        c.out_bary = (float*)dev[4];
        c.out_point = (float*)dev[5];
        c.out_valid = (int*)dev[6];
        c.out_annot = (float*)dev[7];
        c.sv = s->view();
        c.exact = s->exact;
        set_schedule(s, c);
        c.counters = nullptr;
        CK(cast_launch(c, cs));
        CK(cudaEventRecord(s->e2e_event[slot], cs));
        CK(cudaStreamWaitEvent(xs, s->e2e_event[slot], 0));
        const int64_t off = (int64_t)e0 * elems_per_env;
        if (direct) {
            for (int q = 0; q < NCH; ++q)
                if (ch[q].host)
                    CK(cudaMemcpyAsync((char*)ch[q].host + off * ch[q].bytes, dev[q], ch[q].bytes * n,
                                       cudaMemcpyDeviceToHost, xs));
            CK(cudaEventRecord(s->e2e_event[2 + slot], xs));
        } else {
            CK(cudaMemcpyAsync(s->e2e_host[slot], base, (size_t)(p - base), cudaMemcpyDeviceToHost, xs));
            CK(cudaEventRecord(s->e2e_event[2 + slot], xs));
            CK(cudaEventSynchronize(s->e2e_event[2 + slot]));
            const char* hsrc = (const char*)s->e2e_host[slot];
            for (int q = 0; q < NCH; ++q)
                if (ch[q].host) {
                    memcpy((char*)ch[q].host + off * ch[q].bytes, hsrc, ch[q].bytes * n);
                    hsrc += ch[q].bytes * n;
                }
        }
    }
    CK(cudaStreamSynchronize(xs));
    CK(cudaStreamSynchronize(cs));
    return AGR_OK;
}

agr_status agr_cast_pinhole_host(agr_scene s, const agr_pinhole* cam, agr_distance kind,
                                 const float* poses_host, int32_t n_sensors, float max_range,
                                 agr_outputs out_host) {
    NvtxRange nvtx_range("agr_cast_pinhole_host");
    g_err.clear();
    agr_status st = check_cast_state(s, max_range, out_host);
    if (st != AGR_OK) return st;
    if (!cam || !poses_host || n_sensors < 1) return fail(AGR_EINVAL, "need cam, poses and n_sensors >= 1");
    if (cam->width < 1 || cam->height < 1 || !(cam->fx > 0.0f) || !(cam->fy > 0.0f))
        return fail(AGR_EINVAL, "bad pinhole intrinsics");
    if (kind != AGR_DEPTH && kind != AGR_RANGE) return fail(AGR_EINVAL, "bad distance kind");
    DeviceGuard guard(s->device);
    st = e2e_prepare(s, sizeof(float) * 12 * (size_t)n_sensors * s->n_envs, 0);
    if (st != AGR_OK) return st;
    CK(cudaMemcpyAsync(s->e2e_poses, poses_host, sizeof(float) * 12 * (size_t)n_sensors * s->n_envs,
                       cudaMemcpyHostToDevice, s->e2e_stream[0]));
    CastArgs a = base_args(s, max_range, agr_outputs{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr});
    a.model = 1;
    a.kind = (int)kind;
    a.W = cam->width;
    a.H = cam->height;
    a.fx = cam->fx;
    a.fy = cam->fy;
    a.cx = cam->cx;
    a.cy = cam->cy;
    a.inv_fx64 = 1.0 / (double)cam->fx;
    a.inv_fy64 = 1.0 / (double)cam->fy;
    a.poses = s->e2e_poses;
    a.S = n_sensors;
    return e2e_run(s, a, (int64_t)n_sensors * cam->width * cam->height, out_host);
}

agr_status agr_cast_beams_host(agr_scene s, const float* dirs_host, int32_t C, int32_t K,
                               const float* poses_host, int32_t n_sensors, float max_range,
                               agr_outputs out_host) {
    NvtxRange nvtx_range("agr_cast_beams_host");
    g_err.clear();
    agr_status st = check_cast_state(s, max_range, out_host);
    if (st != AGR_OK) return st;
    if (!dirs_host || !poses_host || C < 1 || K < 1 || n_sensors < 1)
        return fail(AGR_EINVAL, "need dirs, poses, C, K, n_sensors >= 1");
    DeviceGuard guard(s->device);
    st = e2e_prepare(s, sizeof(float) * 12 * (size_t)n_sensors * s->n_envs, 0);
    if (st != AGR_OK) return st;
    size_t bb = sizeof(float) * 3 * (size_t)C * K;
    if (bb > s->e2e_beams_bytes) {
        if (s->e2e_beams) cudaFree(s->e2e_beams);
        s->e2e_beams = nullptr;
        CK(cudaMalloc(&s->e2e_beams, bb));
        s->e2e_beams_bytes = bb;
    }
    CK(cudaMemcpyAsync(s->e2e_beams, dirs_host, bb, cudaMemcpyHostToDevice, s->e2e_stream[0]));
    CK(cudaMemcpyAsync(s->e2e_poses, poses_host, sizeof(float) * 12 * (size_t)n_sensors * s->n_envs,
                       cudaMemcpyHostToDevice, s->e2e_stream[0]));
    CastArgs a = base_args(s, max_range, agr_outputs{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr});
    a.model = 2;
    a.W = K;
    a.H = C;
    a.beams = s->e2e_beams;
    a.poses = s->e2e_poses;
    a.S = n_sensors;
    return e2e_run(s, a, (int64_t)n_sensors * C * K, out_host);
}

agr_status agr_checksum(agr_scene s, agr_outputs out, int64_t elems_per_env, uint64_t* sums, void* stream) {
    NvtxRange nvtx_range("agr_checksum");
    g_err.clear();
    if (!s || !sums || elems_per_env < 0) return fail(AGR_EINVAL, "bad argument");
    DeviceGuard guard(s->device);
    CK(checksum_launch(out.dist, out.seg, out.face, elems_per_env, s->n_envs,
                       (unsigned long long*)sums, (cudaStream_t)stream));
    return AGR_OK;
}

agr_status agr_set_exact_mode(agr_scene s, int32_t exact) {
    g_err.clear();
    if (!s) return fail(AGR_EINVAL, "scene is NULL");
    s->exact = exact ? 1 : 0;
    return AGR_OK;
}

agr_status agr_set_stereo(agr_scene s, float ox, float oy, float oz, float eps) {
    g_err.clear();
    if (!s) return fail(AGR_EINVAL, "scene is NULL");
    if (!std::isfinite(ox) || !std::isfinite(oy) || !std::isfinite(oz) || !(eps > 0.0f) || !std::isfinite(eps))
        return fail(AGR_EINVAL, "stereo offset must be finite and eps > 0");
    s->stereo[0] = ox;
    s->stereo[1] = oy;
    s->stereo[2] = oz;
    s->stereo_eps = eps;
    return AGR_OK;
}

agr_status agr_set_tlas_builder(agr_scene s, int32_t builder) {
    g_err.clear();
    if (!s) return fail(AGR_EINVAL, "scene is NULL");
    if (builder != 0 && builder != 1) return fail(AGR_EINVAL, "TLAS builder must be 0 (LBVH) or 1 (SAH)");
    s->tlas_builder = builder;
    return AGR_OK;
}

agr_status agr_set_traversal(agr_scene s, int32_t mode) {
    g_err.clear();
    if (!s) return fail(AGR_EINVAL, "scene is NULL");
    if (mode < 0 || mode > 3) return fail(AGR_EINVAL, "traversal mode must be 0, 1, 2 or 3");
    s->traversal = mode;
    return AGR_OK;
}

agr_status agr_enable_counters(agr_scene s, int32_t enable) {
    g_err.clear();
    if (!s) return fail(AGR_EINVAL, "scene is NULL");
    s->counting = enable != 0;
    return AGR_OK;
}

agr_status agr_get_counters(agr_scene s, int64_t counters[8]) {
    g_err.clear();
    if (!s || !counters) return fail(AGR_EINVAL, "bad argument");
    DeviceGuard guard(s->device);
    unsigned long long c[8];
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(c, s->counters, sizeof c, cudaMemcpyDeviceToHost));
    for (int k = 0; k < 8; ++k) counters[k] = (int64_t)c[k];
    return AGR_OK;
}

agr_status agr_debug_export_blas(agr_scene s, int32_t asset, float* nodes, int32_t* leaf_face,
                                 uint32_t* morton, int64_t* n_nodes, int64_t* n_leaves) {
    g_err.clear();
    if (!s || !n_nodes || !n_leaves) return fail(AGR_EINVAL, "bad argument");
    if (asset < 0 || asset >= s->n_assets) return fail(AGR_EINVAL, "asset out of range");
    if (s->h_part_off[asset + 1] - s->h_part_off[asset] != 1)
        return fail(AGR_EUNSUPPORTED, "asset %d is split into %d BLAS parts (create with part_policy = 1 to "
                    "export it as one LBVH)", asset, s->h_part_off[asset + 1] - s->h_part_off[asset]);
    DeviceGuard guard(s->device);
    agr_status rs = refresh_parts(s);
    if (rs != AGR_OK) return rs;
    const BlasInfo& a = s->h_parts[s->h_part_off[asset]];
    int64_t nn = a.n_leaves > 1 ? a.n_leaves - 1 : 1;
    *n_nodes = nn;
    *n_leaves = a.n_leaves;
    if (!nodes && !leaf_face && !morton) return AGR_OK;
    if (nodes && s->h_bin_stale[asset])
        return fail(AGR_ESTATE, "binary LBVH nodes are exported for create-time builds only (mesh updated)");
    CK(cudaDeviceSynchronize());
    if (nodes) {
        std::vector<float4> h(4 * nn);
        CK(cudaMemcpy(h.data(), s->bnodes + 4 * (size_t)a.node_base, sizeof(float4) * 4 * nn,
                      cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < nn; ++i) {
            memcpy(nodes + 16 * i, &h[4 * i], 64);
            // make child refs asset-relative
            int* ref = (int*)(nodes + 16 * i + 12);
            for (int c = 0; c < 2; ++c) {
                if (ref[c] == REF_EMPTY) continue;
                ref[c] = ref[c] >= 0 ? ref[c] - a.node_base : ~(~ref[c] - a.leaf_base);
            }
        }
    }
    if (leaf_face && a.n_leaves > 0) {
        std::vector<float4> h(3 * (size_t)a.n_leaves);
        CK(cudaMemcpy(h.data(), s->tris + 3 * (size_t)a.leaf_base, sizeof(float4) * 3 * a.n_leaves,
                      cudaMemcpyDeviceToHost));
        for (int i = 0; i < a.n_leaves; ++i) {
            float w = h[3 * i + 2].w;
            memcpy(&leaf_face[i], &w, 4);
        }
    }
    if (morton && a.n_leaves > 0)
        CK(cudaMemcpy(morton, s->morton + a.leaf_base, sizeof(uint32_t) * a.n_leaves, cudaMemcpyDeviceToHost));
    return AGR_OK;
}

agr_status agr_debug_export_bvh4(agr_scene s, int32_t which, float* nodes, int32_t* root,
                                 int64_t* n_nodes) {
    g_err.clear();
    if (!s || !n_nodes) return fail(AGR_EINVAL, "bad argument");
    int64_t base, count;
    if (which >= 0) {
        if (which >= s->n_assets) return fail(AGR_EINVAL, "asset out of range");
        if (s->h_part_off[which + 1] - s->h_part_off[which] != 1)
            return fail(AGR_EUNSUPPORTED, "asset %d is split into BLAS parts (part_policy = 1 exports it whole)",
                        which);
        {
            DeviceGuard g2(s->device);
            agr_status rs = refresh_parts(s);
            if (rs != AGR_OK) return rs;
        }
        const BlasInfo& a = s->h_parts[s->h_part_off[which]];
        base = a.node_base;
        count = a.n_nodes4;  // the compacted BVH4 (every node reachable from the root)
    } else {
        const int e = -1 - which;
        if (e >= s->n_envs) return fail(AGR_EINVAL, "env out of range");
        if (!s->built) return fail(AGR_ESTATE, "TLAS not built");
        int n = s->h_item_off[e + 1] - s->h_item_off[e];
        base = (int64_t)s->nb_blas + s->h_tlas_off[e];
        count = n > 1 ? n - 1 : 1;
    }
    *n_nodes = count;
    if (root) *root = (int32_t)base;
    if (!nodes) return AGR_OK;
    DeviceGuard guard(s->device);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(nodes, s->nodes + 8 * (size_t)base, sizeof(float4) * 8 * count, cudaMemcpyDeviceToHost));
    return AGR_OK;
}

agr_status agr_debug_asset_parts(agr_scene s, int32_t asset, int32_t* part_of_face, int32_t* n_parts) {
    g_err.clear();
    if (!s || !n_parts) return fail(AGR_EINVAL, "bad argument");
    if (asset < 0 || asset >= s->n_assets) return fail(AGR_EINVAL, "asset out of range");
    const int p0 = s->h_part_off[asset], p1 = s->h_part_off[asset + 1];
    *n_parts = p1 - p0;
    if (!part_of_face) return AGR_OK;
    if (p1 - p0 == 1) {
        for (int f = 0; f < s->h_nfaces[asset]; ++f) part_of_face[f] = 0;
        return AGR_OK;
    }
    DeviceGuard guard(s->device);
    for (int p = p0; p < p1; ++p) {
        std::vector<int> ids(s->h_part_nfaces[p]);
        CK(cudaMemcpy(ids.data(), s->part_face_ids + s->h_part_foff[p], sizeof(int) * ids.size(),
                      cudaMemcpyDeviceToHost));
        for (int f : ids) part_of_face[f] = p - p0;
    }
    return AGR_OK;
}

}  // extern "C"
