// cast.cu -- the hot path: fused ray generation + two-level BVH traversal +
// FP64 arbitration/epilogue + coalesced stores (SURVEY.md §8(a) a4-a6,
// kernels K9 pinhole, K10 beams, K9b explicit rays).
//
// PAPER.md:228 (§III.D.1): "individual rays are cast outwards per-pixel to
// evaluate intersection with M_{i,t}.  The distance between the sensor and
// the point-of-intersection is reported as range for ToF sensors and
// LiDARs, while the distance of this point from the image plane is reported
// as depth"; PAPER.md:218 (Fig. 3): depth, segmentation, face-index images;
// PAPER.md:215 / :228: LiDAR and custom projection models.
//
// Numerics: traversal and Moller-Trumbore tests run in FP32
// in object space, with every decision FP32 cannot certify deferred: boxes
// are widened by the ray's error bound delta, and a triangle test is
//   * rejected only if FP32 proves a miss (outside by more than the error
//     band, or t provably beyond the current bound U),
//   * "certain" if FP32 proves a hit (inside by more than the band and t
//     provably in (0, max_range]) -- only these tighten U,
//   * otherwise kept as a candidate.
// Candidates with t_lo <= U live in a 4-slot per-lane list; at the end each
// surviving candidate is re-tested in FP64 on the world-space triangle
// (A v + b from the FP32 inputs) with the FP64 ray, and the smallest
// (t, face) wins.  A lane whose list overflows re-traverses in exact mode
// (every leaf tested in FP64).  The reported distance is the FP64 t rounded
// to FP32.
#include "agr_internal.cuh"

namespace agr {
namespace {

#ifndef CAST_BLOCK
#define CAST_BLOCK 64
#endif
#ifndef AGR_IPACKET
#define AGR_IPACKET 1  // interval packets for primary pinhole / beam tiles
#endif
constexpr int CAST_THREADS = CAST_BLOCK;
// Tile of one warp: W x H pixels (beams: columns x channels).  Pinholes
// use 4 x 8 (8 x 4: c3 -3.6 %), LiDAR beam tables 8 x 4 (c4 +1.9 % over
// 4 x 8: an 8-column x 4-channel tile spans 5.6 x 2.8 deg of an OS0-128).
#ifndef TILE_W_PINHOLE
#define TILE_W_PINHOLE 4
#endif
#ifndef TILE_W_BEAMS
#define TILE_W_BEAMS 8
#endif
template <int MODEL>
struct Tile {
    static constexpr int W = MODEL == 2 ? TILE_W_BEAMS : TILE_W_PINHOLE;
    static constexpr int H = 32 / W;
    static constexpr int CL = (H / 2 - 1) * W + W / 2 - 1;  // the lane of the tile's centre ray
};
// 32 resident warps per SM: 64 registers per thread
#ifndef CAST_MIN_BLOCKS
#define CAST_MIN_BLOCKS (1024 / CAST_BLOCK)
#endif
// Pinhole interval packets (with pop-time culling, a second warp stack in
// shared memory) run best at 14 blocks of 64 (72 registers, more L1): c3
// +0.7 %, c5 +1.7 % over 16; LiDAR packets (-0.8 %) and per-lane casts
// (-4.8 %) keep 16.
#ifndef CAST_MIN_BLOCKS_PINHOLE
#define CAST_MIN_BLOCKS_PINHOLE 14
#endif
constexpr int cast_min_blocks(int model, int trav) {
    return model == 1 && trav == 1 ? CAST_MIN_BLOCKS_PINHOLE : CAST_MIN_BLOCKS;
}
constexpr int NSLOT = 4;
constexpr int SENTINEL = REF_EMPTY;  // "return to the TLAS" marker on the stack

__device__ __forceinline__ float inf_f() { return __int_as_float(0x7f800000); }

// Ray state for box tests at one level (env or object space).
struct SlabRay {
    float idx, idy, idz;      // 1 / d (zero components clamped)
    float lox, loy, loz;      // -(o + delta) * id
    float hix, hiy, hiz;      // -(o - delta) * id
};

// Approximate reciprocal (MUFU.RCP, ~1 ulp): every FP32 quantity it feeds is
// covered by the error budget of DESIGN.md §5.2, so no IEEE division.
// Flush-to-zero (one MUFU.RCP, no denormal fix-up): exact for inputs with
// 1e-30 <= |x| < 8.5e37, where neither the input nor the result is
// denormal -- safe_inv's inputs (ray direction components, offset by
// copysign(1e-30)) are in that range for any ray with finite, sub-1e37
// object-space direction.
__device__ __forceinline__ float rcp_approx_ftz(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// |x|^-1/2 without the denormal fix-up; a denormal x gives inf, and the
// NaN / inf that follow only widen the FP32 filter's bands.
__device__ __forceinline__ float rsqrt_approx_ftz(float x) {
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ float safe_inv(float d) {
    // d + copysign(1e-30, d) == d unless |d| < ~1e-22: never a zero divisor
    return rcp_approx_ftz(d + copysignf(1e-30f, d));
}

__device__ __forceinline__ SlabRay make_slab(f3 o, f3 d, float delta) {
    SlabRay s;
    s.idx = safe_inv(d.x);
    s.idy = safe_inv(d.y);
    s.idz = safe_inv(d.z);
    s.lox = -(o.x + delta) * s.idx;
    s.loy = -(o.y + delta) * s.idy;
    s.loz = -(o.z + delta) * s.idz;
    s.hix = -(o.x - delta) * s.idx;
    s.hiy = -(o.y - delta) * s.idy;
    s.hiz = -(o.z - delta) * s.idz;
    return s;
}

// Slab test of one child box (lo/hi per axis) against [0, U].
__device__ __forceinline__ bool slab(const SlabRay& r, float lx, float hx, float ly, float hy,
                                     float lz, float hz, float U, float& tnear) {
    float ax = fmaf(lx, r.idx, r.lox), bx = fmaf(hx, r.idx, r.hix);
    float ay = fmaf(ly, r.idy, r.loy), by = fmaf(hy, r.idy, r.hiy);
    float az = fmaf(lz, r.idz, r.loz), bz = fmaf(hz, r.idz, r.hiz);
    float tn = fmaxf(fmaxf(fminf(ax, bx), fminf(ay, by)), fmaxf(fminf(az, bz), 0.0f));
    float tf = fminf(fminf(fmaxf(ax, bx), fmaxf(ay, by)), fminf(fmaxf(az, bz), U));
    tnear = tn;
    return tn <= tf;
}

// ---- FP64 ray and FP64 world-space triangle test ----------------------------
struct Ray64 { d3 o, d; };

// FP64 Moller-Trumbore on the world-space triangle A v + b (closed,
// double-sided); returns the ray parameter t of the plane hit.
__device__ __forceinline__ bool tri64(const SceneView& sv, int inst, int leaf, const Ray64& r, double& t) {
    const float* T = sv.inst_T + 12 * inst;
    const float4* v = reinterpret_cast<const float4*>(sv.triv) + 3 * (size_t)leaf;
    double A[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) A[k] = (double)__ldg(T + k);
    d3 w[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const float4 q = __ldg(v + c);
        double x = q.x, y = q.y, z = q.z;
        w[c].x = A[0] * x + A[1] * y + A[2] * z + A[3];
        w[c].y = A[4] * x + A[5] * y + A[6] * z + A[7];
        w[c].z = A[8] * x + A[9] * y + A[10] * z + A[11];
    }
    d3 e1 = subd(w[1], w[0]), e2 = subd(w[2], w[0]);
    d3 p = crossd(r.d, e2);
    double det = dotd(e1, p);
    if (det == 0.0) return false;
    d3 s = subd(r.o, w[0]);
    double u = dotd(s, p);
    d3 q = crossd(s, e1);
    double vv = dotd(r.d, q);
    double tn = dotd(e2, q);
    if (det < 0.0) { det = -det; u = -u; vv = -vv; tn = -tn; }
    if (u < 0.0 || vv < 0.0 || u + vv > det) return false;
    t = tn / det;
    return true;
}

__device__ __forceinline__ bool test64(const SceneView& sv, int inst, int leaf, const Ray64& r,
                                       double tmax, double& t) {
    return tri64(sv, inst, leaf, r, t) && t > 0.0 && t <= tmax;
}

// ---- per-lane candidate list and resolved best ---------------------------------
struct Slots {
    float tl[NSLOT];
    int inst[NSLOT];
    int leaf[NSLOT];
};

struct Counters { unsigned nodes, leaves, insts, f64, overflow, tnodes, empty; };

struct Best64 {
    double t;
    int face;   // per-env face index, -1 none
    int inst;
    int leaf;
};

__device__ __forceinline__ bool better(double t, int face, const Best64& b) {
    return b.face < 0 || t < b.t || (t == b.t && face < b.face);
}

__device__ __forceinline__ void consider64(const SceneView& sv, int inst, int leaf, const Ray64& r64,
                                           double tmax, Best64& best) {
    double t;
    if (test64(sv, inst, leaf, r64, tmax, t)) {
        int face = __ldg(sv.inst_face_off + inst) + __float_as_int(__ldg(&sv.tris[3 * leaf + 2].w));
        if (better(t, face, best)) { best.t = t; best.face = face; best.inst = inst; best.leaf = leaf; }
    }
}

// Brute force over every triangle of the env in FP64: the path of last resort
// when a traversal stack would overflow (a pathological TLAS/BLAS depth).
__device__ __noinline__ void brute64(SceneView sv, int env, Ray64 r64, double tmax, Best64* best) {
    Best64 b = *best;
    for (int inst = __ldg(sv.env_off + env); inst < __ldg(sv.env_off + env + 1); ++inst) {
        const int a = __ldg(sv.inst_asset + inst);
        for (int p = __ldg(sv.part_off + a); p < __ldg(sv.part_off + a + 1); ++p) {
            const BlasInfo& bl = sv.parts[p];
            for (int l = 0; l < bl.n_leaves; ++l) consider64(sv, inst, bl.leaf_base + l, r64, tmax, b);
        }
    }
    *best = b;
}

// ---- per-ray traversal state (shared by the per-lane and the packet drivers) -----
// Hot state (used at every node) lives in registers; cold state (the object-
// space ray for triangle tests, the candidate list and the FP64-resolved
// best) lives in a per-lane column of shared memory so the node loop stays
// within 64 registers without spills.
enum ColdField {
    C_OX, C_OY, C_OZ, C_DX, C_DY, C_DZ, C_Q,
    C_OOX, C_OOY, C_OOZ, C_ODX, C_ODY, C_ODZ, C_DELTA, C_DLEN,
    C_TL0, C_INST0 = C_TL0 + NSLOT, C_LEAF0 = C_INST0 + NSLOT,
    C_FACE = C_LEAF0 + NSLOT, C_BINST, C_BLEAF,
    C_OVF,  // traversal stack overflowed (-> FP64 brute force); kept out of registers
    C_COL, C_ROW, C_IMG,  // pixel / beam and env * S + sensor: the FP64 ray's inputs
    N_COLD
};

// Per-lane cold columns of the block (file scope so the out-of-line FP64
// testers can read the lane's ray identity without an extra argument).
__shared__ float s_cold[N_COLD][CAST_THREADS];
__shared__ double s_best_t[CAST_THREADS];

struct Cold {
    float* p;     // &s_cold[0][lane of block]
    double* bt;   // &s_best_t[lane of block]
    __device__ __forceinline__ float& f(int k) const { return p[k * CAST_THREADS]; }
    __device__ __forceinline__ int& i(int k) const { return *reinterpret_cast<int*>(&p[k * CAST_THREADS]); }

    __device__ __forceinline__ Best64 best() const {
        Best64 b;
        b.t = *bt;
        b.face = i(C_FACE);
        b.inst = i(C_BINST);
        b.leaf = i(C_BLEAF);
        return b;
    }
    __device__ __forceinline__ void set_best(const Best64& b) const {
        *bt = b.t;
        i(C_FACE) = b.face;
        i(C_BINST) = b.inst;
        i(C_BLEAF) = b.leaf;
    }
};

struct RayState {
    float tmin;       // any-hit (shadow) queries: hits must have t in (tmin, tmax)
    float tmax;
    float U;          // upper bound on the winning t (certain FP32 hits, FP64 hits)
    SlabRay sr;       // box-test state of the current level
    int cur_inst;     // -1 at the TLAS level
    Cold c;           // env-level ray o, d, q; object-space ray; candidates; best

    __device__ __forceinline__ f3 o() const { return mk(c.f(C_OX), c.f(C_OY), c.f(C_OZ)); }
    __device__ __forceinline__ f3 d() const { return mk(c.f(C_DX), c.f(C_DY), c.f(C_DZ)); }

    __device__ __forceinline__ void init(f3 o, f3 d, float tmax_, Cold cold) {
        c = cold;
        tmin = 0.0f;
        tmax = tmax_;
        U = tmax_;
        // |o|_1 + tmax |d|_1: scale of the FP32 ray's position error
        const float q = fabsf(o.x) + fabsf(o.y) + fabsf(o.z) + tmax * (fabsf(d.x) + fabsf(d.y) + fabsf(d.z));
        c.f(C_OX) = o.x; c.f(C_OY) = o.y; c.f(C_OZ) = o.z;
        c.f(C_DX) = d.x; c.f(C_DY) = d.y; c.f(C_DZ) = d.z;
        c.f(C_Q) = q;
        // env level: the origin is an exact input, the direction carries rounding
        sr = make_slab(o, d, K_ERR * q);
        cur_inst = -1;
#pragma unroll
        for (int k = 0; k < NSLOT; ++k) { c.f(C_TL0 + k) = inf_f(); c.i(C_INST0 + k) = -1; c.i(C_LEAF0 + k) = -1; }
        c.i(C_OVF) = 0;
        Best64 b;
        b.t = 0.0;
        b.face = -1;
        b.inst = -1;
        b.leaf = -1;
        c.set_best(b);
    }

    __device__ __forceinline__ void exit_instance() {
        sr = make_slab(this->o(), this->d(), K_ERR * c.f(C_Q));  // env-level box-test state
        cur_inst = -1;
    }

    // TLAS leaf: move the ray into the object space of item `item` (an
    // instance's part); returns the part's BLAS root node.
    __device__ __forceinline__ int enter_instance(const SceneView& sv, int item) {
        f3 oo, od;
        float delta;
        const int root = enter_object(sv, item, oo, od, delta);
        sr = make_slab(oo, od, delta);
        return root;
    }

    // enter_instance without the per-lane box-test state (interval packets
    // build their own): object-space ray, its error bound, cold columns.
    __device__ __forceinline__ int enter_object(const SceneView& sv, int item, f3& oo_, f3& od_, float& delta_) {
        const float4* rp = sv.irec + 4 * item;
        float4 r0 = __ldg(rp), r1 = __ldg(rp + 1), r2 = __ldg(rp + 2), r3 = __ldg(rp + 3);
        const f3 o = this->o(), d = this->d();
        const float q = c.f(C_Q);
        f3 oo = mk(fmaf(r0.x, o.x, fmaf(r0.y, o.y, fmaf(r0.z, o.z, r0.w))),
                   fmaf(r1.x, o.x, fmaf(r1.y, o.y, fmaf(r1.z, o.z, r1.w))),
                   fmaf(r2.x, o.x, fmaf(r2.y, o.y, fmaf(r2.z, o.z, r2.w))));
        f3 od = mk(fmaf(r0.x, d.x, fmaf(r0.y, d.y, r0.z * d.z)),
                   fmaf(r1.x, d.x, fmaf(r1.y, d.y, r1.z * d.z)),
                   fmaf(r2.x, d.x, fmaf(r2.y, d.y, r2.z * d.z)));
        // object-space position error bound
        float delta = K_ERR * fmaf(r3.y, q, r3.z);
        c.f(C_OOX) = oo.x; c.f(C_OOY) = oo.y; c.f(C_OOZ) = oo.z;
        c.f(C_ODX) = od.x; c.f(C_ODY) = od.y; c.f(C_ODZ) = od.z;
        c.f(C_DELTA) = delta;
        const float dd = dot(od, od);
        c.f(C_DLEN) = dd > 0.0f ? dd * rsqrt_approx_ftz(dd) * 1.000001f : 0.0f;
        cur_inst = __float_as_int(r3.w);  // the item's instance (FP64 tests, face offset, label)
        oo_ = oo;
        od_ = od;
        delta_ = delta;
        return __float_as_int(r3.x);
    }

    // The box-test state is parked in shared memory while a triangle is
    // tested and reloaded afterwards, so it holds no registers there.
    // The box-test state is not kept live across a triangle test (register
    // pressure): it is rebuilt from the object-space ray in shared memory.
    __device__ __forceinline__ void load_slab() {
        sr = make_slab(mk(c.f(C_OOX), c.f(C_OOY), c.f(C_OOZ)), mk(c.f(C_ODX), c.f(C_ODY), c.f(C_ODZ)),
                       c.f(C_DELTA));
    }

    __device__ __forceinline__ void node4_test(const float4* f, float tn[4], bool h[4]) const {
        h[0] = slab(sr, f[0].x, f[1].x, f[2].x, f[3].x, f[4].x, f[5].x, U, tn[0]);
        h[1] = slab(sr, f[0].y, f[1].y, f[2].y, f[3].y, f[4].y, f[5].y, U, tn[1]);
        h[2] = slab(sr, f[0].z, f[1].z, f[2].z, f[3].z, f[4].z, f[5].z, U, tn[2]);
        h[3] = slab(sr, f[0].w, f[1].w, f[2].w, f[3].w, f[4].w, f[5].w, U, tn[3]);
    }

    // Resolve leaf `leaf` of the current instance in FP64 now (exact mode,
    // full candidate list); `res` is the out-of-line FP64 tester.
    template <class RES>
    __device__ __forceinline__ void resolve64(int leaf, const RES& res) {
        Best64 b = c.best();
        res(cur_inst, leaf, b);
        c.set_best(b);
        if (b.face >= 0) U = fminf(U, __double2float_ru(b.t));
    }

    // FP32 filter test of BLAS leaf `leaf`: reject what FP32
    // proves a miss, tighten U with what it proves a hit, keep the rest as
    // candidates for FP64 arbitration.  A full list resolves in FP64 inline.
    template <bool COUNT, class RES>
    __device__ __forceinline__ void leaf_filter(const SceneView& sv, int leaf, const RES& res,
                                                Counters& cnt) {
        const float4* tp = sv.tris + 3 * leaf;
        float4 a = __ldg(tp), b = __ldg(tp + 1), cc = __ldg(tp + 2);
        const f3 oo = mk(c.f(C_OOX), c.f(C_OOY), c.f(C_OOZ));
        const f3 od = mk(c.f(C_ODX), c.f(C_ODY), c.f(C_ODZ));
        const float delta = c.f(C_DELTA);
        f3 v0 = mk(a.x, a.y, a.z), e1 = mk(b.x, b.y, b.z), e2 = mk(cc.x, cc.y, cc.z);
        f3 p = cross(od, e2);
        float det = dot(e1, p);
        f3 s = sub(oo, v0);
        bool keep, certain = false;
        float tl = 0.0f, th = 0.0f;
        if (det != 0.0f) {
            float inv = rcp_approx_ftz(det);  // denormal det -> inf: kept as a candidate (NaN-safe tests below)
            f3 qv = cross(s, e1);
            float u = dot(s, p) * inv;
            float v = dot(od, qv) * inv;
            float t = dot(e2, qv) * inv;
            float g = delta * b.w * fabsf(inv);          // t error bound
            float beta = g * c.f(C_DLEN) * a.w;          // barycentric band
            float terr = fmaf(fabsf(t), T_REL, g);
            tl = t - terr;
            th = t + terr;
            bool out = u < -beta || v < -beta || u + v > 1.0f + beta || th < 0.0f || tl > U;
            keep = !out;
            if (!(tl == tl)) tl = 0.0f;  // NaN (denormal det): keep conservatively
            certain = keep && u > beta && v > beta && u + v < 1.0f - beta && tl > 0.0f && th <= tmax;
        } else {
            // parallel in FP32: keep only if the origin is within delta of the plane
            f3 nn = cross(e1, e2);
            keep = fabsf(dot(s, nn)) <= delta * b.w;
        }
        if (keep) {
            if (certain && th < U) U = th;
            int slot = -1;
#pragma unroll
            for (int k = NSLOT - 1; k >= 0; --k)  // lowest free slot: empty or pruned by U
                if (!(c.f(C_TL0 + k) <= U)) slot = k;
            if (slot >= 0) {
                c.f(C_TL0 + slot) = tl;
                c.i(C_INST0 + slot) = cur_inst;
                c.i(C_LEAF0 + slot) = leaf;
            } else {
                if (COUNT) cnt.overflow++;
                if (COUNT) cnt.f64++;
                resolve64(leaf, res);
            }
        }
    }

    // Any-hit FP32 filter for shadow segments (f2 stereo mask): a hit needs t
    // in (tmin, tmax).  A certain hit ends the query (U = -1 culls every
    // box); an uncertain one is decided by the out-of-line FP64 test `res`.
    template <bool COUNT, class RES>
    __device__ __forceinline__ void leaf_anyhit(const SceneView& sv, int leaf, const RES& res, Counters& cnt) {
        if (U < 0.0f) return;
        const float4* tp = sv.tris + 3 * leaf;
        float4 a = __ldg(tp), b = __ldg(tp + 1), cc = __ldg(tp + 2);
        const f3 oo = mk(c.f(C_OOX), c.f(C_OOY), c.f(C_OOZ));
        const f3 od = mk(c.f(C_ODX), c.f(C_ODY), c.f(C_ODZ));
        const float delta = c.f(C_DELTA);
        f3 v0 = mk(a.x, a.y, a.z), e1 = mk(b.x, b.y, b.z), e2 = mk(cc.x, cc.y, cc.z);
        f3 p = cross(od, e2);
        float det = dot(e1, p);
        f3 s = sub(oo, v0);
        bool keep, certain = false;
        if (det != 0.0f) {
            float inv = rcp_approx_ftz(det);  // denormal det -> inf: kept as a candidate (NaN-safe tests below)
            f3 qv = cross(s, e1);
            float u = dot(s, p) * inv;
            float v = dot(od, qv) * inv;
            float t = dot(e2, qv) * inv;
            float g = delta * b.w * fabsf(inv);
            float beta = g * c.f(C_DLEN) * a.w;
            float terr = fmaf(fabsf(t), T_REL, g);
            float tl = t - terr, th = t + terr;
            bool out = u < -beta || v < -beta || u + v > 1.0f + beta || th <= tmin || tl >= tmax;
            keep = !out;
            certain = keep && u > beta && v > beta && u + v < 1.0f - beta && tl > tmin && th < tmax;
        } else {
            f3 nn = cross(e1, e2);
            keep = fabsf(dot(s, nn)) <= delta * b.w;
        }
        if (certain) {
            U = -1.0f;
        } else if (keep) {
            if (COUNT) cnt.f64++;
            if (res(cur_inst, leaf)) U = -1.0f;
        }
    }

    // FP64 arbitration of the surviving candidates (slot loop, warp-uniform).
    template <bool COUNT, class RES>
    __device__ __forceinline__ Best64 arbitrate(const RES& res, Counters& cnt) {
        Best64 b = c.best();
#pragma unroll
        for (int k = 0; k < NSLOT; ++k) {
            if (c.f(C_TL0 + k) <= U) {
                if (COUNT) cnt.f64++;
                res(c.i(C_INST0 + k), c.i(C_LEAF0 + k), b);
            }
        }
        return b;
    }
};

// Load the 6 box float4s and the refs of BVH4 node `node` (broadcast loads
// in packet mode).
__device__ __forceinline__ void load_node4(const SceneView& sv, int node, float4 f[6], int ref[4]) {
    const float4* np = sv.nodes + 8 * (size_t)node;
#pragma unroll
    for (int k = 0; k < 6; ++k) f[k] = __ldg(np + k);
    const float4 r = __ldg(np + 6);
    ref[0] = __float_as_int(r.x);
    ref[1] = __float_as_int(r.y);
    ref[2] = __float_as_int(r.z);
    ref[3] = __float_as_int(r.w);
}

__device__ __forceinline__ void cswap(unsigned& ka, int& ra, unsigned& kb, int& rb) {
    const bool sw = kb < ka;
    const unsigned k = sw ? kb : ka;
    const int r = sw ? rb : ra;
    kb = sw ? ka : kb;
    rb = sw ? ra : rb;
    ka = k;
    ra = r;
}

// Ascending sort of 4 (key, ref) pairs (5 compare-exchanges).
__device__ __forceinline__ void sort4(unsigned k[4], int r[4]) {
    cswap(k[0], r[0], k[1], r[1]);
    cswap(k[2], r[2], k[3], r[3]);
    cswap(k[0], r[0], k[2], r[2]);
    cswap(k[1], r[1], k[3], r[3]);
    cswap(k[1], r[1], k[2], r[2]);
}

// The traversal decodes BLAS leaves of one or two triangles (a loop over
// up to LEAF_MAX records measured 3 % slower on c3 and gained < 0.5 % at
// LEAF_MAX = 3 or 4).
static_assert(LEAF_MAX >= 1 && LEAF_MAX <= 2, "cast.cu decodes single and pair leaves only");

constexpr unsigned KEY_MISS = 0x7f800000u;  // +inf bits: sorts after every hit (t >= 0)

// ---- per-lane traversal (explicit rays; exact-mode fallback) -------------------
// Ordered stackful traversal of the two-level BVH, one independent ray per
// lane (Aila & Laine style, stack in local memory).
// LEAF(leaf) tests BLAS leaf `leaf` of rs.cur_inst; ANYHIT stops a ray once
// its U < 0 (shadow queries).
template <bool ANYHIT, bool COUNT, class LEAF>
__device__ __forceinline__ void traverse_lane(const SceneView& sv, int env, RayState& rs,
                                              const LEAF& leaf_fn, Counters& cnt) {
    int stack[STACK_SIZE];
    int sp = 0;
    int node = __ldg(sv.tlas_root + env);
    bool fresh = false;  // COUNT: the node is the root of a just-entered BLAS
    for (;;) {
        if (node >= 0) {
            if (COUNT) cnt.nodes++;
            if (COUNT && rs.cur_inst < 0) cnt.tnodes++;
            float4 f[6];
            int ref[4];
            load_node4(sv, node, f, ref);
            float tn[4];
            bool h[4];
            rs.node4_test(f, tn, h);
            unsigned key[4];
            int nh = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                key[k] = h[k] ? __float_as_uint(tn[k]) : KEY_MISS;
                nh += h[k] ? 1 : 0;
            }
            if (COUNT && fresh) {
                if (nh == 0) cnt.empty++;
                fresh = false;
            }
            if (nh == 0) {
                if (sp == 0) break;
                node = stack[--sp];
                continue;
            }
            sort4(key, ref);
            // push the farther hit children (farthest first), descend the nearest
#pragma unroll
            for (int k = 3; k >= 1; --k) {
                if (k < nh) {
                    if (sp < STACK_SIZE) stack[sp++] = ref[k];
                    else rs.c.i(C_OVF) = 1;
                }
            }
            node = ref[0];
            continue;
        }
        if (node == SENTINEL) {  // leave the instance: back to the env-level ray
            rs.exit_instance();
            if (sp == 0) break;
            node = stack[--sp];
            continue;
        }
        const int leaf = ~node;
        if (rs.cur_inst < 0) {
            if (COUNT) cnt.insts++;
            if (COUNT) fresh = true;
            if (sp < STACK_SIZE) stack[sp++] = SENTINEL;
            else { rs.c.i(C_OVF) = 1; break; }
            node = rs.enter_instance(sv, leaf);
            continue;
        }
        if (COUNT) cnt.leaves++;
        leaf_fn(leaf & LEAF_MASK);
        if (leaf >> LEAF_SHIFT) {  // pair leaf (LEAF_MAX == 2)
            if (COUNT) cnt.leaves++;
            leaf_fn((leaf & LEAF_MASK) + 1);
        }
        rs.load_slab();
        if (sp == 0 || (ANYHIT && rs.U < 0.0f)) break;
        node = stack[--sp];
    }
}

// ---- packet traversal (pinhole / beams tiles) ------------------------------------
// The 32 rays of a tile (Tile<MODEL>: 4x8 pinhole, 8x4 beams) traverse together: the warp visits a node if any
// lane's ray hits it (ballot), descends first into the child most lanes reach
// first, and keeps ONE stack per warp in shared memory.  Control flow is
// warp-uniform (no divergence in the traversal loop); every node / triangle
// fetch is a broadcast load.  Each lane still does its own exact-filter box
// and triangle tests, so results equal the per-lane traversal.
constexpr int PSTACK = 128;  // >= 4 full levels of 32-wide pushes

template <int CL, bool ANYHIT, bool COUNT, class LEAF>
__device__ __forceinline__ void traverse_packet(const SceneView& sv, int env, RayState& rs,
                                                const LEAF& leaf_fn, int* wstack,
                                                Counters& cnt) {
    const unsigned FULL = 0xFFFFFFFFu;
    const bool leader = (threadIdx.x & 31) == 0;
    int sp = 0;
    int node = __ldg(sv.tlas_root + env);
    bool fresh = false;  // COUNT: the node is the root of a just-entered BLAS
    for (;;) {
        if (node >= 0) {
            if (COUNT) cnt.nodes++;
            if (COUNT && rs.cur_inst < 0) cnt.tnodes++;
            float4 f[6];
            int ref[4];
            load_node4(sv, node, f, ref);
            float tn[4];
            bool h[4];
            rs.node4_test(f, tn, h);
            // 4-bit mask of the children some lane hits
            const unsigned hm = (h[0] ? 1u : 0u) | (h[1] ? 2u : 0u) | (h[2] ? 4u : 0u) | (h[3] ? 8u : 0u);
            if (COUNT && fresh) {
                if (hm == 0) cnt.empty++;  // this lane's own ray
                fresh = false;
            }
            const unsigned cm = __reduce_or_sync(FULL, hm);
            const int nh = __popc(cm);
            if (nh == 0) {
                if (sp == 0) break;
                __syncwarp();
                node = wstack[--sp];
                continue;
            }
            if (nh == 1) {
                const int only = __ffs(cm) - 1;
                node = only == 0 ? ref[0] : only == 1 ? ref[1] : only == 2 ? ref[2] : ref[3];
                continue;
            }
            // order the children by the entry distance of the tile's centre
            // ray (lane CL), misses last
            unsigned key[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const unsigned kc = __shfl_sync(FULL, __float_as_uint(tn[k]), CL);
                key[k] = (cm >> k) & 1u ? kc : KEY_MISS;
            }
            sort4(key, ref);
            // push the farther children, farthest first
            if (sp + 3 <= PSTACK) {
                __syncwarp();  // every lane has read the slots before they are reused
                if (leader) {
                    int q = sp;
                    if (nh > 3) wstack[q++] = ref[3];
                    if (nh > 2) wstack[q++] = ref[2];
                    wstack[q] = ref[1];
                }
                sp += nh - 1;  // nh is warp-uniform
            } else {
                rs.c.i(C_OVF) = 1;
            }
            node = ref[0];
            continue;
        }
        if (node == SENTINEL) {
            rs.exit_instance();
            if (sp == 0) break;
            __syncwarp();
            node = wstack[--sp];
            continue;
        }
        const int leaf = ~node;
        if (rs.cur_inst < 0) {
            if (COUNT) cnt.insts++;
            if (COUNT) fresh = true;
            if (sp < PSTACK) {
                __syncwarp();  // every lane has read the slot before it is reused
                if (leader) wstack[sp] = SENTINEL;
                ++sp;
            } else {
                rs.c.i(C_OVF) = 1;
                break;
            }
            node = rs.enter_instance(sv, leaf);
            continue;
        }
        if (COUNT) cnt.leaves++;
        leaf_fn(leaf & LEAF_MASK);
        if (leaf >> LEAF_SHIFT) {  // pair leaf (LEAF_MAX == 2), warp-uniform
            if (COUNT) cnt.leaves++;
            leaf_fn((leaf & LEAF_MASK) + 1);
        }
        rs.load_slab();
        if (sp == 0 || (ANYHIT && __all_sync(FULL, rs.U < 0.0f))) break;
        __syncwarp();
        node = wstack[--sp];
    }
}

// ---- interval-packet traversal (primary pinhole / beam tiles) ---------------------
// The 32 rays of a tile share their origin (the sensor's), so the set of
// their directions lies in the per-axis interval [dmin, dmax] over the
// lanes.  A node is visited if the *packet* may reach a child: lanes 0-3
// each test one child against the whole interval (conservative: any lane's
// own widened slab test passing implies this one passes),
// lanes 4-7 test the same child with the tile's centre ray for the visiting
// order.  One slab test per lane per node instead of four; leaves are still
// tested by every lane on its own ray.
//
// Box-test state of one lane (its role: interval or centre ray) at one
// level: per axis the widened origin offsets and the reciprocals of the
// two direction endpoints.
struct PSlab {
    float olx, oly, olz;  // o + dp
    float ohx, ohy, ohz;  // o - dp
    float i0x, i0y, i0z;  // 1 / (lower direction endpoint)
    float i1x, i1y, i1z;  // 1 / (upper direction endpoint)
    int strad;            // warp-uniform: some lane's interval contains 0 on some axis
};
constexpr int PS_N = 13;
constexpr int PS_MAXN = 20;  // >= PS_N and the BVH8 FMA form's PS8_N
#ifndef AGR_STRAD_FAST
#define AGR_STRAD_FAST 1  // BVH8 packets: no-straddle slab specialisation
#endif
#ifndef AGR_RANK_MODE
#define AGR_RANK_MODE 1   // BVH8 child order: 0 full rank with ties, 1 REDUX nearest + rank for nh > 2, 2 nearest only
#endif
#ifndef AGR_SLAB_FMA
#define AGR_SLAB_FMA 1    // BVH8 packets: FMA-form interval slab with the entry / exit planes by direction sign
#endif
#ifndef AGR_POP_CULL
#define AGR_POP_CULL 1    // wide pinhole packets: skip popped stack entries whose pushed entry bound exceeds Umax
#endif
#ifndef AGR_PS_RELOAD
#define AGR_PS_RELOAD 1   // reload the packet slab state from shared memory after a leaf
#endif

__device__ __forceinline__ int f2ord(float f) {
    const int k = __float_as_int(f);
    return k ^ ((k >> 31) & 0x7FFFFFFF);
}
__device__ __forceinline__ float ord2f(int k) { return __int_as_float(k ^ ((k >> 31) & 0x7FFFFFFF)); }

// Reciprocal endpoints of a direction interval [lo, hi].  An interval
// containing 0 keeps i0 = 1 / min(lo, -tiny) < 0 < i1 = 1 / max(hi, tiny):
// pslab_axis tells it apart by the differing signs.
__device__ __forceinline__ void iv_recip(float lo, float hi, float& i0, float& i1) {
    if (lo > 0.0f || hi < 0.0f) {
        i0 = rcp_approx_ftz(lo);
        i1 = rcp_approx_ftz(hi);
    } else {
        i0 = rcp_approx_ftz(fminf(lo, -1e-30f));
        i1 = rcp_approx_ftz(fmaxf(hi, 1e-30f));
    }
}

// Packet box-test state from every lane's ray (o shared by all lanes, d its
// own, delta its error bound); lanes with (lane & CENTRE_BIT) take the centre
// ray (BVH4: lanes 4-7, BVH8: lanes 8-15).
template <int CL, int CENTRE_BIT = 4>
__device__ __forceinline__ PSlab make_pslab(f3 o, f3 d, float delta) {
    const unsigned FULL = 0xFFFFFFFFu;
    const bool centre = ((threadIdx.x & 31) & CENTRE_BIT) != 0;  // CENTRE_BIT 32: no centre lanes
    const float dcx = __shfl_sync(FULL, d.x, CL);
    const float dcy = __shfl_sync(FULL, d.y, CL);
    const float dcz = __shfl_sync(FULL, d.z, CL);
    const float mnx = ord2f(__reduce_min_sync(FULL, f2ord(d.x))), mxx = ord2f(__reduce_max_sync(FULL, f2ord(d.x)));
    const float mny = ord2f(__reduce_min_sync(FULL, f2ord(d.y))), mxy = ord2f(__reduce_max_sync(FULL, f2ord(d.y)));
    const float mnz = ord2f(__reduce_min_sync(FULL, f2ord(d.z))), mxz = ord2f(__reduce_max_sync(FULL, f2ord(d.z)));
    // twice the largest lane error bound: the interval arithmetic's own
    // rounding (a few ulps of t) is far inside one delta
    const float dp = 2.0f * __int_as_float(__reduce_max_sync(FULL, __float_as_int(delta)));
    PSlab p;
    p.olx = o.x + dp; p.oly = o.y + dp; p.olz = o.z + dp;
    p.ohx = o.x - dp; p.ohy = o.y - dp; p.ohz = o.z - dp;
    iv_recip(centre ? dcx : mnx, centre ? dcx : mxx, p.i0x, p.i1x);
    iv_recip(centre ? dcy : mny, centre ? dcy : mxy, p.i0y, p.i1y);
    iv_recip(centre ? dcz : mnz, centre ? dcz : mxz, p.i0z, p.i1z);
    // the interval straddles 0 on an axis (same test as iv_recip's); the
    // centre lanes only order children, so only the interval's counts
    const bool st = !(mnx > 0.0f || mxx < 0.0f) || !(mny > 0.0f || mxy < 0.0f) || !(mnz > 0.0f || mxz < 0.0f);
    p.strad = st ? 1 : 0;
    return p;
}

// Slab of one axis over every direction d in the interval (a = lo - o - dp,
// b = hi - o + dp, b >= a):
//   same-sign interval: near = min, far = max of {a, b} x {1/d0, 1/d1};
//   interval containing 0 (i0 < 0 < i1): rays with d of the right sign
//     enter no earlier than max(a / dmax, b / dmin) (o below lo: a / dmax,
//     o above hi: b / dmin, o inside: negative) and, as d -> 0, never
//     leave: far = +inf.
__device__ __forceinline__ void pslab_axis(float lo, float hi, float ol, float oh, float i0, float i1,
                                           float& n, float& f) {
    const float a = lo - ol, b = hi - oh;
    const float a0 = a * i0, a1 = a * i1, b0 = b * i0, b1 = b * i1;
    const bool straddle = (__float_as_int(i0) ^ __float_as_int(i1)) < 0;
    n = straddle ? fmaxf(a1, b0) : fminf(fminf(a0, a1), fminf(b0, b1));
    f = straddle ? inf_f() : fmaxf(fmaxf(a0, a1), fmaxf(b0, b1));
}

// Interval slab test of child c of the node at nb against [0, U].
__device__ __forceinline__ bool pslab_test(const PSlab& p, const float* nb, int c, float U, float& tnear) {
    float nx, fx, ny, fy, nz, fz;
    pslab_axis(__ldg(nb + c), __ldg(nb + 4 + c), p.olx, p.ohx, p.i0x, p.i1x, nx, fx);
    pslab_axis(__ldg(nb + 8 + c), __ldg(nb + 12 + c), p.oly, p.ohy, p.i0y, p.i1y, ny, fy);
    pslab_axis(__ldg(nb + 16 + c), __ldg(nb + 20 + c), p.olz, p.ohz, p.i0z, p.i1z, nz, fz);
    const float tn = fmaxf(fmaxf(nx, ny), fmaxf(nz, 0.0f));
    const float tf = fminf(fminf(fx, fy), fminf(fz, U));
    tnear = tn;
    return tn <= tf;
}

__device__ __forceinline__ void pslab_store(float* dst, const PSlab& p) {
    dst[0] = p.olx; dst[1] = p.oly; dst[2] = p.olz;
    dst[3] = p.ohx; dst[4] = p.ohy; dst[5] = p.ohz;
    dst[6] = p.i0x; dst[7] = p.i0y; dst[8] = p.i0z;
    dst[9] = p.i1x; dst[10] = p.i1y; dst[11] = p.i1z;
    dst[12] = __int_as_float(p.strad);
}
__device__ __forceinline__ PSlab pslab_load(const float* src) {
    PSlab p;
    p.olx = src[0]; p.oly = src[1]; p.olz = src[2];
    p.ohx = src[3]; p.ohy = src[4]; p.ohz = src[5];
    p.i0x = src[6]; p.i0y = src[7]; p.i0z = src[8];
    p.i1x = src[9]; p.i1y = src[10]; p.i1z = src[11];
    p.strad = __float_as_int(src[12]);
    return p;
}

#if !AGR_SLAB_FMA
// pslab_axis for an interval of one sign (every lane's, i.e. !strad): near
// and far are the min and max of the four products (no straddle branch).
__device__ __forceinline__ void pslab_axis_fast(float lo, float hi, float ol, float oh, float i0, float i1,
                                                float& n, float& f) {
    const float a = lo - ol, b = hi - oh;
    const float a0 = a * i0, a1 = a * i1, b0 = b * i0, b1 = b * i1;
    n = fminf(fminf(a0, a1), fminf(b0, b1));
    f = fmaxf(fmaxf(a0, a1), fmaxf(b0, b1));
}
#endif

#if AGR_SLAB_FMA
// BVH8 packet box-test state in FMA form: per axis the two reciprocal
// endpoints and, for the entry plane E (lo if the directions are positive,
// hi if negative) and the exit plane X, the products -o_E i and -o_X i, so
// each of the four candidate distances is one FMA of the node's plane:
//   entry = min(E i0 + cE0, E i1 + cE1), exit = max(X i0 + cX0, X i1 + cX1)
// (the min / max over the interval of a monotone 1/d, i.e. the same values
// as pslab_axis's min / max of all four products, rounded once instead of
// twice: the difference is ~2^-24 |o| in position, inside the 2 delta
// widening, which is >= 2^-16 |o|).  An axis whose interval contains 0
// keeps E = lo, X = hi: entry = max(lo i1 + cE1, hi i0 + cX0), exit = inf.
struct __align__(16) PSlab8 {
    float i0x, i0y, i0z, i1x, i1y, i1z;
    float ex0, ex1, xx0, xx1;  // x: cE0, cE1, cX0, cX1
    float ey0, ey1, xy0, xy1;
    float ez0, ez1, xz0, xz1;
    int neg;    // bit k: axis k's directions are negative (E = hi)
    int strad;  // warp-uniform: some lane's interval contains 0 on some axis
};
constexpr int PS8_N = 20;

__device__ __forceinline__ void ps8_axis(float o, float dp, float lo, float hi, float& i0, float& i1, float& e0,
                                         float& e1, float& x0, float& x1, int& neg, int bit) {
    iv_recip(lo, hi, i0, i1);
    const bool straddle = (__float_as_int(i0) ^ __float_as_int(i1)) < 0;
    const bool n = !straddle && i0 < 0.0f;
    const float oe = n ? o - dp : o + dp, ox = n ? o + dp : o - dp;
    e0 = -oe * i0; e1 = -oe * i1; x0 = -ox * i0; x1 = -ox * i1;
    neg |= n ? bit : 0;
}

template <int CL, int CENTRE_BIT = 8>
__device__ __forceinline__ PSlab8 make_pslab8(f3 o, f3 d, float delta) {
    const unsigned FULL = 0xFFFFFFFFu;
    const bool centre = ((threadIdx.x & 31) & CENTRE_BIT) != 0;  // CENTRE_BIT 32: no centre lanes
    const float dcx = __shfl_sync(FULL, d.x, CL);
    const float dcy = __shfl_sync(FULL, d.y, CL);
    const float dcz = __shfl_sync(FULL, d.z, CL);
    const float mnx = ord2f(__reduce_min_sync(FULL, f2ord(d.x))), mxx = ord2f(__reduce_max_sync(FULL, f2ord(d.x)));
    const float mny = ord2f(__reduce_min_sync(FULL, f2ord(d.y))), mxy = ord2f(__reduce_max_sync(FULL, f2ord(d.y)));
    const float mnz = ord2f(__reduce_min_sync(FULL, f2ord(d.z))), mxz = ord2f(__reduce_max_sync(FULL, f2ord(d.z)));
    const float dp = 2.0f * __int_as_float(__reduce_max_sync(FULL, __float_as_int(delta)));
    PSlab8 p;
    p.neg = 0;
    ps8_axis(o.x, dp, centre ? dcx : mnx, centre ? dcx : mxx, p.i0x, p.i1x, p.ex0, p.ex1, p.xx0, p.xx1, p.neg, 1);
    ps8_axis(o.y, dp, centre ? dcy : mny, centre ? dcy : mxy, p.i0y, p.i1y, p.ey0, p.ey1, p.xy0, p.xy1, p.neg, 2);
    ps8_axis(o.z, dp, centre ? dcz : mnz, centre ? dcz : mxz, p.i0z, p.i1z, p.ez0, p.ez1, p.xz0, p.xz1, p.neg, 4);
    const bool st = !(mnx > 0.0f || mxx < 0.0f) || !(mny > 0.0f || mxy < 0.0f) || !(mnz > 0.0f || mxz < 0.0f);
    p.strad = __any_sync(FULL, st && !centre) ? 1 : 0;
    return p;
}

// The state is 5 float4s in a 16-B aligned shared-memory slot: stored and
// reloaded (at instance exits and after every leaf) with 128-bit accesses.
static_assert(PS8_N == 20 && sizeof(PSlab8) == 80, "PSlab8 is 5 float4s");
__device__ __forceinline__ void ps8_store(float* dst, const PSlab8& p) {
    const float4* q = reinterpret_cast<const float4*>(&p);
    float4* d = reinterpret_cast<float4*>(dst);
#pragma unroll
    for (int k = 0; k < 5; ++k) d[k] = q[k];
}
__device__ __forceinline__ PSlab8 ps8_load(const float* src) {
    PSlab8 p;
    const float4* q = reinterpret_cast<const float4*>(src);
    float4* d = reinterpret_cast<float4*>(&p);
#pragma unroll
    for (int k = 0; k < 5; ++k) d[k] = q[k];
    return p;
}

// One axis, intervals of one sign (the warp-uniform fast path).
__device__ __forceinline__ void ps8_axis_fast(float lo, float hi, bool neg, float i0, float i1, float e0, float e1,
                                              float x0, float x1, float& n, float& f) {
    const float E = neg ? hi : lo, X = neg ? lo : hi;
    n = fminf(fmaf(E, i0, e0), fmaf(E, i1, e1));
    f = fmaxf(fmaf(X, i0, x0), fmaf(X, i1, x1));
}
// One axis, any interval (some lane straddles somewhere).
__device__ __forceinline__ void ps8_axis_any(float lo, float hi, bool neg, float i0, float i1, float e0, float e1,
                                             float x0, float x1, float& n, float& f) {
    if ((__float_as_int(i0) ^ __float_as_int(i1)) < 0) {
        n = fmaxf(fmaf(lo, i1, e1), fmaf(hi, i0, x0));
        f = inf_f();
    } else {
        ps8_axis_fast(lo, hi, neg, i0, i1, e0, e1, x0, x1, n, f);
    }
}
#endif

// Closest-hit traversal of a tile whose rays share their origin.  ps_env /
// ps_obj: this warp's shared-memory copies of the two roles' box-test state
// at the env / current object level ([2][PS_N] each).
template <int CL, bool COUNT, class LEAF>
__device__ __forceinline__ void traverse_ipacket(const SceneView& sv, int env, RayState& rs,
                                                 const LEAF& leaf_fn, int* wstack, float* ps_env,
                                                 float* ps_obj, Counters& cnt) {
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31;
    const bool leader = lane == 0;
    const int child = lane & 3;
    const int role = (lane >> 2) & 1;
    PSlab ps = make_pslab<CL>(rs.o(), rs.d(), K_ERR * rs.c.f(C_Q));
    if (child == 0 && lane < 8) pslab_store(ps_env + role * PS_N, ps);
    __syncwarp();
    float Umax = __int_as_float(__reduce_max_sync(FULL, __float_as_int(rs.U)));
    int sp = 0;
    int node = __ldg(sv.tlas_root + env);
    for (;;) {
        if (node >= 0) {
            if (COUNT) cnt.nodes++;
            if (COUNT && rs.cur_inst < 0) cnt.tnodes++;
            const float* nb = reinterpret_cast<const float*>(sv.nodes + 8 * (size_t)node);
            const float4 r4 = __ldg(sv.nodes + 8 * (size_t)node + 6);
            float tn;
            const bool h = pslab_test(ps, nb, child, Umax, tn);
            const unsigned cm = __ballot_sync(FULL, h) & 0xFu;
            const int nh = __popc(cm);
            int ref[4] = {__float_as_int(r4.x), __float_as_int(r4.y), __float_as_int(r4.z), __float_as_int(r4.w)};
            if (nh == 0) {
                if (sp == 0) break;
                __syncwarp();
                node = wstack[--sp];
                continue;
            }
            if (nh == 1) {
                const int only = __ffs(cm) - 1;
                node = only == 0 ? ref[0] : only == 1 ? ref[1] : only == 2 ? ref[2] : ref[3];
                continue;
            }
            // order by the centre ray's entry distance (lanes 4-7), misses last
            unsigned key[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const unsigned kc = __shfl_sync(FULL, __float_as_uint(tn), 4 + k);
                key[k] = (cm >> k) & 1u ? kc : KEY_MISS;
            }
            sort4(key, ref);
            if (sp + 3 <= PSTACK) {
                __syncwarp();
                if (leader) {
                    int q = sp;
                    if (nh > 3) wstack[q++] = ref[3];
                    if (nh > 2) wstack[q++] = ref[2];
                    wstack[q] = ref[1];
                }
                sp += nh - 1;
            } else {
                rs.c.i(C_OVF) = 1;
            }
            node = ref[0];
            continue;
        }
        if (node == SENTINEL) {  // back to the env level
            rs.cur_inst = -1;
            ps = pslab_load(ps_env + role * PS_N);
            if (sp == 0) break;
            __syncwarp();
            node = wstack[--sp];
            continue;
        }
        const int leaf = ~node;
        if (rs.cur_inst < 0) {
            if (COUNT) cnt.insts++;
            if (sp < PSTACK) {
                __syncwarp();
                if (leader) wstack[sp] = SENTINEL;
                ++sp;
            } else {
                rs.c.i(C_OVF) = 1;
                break;
            }
            f3 oo, od;
            float delta;
            node = rs.enter_object(sv, leaf, oo, od, delta);
            ps = make_pslab<CL>(oo, od, delta);
            __syncwarp();
            if (child == 0 && lane < 8) pslab_store(ps_obj + role * PS_N, ps);
            __syncwarp();
            continue;
        }
        if (COUNT) cnt.leaves++;
        leaf_fn(leaf & LEAF_MASK);
        if (leaf >> LEAF_SHIFT) {
            if (COUNT) cnt.leaves++;
            leaf_fn((leaf & LEAF_MASK) + 1);
        }
        Umax = __int_as_float(__reduce_max_sync(FULL, __float_as_int(rs.U)));
        __syncwarp();
        ps = pslab_load(ps_obj + role * PS_N);
        if (sp == 0) break;
        node = wstack[--sp];
    }
}

// Interval-packet traversal of the BVH8 copy (nodesw): lanes 0-7 test
// child (lane & 7) against the tile's direction interval, lanes 8-15 the same
// child with the centre ray (the visiting order); lanes 16-31 mirror 0-15.
// Same conservative interval test as traverse_ipacket -- only the node width
// differs, so results are bitwise identical (tested) -- with about half the
// node visits per tile.  The hit children are ranked by the centre ray's
// entry distance (each lane counts the nearer keys of the 8, ties by child
// index) and pushed farthest first by their own lanes in one store.
template <int CL, int WW, bool COUNT, bool POPCULL, class LEAF>
__device__ __forceinline__ void traverse_ipacketw(const SceneView& sv, int env, RayState& rs,
                                                  const LEAF& leaf_fn, int* wstack, float* wdist, float* ps_env,
                                                  float* ps_obj, Counters& cnt) {
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31;
    const int child = lane & (WW - 1);
    const int role = (lane / WW) & 1;
    const bool slot_lane = lane < WW;  // lanes owning child slots for ordering / pushes
    constexpr unsigned SLOTS = WW == 32 ? 0xFFFFFFFFu : (1u << WW) - 1u;
#if AGR_SLAB_FMA
    PSlab8 ps = make_pslab8<CL, WW>(rs.o(), rs.d(), K_ERR * rs.c.f(C_Q));
    if (child == 0 && lane < 2 * WW) ps8_store(ps_env + role * PS8_N, ps);
#else
    PSlab ps = make_pslab<CL, WW>(rs.o(), rs.d(), K_ERR * rs.c.f(C_Q));
    ps.strad = __any_sync(FULL, ps.strad && role == 0) ? 1 : 0;
    if (child == 0 && lane < 2 * WW) pslab_store(ps_env + role * PS_N, ps);
#endif
    __syncwarp();
    float Umax = __int_as_float(__reduce_max_sync(FULL, __float_as_int(rs.U)));
    int sp = 0;
    int node = __ldg(sv.tlas_root + env);
    // pop the next stack entry (POPCULL: the next one the packet can still
    // reach: an entry whose pushed interval entry bound exceeds Umax, which
    // has shrunk since the push, holds no hit nearer than any lane's bound --
    // the node test's own culling criterion, re-applied; SENTINELs carry
    // -inf).  false: nothing left.  Callers check sp > 0 first.
    auto pop = [&]() -> bool {
        if constexpr (!POPCULL) {
            node = wstack[--sp];
            return true;
        } else {
            while (sp > 0) {
                --sp;
                if (!(wdist[sp] > Umax)) {
                    node = wstack[sp];
                    return true;
                }
            }
            return false;
        }
    };
    for (;;) {
        if (node >= 0) {
            if (COUNT) cnt.nodes++;
            if (COUNT && rs.cur_inst < 0) cnt.tnodes++;
            const float4* cp = sv.nodesw + 2 * WW * (size_t)node + 2 * child;
            const float4 ca = __ldg(cp), cb = __ldg(cp + 1);
            float nx, fx, ny, fy, nz, fz;
#if AGR_SLAB_FMA
            if (!ps.strad) {
                ps8_axis_fast(ca.x, ca.w, ps.neg & 1, ps.i0x, ps.i1x, ps.ex0, ps.ex1, ps.xx0, ps.xx1, nx, fx);
                ps8_axis_fast(ca.y, cb.x, ps.neg & 2, ps.i0y, ps.i1y, ps.ey0, ps.ey1, ps.xy0, ps.xy1, ny, fy);
                ps8_axis_fast(ca.z, cb.y, ps.neg & 4, ps.i0z, ps.i1z, ps.ez0, ps.ez1, ps.xz0, ps.xz1, nz, fz);
            } else {
                ps8_axis_any(ca.x, ca.w, ps.neg & 1, ps.i0x, ps.i1x, ps.ex0, ps.ex1, ps.xx0, ps.xx1, nx, fx);
                ps8_axis_any(ca.y, cb.x, ps.neg & 2, ps.i0y, ps.i1y, ps.ey0, ps.ey1, ps.xy0, ps.xy1, ny, fy);
                ps8_axis_any(ca.z, cb.y, ps.neg & 4, ps.i0z, ps.i1z, ps.ez0, ps.ez1, ps.xz0, ps.xz1, nz, fz);
            }
#else
            if (AGR_STRAD_FAST && !ps.strad) {
                pslab_axis_fast(ca.x, ca.w, ps.olx, ps.ohx, ps.i0x, ps.i1x, nx, fx);
                pslab_axis_fast(ca.y, cb.x, ps.oly, ps.ohy, ps.i0y, ps.i1y, ny, fy);
                pslab_axis_fast(ca.z, cb.y, ps.olz, ps.ohz, ps.i0z, ps.i1z, nz, fz);
            } else {
                pslab_axis(ca.x, ca.w, ps.olx, ps.ohx, ps.i0x, ps.i1x, nx, fx);
                pslab_axis(ca.y, cb.x, ps.oly, ps.ohy, ps.i0y, ps.i1y, ny, fy);
                pslab_axis(ca.z, cb.y, ps.olz, ps.ohz, ps.i0z, ps.i1z, nz, fz);
            }
#endif
            const float tn = fmaxf(fmaxf(nx, ny), fmaxf(nz, 0.0f));
            const float tf = fminf(fminf(fx, fy), fminf(fz, Umax));
            const bool h = tn <= tf;
            const int ref = __float_as_int(cb.z);
            const unsigned cm = __ballot_sync(FULL, h) & SLOTS;
            const int nh = __popc(cm);
            if (nh == 0) {
                if (sp == 0) break;
                __syncwarp();
                if (!pop()) break;
                continue;
            }
            if (nh == 1) {
                node = __shfl_sync(FULL, ref, __ffs(cm) - 1);
                continue;
            }
#if AGR_RANK_MODE == 0
            // rank of this lane's child among the hit children by the centre
            // ray's entry distance (lanes 8-15), misses last
            const unsigned kc = __shfl_sync(FULL, __float_as_uint(tn), child + WW);
            const bool hit = slot_lane && ((cm >> child) & 1u);
            const unsigned key = hit ? kc : KEY_MISS;
            int rank = 0;
#pragma unroll
            for (int j = 0; j < WW; ++j) {
                const unsigned kj = __shfl_sync(FULL, key, j);
                rank += (kj < key || (kj == key && j < child)) ? 1 : 0;
            }
            const int first = __ffs(__ballot_sync(FULL, hit && rank == 0)) - 1;
            const int nearest = __shfl_sync(FULL, ref, first);
            if (sp + WW - 1 <= PSTACK) {
                __syncwarp();  // every lane has read the slots before they are reused
                if (hit && rank > 0) wstack[sp + nh - 1 - rank] = ref;
                sp += nh - 1;  // nh is warp-uniform
            } else {
                rs.c.i(C_OVF) = 1;
            }
            node = nearest;
            continue;
#else
            // order keys: the centre ray's entry distance (lanes 8-15) with
            // the child index in the 3 low bits (distinct; near-equal
            // distances go by index), misses last; the nearest by one REDUX
            // (WW = 32: no centre lanes; the key is the interval's own entry bound)
            const unsigned kc = WW == 32 ? __float_as_uint(tn) : __shfl_sync(FULL, __float_as_uint(tn), child + WW);
            const bool hit = slot_lane && ((cm >> child) & 1u);
            const unsigned key = hit ? ((kc & ~(unsigned)(WW - 1)) | (unsigned)child) : 0xFFFFFFFFu;
            const int near_child = (int)(__reduce_min_sync(FULL, key) & (unsigned)(WW - 1));
            const int nearest = __shfl_sync(FULL, ref, near_child);
            if (sp + nh - 1 <= PSTACK) {
                __syncwarp();  // every lane has read the slots before they are reused
                if (AGR_RANK_MODE == 1 && nh > 2) {
                    int rank = 0;  // among the hits, farthest pushed first
                    if (WW <= 8) {
#pragma unroll
                        for (int j = 0; j < WW; ++j) rank += __shfl_sync(FULL, key, j) < key ? 1 : 0;
                    } else {
                        // wide nodes: compare with the other hits only (a
                        // warp-uniform loop of nh - 1 steps, not WW)
                        rank = 1;
                        for (unsigned m = cm & ~(1u << near_child); m; m &= m - 1u)
                            rank += __shfl_sync(FULL, key, __ffs(m) - 1) < key ? 1 : 0;
                        if (child == near_child) rank = 0;
                    }
                    if (hit && rank > 0) {
                        wstack[sp + nh - 1 - rank] = ref;
                        if (POPCULL) wdist[sp + nh - 1 - rank] = tn;
                    }
                } else if (hit && child != near_child) {
                    // nh == 2 (exact), or mode 2: the other hits in child order
                    const unsigned others = cm & ~(1u << near_child);
                    wstack[sp + __popc(others & ((1u << child) - 1u))] = ref;
                    if (POPCULL) wdist[sp + __popc(others & ((1u << child) - 1u))] = tn;
                }
                sp += nh - 1;  // nh is warp-uniform
            } else {
                rs.c.i(C_OVF) = 1;
            }
            node = nearest;
            continue;
#endif
        }
        if (node == SENTINEL) {  // back to the env level
            rs.cur_inst = -1;
#if AGR_SLAB_FMA
            ps = ps8_load(ps_env + role * PS8_N);
#else
            ps = pslab_load(ps_env + role * PS_N);
#endif
            if (sp == 0) break;
            __syncwarp();
            if (!pop()) break;
            continue;
        }
        const int leaf = ~node;
        if (rs.cur_inst < 0) {
            if (COUNT) cnt.insts++;
            if (sp < PSTACK) {
                __syncwarp();
                if (lane == 0) {
                    wstack[sp] = SENTINEL;
                    if (POPCULL) wdist[sp] = -inf_f();
                }
                ++sp;
            } else {
                rs.c.i(C_OVF) = 1;
                break;
            }
            f3 oo, od;
            float delta;
            node = rs.enter_object(sv, leaf, oo, od, delta);
#if AGR_SLAB_FMA
            ps = make_pslab8<CL, WW>(oo, od, delta);
            __syncwarp();
            if (child == 0 && lane < 2 * WW) ps8_store(ps_obj + role * PS8_N, ps);
#else
            ps = make_pslab<CL, WW>(oo, od, delta);
            ps.strad = __any_sync(FULL, ps.strad && role == 0) ? 1 : 0;
            __syncwarp();
            if (child == 0 && lane < 2 * WW) pslab_store(ps_obj + role * PS_N, ps);
#endif
            __syncwarp();
            continue;
        }
        if (COUNT) cnt.leaves++;
        leaf_fn(leaf & LEAF_MASK);
        if (leaf >> LEAF_SHIFT) {
            if (COUNT) cnt.leaves++;
            leaf_fn((leaf & LEAF_MASK) + 1);
        }
        Umax = __int_as_float(__reduce_max_sync(FULL, __float_as_int(rs.U)));
        __syncwarp();
#if AGR_SLAB_FMA
        if (AGR_PS_RELOAD) ps = ps8_load(ps_obj + role * PS8_N);
#else
        if (AGR_PS_RELOAD) ps = pslab_load(ps_obj + role * PS_N);
#endif
        if (sp == 0) break;
        if (!pop()) break;
    }
}

// ---- ray generation -----------------------------------------------------------------
struct RayId {
    int env;
    int64_t out;     // output element index
    bool active;
    int col, row, sensor;
};

__device__ __forceinline__ void pose_ray(const float* P, f3 ds, f3& o, f3& d) {
    o = mk(__ldg(P + 3), __ldg(P + 7), __ldg(P + 11));
    d = mk(fmaf(__ldg(P + 0), ds.x, fmaf(__ldg(P + 1), ds.y, __ldg(P + 2) * ds.z)),
           fmaf(__ldg(P + 4), ds.x, fmaf(__ldg(P + 5), ds.y, __ldg(P + 6) * ds.z)),
           fmaf(__ldg(P + 8), ds.x, fmaf(__ldg(P + 9), ds.y, __ldg(P + 10) * ds.z)));
}

__device__ __forceinline__ void pose_ray64(const float* P, d3 ds, Ray64& r) {
    double p[12];
#pragma unroll
    for (int k = 0; k < 12; ++k) p[k] = (double)__ldg(P + k);
    r.o = mkd(p[3], p[7], p[11]);
    r.d = mkd(p[0] * ds.x + p[1] * ds.y + p[2] * ds.z,
              p[4] * ds.x + p[5] * ds.y + p[6] * ds.z,
              p[8] * ds.x + p[9] * ds.y + p[10] * ds.z);
}

// FP32 ray for traversal (a4: raygen fused into the cast; registers only).
template <int MODEL>
__device__ __forceinline__ void gen_ray(const CastArgs& a, const RayId& id, f3& o, f3& d) {
    if (MODEL == 0) {
        const float* po = a.orig + 3 * id.out;
        const float* pd = a.dir + 3 * id.out;
        o = mk(__ldg(po), __ldg(po + 1), __ldg(po + 2));
        d = mk(__ldg(pd), __ldg(pd + 1), __ldg(pd + 2));
        return;
    }
    const float* P = a.poses + 12 * ((int64_t)id.env * a.S + id.sensor);
    f3 ds;
    if (MODEL == 1) {
        float xs = __fdividef((float)id.col + 0.5f - a.cx, a.fx);
        float ys = __fdividef((float)id.row + 0.5f - a.cy, a.fy);
        ds = mk(1.0f, -xs, -ys);
        if (a.kind == 1) {
            float rn = rsqrtf(dot(ds, ds));
            ds = mk(ds.x * rn, ds.y * rn, ds.z * rn);
        }
    } else {
        const float* b = a.beams + 3 * ((int64_t)id.row * a.W + id.col);
        ds = mk(__ldg(b), __ldg(b + 1), __ldg(b + 2));
        float rn = rsqrtf(dot(ds, ds));
        ds = mk(ds.x * rn, ds.y * rn, ds.z * rn);
    }
    pose_ray(P, ds, o, d);
}

// FP64 ray of the same pixel / beam from the same FP32 inputs (DESIGN.md §3:
// the plain definition promotes the inputs to FP64); built lazily, only when
// a candidate is arbitrated, so it holds no registers during traversal.
template <int MODEL>
__device__ __forceinline__ Ray64 gen_ray64(const CastArgs& a, const RayId& id) {
    Ray64 r64;
    if (MODEL == 0) {
        const float* po = a.orig + 3 * id.out;
        const float* pd = a.dir + 3 * id.out;
        r64.o = mkd(__ldg(po), __ldg(po + 1), __ldg(po + 2));
        r64.d = mkd(__ldg(pd), __ldg(pd + 1), __ldg(pd + 2));
        return r64;
    }
    const float* P = a.poses + 12 * ((int64_t)id.env * a.S + id.sensor);
    d3 ds64;
    if (MODEL == 1) {
        double xs64 = ((double)id.col + 0.5 - (double)a.cx) * a.inv_fx64;
        double ys64 = ((double)id.row + 0.5 - (double)a.cy) * a.inv_fy64;
        ds64 = mkd(1.0, -xs64, -ys64);
        if (a.kind == 1) {
            double n = sqrt(dotd(ds64, ds64));
            ds64 = mkd(ds64.x / n, ds64.y / n, ds64.z / n);
        }
    } else {
        const float* b = a.beams + 3 * ((int64_t)id.row * a.W + id.col);
        ds64 = mkd(__ldg(b), __ldg(b + 1), __ldg(b + 2));
        double n = sqrt(dotd(ds64, ds64));
        ds64 = mkd(ds64.x / n, ds64.y / n, ds64.z / n);
    }
    pose_ray64(P, ds64, r64);
    return r64;
}

// ---- f2: stereo shadow segments ------------------------------------------------------
// FP64 segment from the FP64 hit point p = o + t d towards the second
// sensor's origin o2 = P (stereo offset) (reading R21).
// Returns its length L (<= 0 when undefined) and the unit direction.
template <int MODEL>
__device__ __forceinline__ double shadow_ray64(const CastArgs* a, int env, int sensor, int col, int row,
                                               double t_hit, Ray64& sr) {
    RayId id;
    id.env = env;
    id.sensor = sensor;
    id.col = col;
    id.row = row;
    id.out = 0;
    id.active = true;
    const Ray64 r = gen_ray64<MODEL>(*a, id);
    const float* P = a->poses + 12 * ((int64_t)env * a->S + sensor);
    const d3 off = mkd(a->stereo[0], a->stereo[1], a->stereo[2]);
    const d3 o2 = mkd((double)P[0] * off.x + (double)P[1] * off.y + (double)P[2] * off.z + (double)P[3],
                      (double)P[4] * off.x + (double)P[5] * off.y + (double)P[6] * off.z + (double)P[7],
                      (double)P[8] * off.x + (double)P[9] * off.y + (double)P[10] * off.z + (double)P[11]);
    const d3 p = mkd(r.o.x + t_hit * r.d.x, r.o.y + t_hit * r.d.y, r.o.z + t_hit * r.d.z);
    const d3 v = subd(o2, p);
    const double L = sqrt(dotd(v, v));
    sr.o = p;
    sr.d = L > 0.0 ? mkd(v.x / L, v.y / L, v.z / L) : mkd(1.0, 0.0, 0.0);
    return L;
}

template <int MODEL>
__device__ __noinline__ float shadow_segment(const CastArgs* a, int env, int sensor, int col, int row,
                                             double t_hit, float3* o32, float3* d32) {
    Ray64 sr;
    const double L = shadow_ray64<MODEL>(a, env, sensor, col, row, t_hit, sr);
    *o32 = make_float3((float)sr.o.x, (float)sr.o.y, (float)sr.o.z);
    *d32 = make_float3((float)sr.d.x, (float)sr.d.y, (float)sr.d.z);
    return (float)L;
}

// FP64 decision for an uncertain shadow candidate: hit with t in (eps, L - eps).
template <int MODEL>
__device__ __forceinline__ RayId ray_id(const CastArgs& a);

// Ray identity of this lane from its cold column (written once by the
// kernel), so an FP64 test does not redo the tile decode.
template <int MODEL>
__device__ __forceinline__ RayId cold_id(const CastArgs& a) {
    if (MODEL == 0) return ray_id<MODEL>(a);
    RayId id;
    id.col = __float_as_int(s_cold[C_COL][threadIdx.x]);
    id.row = __float_as_int(s_cold[C_ROW][threadIdx.x]);
    const int img = __float_as_int(s_cold[C_IMG][threadIdx.x]);
    id.env = img / a.S;  // only used with id.sensor through env * S + sensor
    id.sensor = img - id.env * a.S;
    id.out = 0;
    id.active = true;
    return id;
}

template <int MODEL>
__device__ __noinline__ bool shadow_test64(const CastArgs* a, double t_hit, int inst, int leaf) {
    RayId id = ray_id<MODEL>(*a);
    id.col = min(id.col, a->W - 1);
    id.row = min(id.row, a->H - 1);
    Ray64 sr;
    const double L = shadow_ray64<MODEL>(a, id.env, id.sensor, id.col, id.row, t_hit, sr);
    double t;
    const double eps = (double)a->stereo_eps;
    return tri64(a->sv, inst, leaf, sr, t) && t > eps && t < L - eps;
}

// Stack-overflow fallback of the shadow query: every triangle of the env.
template <int MODEL>
__device__ __noinline__ bool shadow_brute64(const CastArgs* a, int env, double t_hit) {
    RayId id = ray_id<MODEL>(*a);
    id.col = min(id.col, a->W - 1);
    id.row = min(id.row, a->H - 1);
    Ray64 sr;
    const double L = shadow_ray64<MODEL>(a, env, id.sensor, id.col, id.row, t_hit, sr);
    const double eps = (double)a->stereo_eps;
    for (int inst = __ldg(a->sv.env_off + env); inst < __ldg(a->sv.env_off + env + 1); ++inst) {
        const int as = __ldg(a->sv.inst_asset + inst);
        for (int p = __ldg(a->sv.part_off + as); p < __ldg(a->sv.part_off + as + 1); ++p) {
            const BlasInfo& bl = a->sv.parts[p];
            for (int l = 0; l < bl.n_leaves; ++l) {
                double t;
                if (tri64(a->sv, inst, bl.leaf_base + l, sr, t) && t > eps && t < L - eps) return true;
            }
        }
    }
    return false;
}

// Out-of-line FP64 test of (inst, leaf) for the ray `id`: keeps the FP64
// registers out of the traversal loop's allocation.
template <int MODEL>
__device__ __noinline__ void resolve_leaf64(const CastArgs* a, int inst, int leaf, Best64* best) {
    const RayId id = cold_id<MODEL>(*a);
    const Ray64 r = gen_ray64<MODEL>(*a, id);
    Best64 b = *best;
    consider64(a->sv, inst, leaf, r, (double)a->max_range, b);
    *best = b;
}

// FP64 arbitration of every candidate slot with t_lo <= U,
// reading the slots and the ray identity from the lane's cold column.
template <int MODEL>
__device__ __noinline__ void arbitrate64(const CastArgs* a, float U, Best64* best) {
    const RayId id = cold_id<MODEL>(*a);
    const Ray64 r = gen_ray64<MODEL>(*a, id);
    Best64 b = *best;
    const int t = threadIdx.x;
#pragma unroll
    for (int k = 0; k < NSLOT; ++k) {
        if (s_cold[C_TL0 + k][t] <= U)
            consider64(a->sv, __float_as_int(s_cold[C_INST0 + k][t]), __float_as_int(s_cold[C_LEAF0 + k][t]), r,
                       (double)a->max_range, b);
    }
    *best = b;
}

// Per-hit channels of PAPER.md:218 / :228 (surface normal, barycentrics,
// point cloud), in FP64 from the winning triangle (reading R20).
template <int MODEL>
__device__ __noinline__ void write_extra(const CastArgs* a, RayId id, Best64 best) {
    const Ray64 r = gen_ray64<MODEL>(*a, id);
    const int64_t o = id.out;
    double t = best.face >= 0 ? best.t : (double)a->max_range;
    if (a->out_point) {
        a->out_point[3 * o + 0] = (float)(r.o.x + t * r.d.x);
        a->out_point[3 * o + 1] = (float)(r.o.y + t * r.d.y);
        a->out_point[3 * o + 2] = (float)(r.o.z + t * r.d.z);
    }
    if (!a->out_normal && !a->out_bary && !a->out_annot) return;
    const int K = a->sv.annot_k;
    if (best.face < 0) {
        if (a->out_normal) a->out_normal[3 * o] = a->out_normal[3 * o + 1] = a->out_normal[3 * o + 2] = 0.0f;
        if (a->out_bary) a->out_bary[2 * o] = a->out_bary[2 * o + 1] = -1.0f;
        if (a->out_annot)
            for (int k = 0; k < K; ++k) a->out_annot[(int64_t)K * o + k] = __int_as_float(0x7fc00000);
        return;
    }
    const float* T = a->sv.inst_T + 12 * best.inst;
    const float4* v = reinterpret_cast<const float4*>(a->sv.triv) + 3 * (size_t)best.leaf;
    d3 w[3];
    for (int c = 0; c < 3; ++c) {
        const float4 q = v[c];
        double x = q.x, y = q.y, z = q.z;
        w[c].x = (double)T[0] * x + (double)T[1] * y + (double)T[2] * z + (double)T[3];
        w[c].y = (double)T[4] * x + (double)T[5] * y + (double)T[6] * z + (double)T[7];
        w[c].z = (double)T[8] * x + (double)T[9] * y + (double)T[10] * z + (double)T[11];
    }
    const d3 e1 = subd(w[1], w[0]), e2 = subd(w[2], w[0]);
    d3 n = crossd(e1, e2);
    if (a->out_normal) {
        double s = 1.0 / sqrt(dotd(n, n));
        if (dotd(n, r.d) > 0.0) s = -s;  // face the ray origin
        a->out_normal[3 * o + 0] = (float)(n.x * s);
        a->out_normal[3 * o + 1] = (float)(n.y * s);
        a->out_normal[3 * o + 2] = (float)(n.z * s);
    }
    if (a->out_bary || a->out_annot) {
        // Moller-Trumbore barycentrics of the FP64 ray: weights of v1, v2
        const d3 p = crossd(r.d, e2);
        const double det = dotd(e1, p);
        const d3 s = subd(r.o, w[0]);
        const double b1 = dotd(s, p) / det;
        const d3 q = crossd(s, e1);
        const double b2 = dotd(r.d, q) / det;
        if (a->out_bary) {
            a->out_bary[2 * o + 0] = (float)b1;
            a->out_bary[2 * o + 1] = (float)b2;
        }
        if (a->out_annot) {
            // PAPER.md:228 vertex-level annotations of the winning face,
            // interpolated with its FP64 barycentrics (reading R23)
            const int asset = __ldg(a->sv.inst_asset + best.inst);
            const int f = __float_as_int(__ldg(&a->sv.tris[3 * best.leaf + 2].w));  // asset-local face
            const int* fv = a->sv.mesh_faces + 3 * (int64_t)(__ldg(a->sv.asset_foff + asset) + f);
            const int vb = __ldg(a->sv.asset_voff + asset);
            const float* A0 = a->sv.annot + (int64_t)K * (vb + __ldg(fv));
            const float* A1 = a->sv.annot + (int64_t)K * (vb + __ldg(fv + 1));
            const float* A2 = a->sv.annot + (int64_t)K * (vb + __ldg(fv + 2));
            for (int k = 0; k < K; ++k)
                a->out_annot[(int64_t)K * o + k] =
                    (float)((1.0 - b1 - b2) * (double)__ldg(A0 + k) + b1 * (double)__ldg(A1 + k) +
                            b2 * (double)__ldg(A2 + k));
        }
    }
}

// n / d for n < 2^31 with m = floor(2^(31+l) / d) + 1, s = 31 + l,
// l = ceil(log2 d): n m / 2^s = n / d + n e / 2^s with 0 < e <= 1, and
// n e / 2^s < 2^-l <= 1 / d, which never carries past the next integer.
__device__ __forceinline__ unsigned fast_div(unsigned n, unsigned m, int s) {
    return (unsigned)(((unsigned long long)n * m) >> s);
}

template <int MODEL>
__device__ __forceinline__ RayId ray_id(const CastArgs& a) {
    RayId id;
    id.sensor = 0;
    id.col = id.row = 0;
    if (MODEL == 0) {
        int bpe = (a.R + CAST_THREADS - 1) / CAST_THREADS;
        int e = a.env_begin + blockIdx.x / bpe;
        int r = (blockIdx.x % bpe) * CAST_THREADS + threadIdx.x;
        id.env = e;
        id.active = r < a.R && e < a.env_end;
        id.out = (int64_t)(e - a.out_env_base) * a.R + (id.active ? r : 0);
        return id;
    }
    // 32-bit index math: a launch covers < 2^32 warps (grid.x < 2^31 blocks
    // of CAST_THREADS / 32 = 2 warps) and tiles_img < 2^31 (cast_launch)
    constexpr int TILE_W = Tile<MODEL>::W, TILE_H = Tile<MODEL>::H;
    const unsigned tiles_x = (unsigned)(a.W + TILE_W - 1) / TILE_W;
    const unsigned tiles_img = tiles_x * (unsigned)((a.H + TILE_H - 1) / TILE_H);
    const unsigned warp = blockIdx.x * (unsigned)(CAST_THREADS / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    const unsigned img = fast_div(warp, a.div_m[0], a.div_s[0]);
    const unsigned tile = warp - img * tiles_img;
    const unsigned ty = fast_div(tile, a.div_m[1], a.div_s[1]), tx = tile - ty * tiles_x;
    const unsigned env_rel = a.S == 1 ? img : fast_div(img, a.div_m[2], a.div_s[2]);
    id.env = a.env_begin + (int)env_rel;
    id.sensor = (int)(img - env_rel * (unsigned)a.S);
    id.col = (int)tx * TILE_W + (lane % TILE_W);
    id.row = (int)ty * TILE_H + (lane / TILE_W);
    id.active = id.env < a.env_end && id.col < a.W && id.row < a.H;
    id.out = (((int64_t)(id.env - a.out_env_base) * a.S + id.sensor) * a.H + id.row) * a.W + id.col;
    return id;
}

// TRAV: 0 per-lane FP32 filter, 1 warp packet (pinhole / beams), 2 exact (FP64 leaves)
template <int MODEL, int TRAV, bool COUNT, bool STEREO, int WIDE>
__global__ void __launch_bounds__(CAST_THREADS, cast_min_blocks(MODEL, TRAV)) k_cast(const __grid_constant__ CastArgs a) {
    __shared__ int s_stack[TRAV == 1 ? CAST_THREADS / 32 : 1][TRAV == 1 ? PSTACK : 1];
    // pushed entry bounds of the pop-time culling (pinhole tiles: c5 +7.5 %,
    // c3 +0.7 %; LiDAR beam tiles -2.3 %, so they keep the plain pops)
    constexpr bool POPC = TRAV == 1 && AGR_POP_CULL && MODEL == 1;
    __shared__ float s_stackd[POPC ? CAST_THREADS / 32 : 1][POPC ? PSTACK : 1];
    __shared__ __align__(16) float s_pslab[TRAV == 1 ? CAST_THREADS / 32 : 1][2][2 * PS_MAXN];  // [warp][env, obj][role][..]
    RayId id = ray_id<MODEL>(a);
    // ragged tile lanes keep the warp whole for the traversal: they trace a
    // copy of a valid pixel and store nothing
    const bool trace = id.env < a.env_end && (id.active || MODEL != 0);
    id.col = min(id.col, a.W - 1);
    id.row = min(id.row, a.H - 1);
    Counters cnt = {0, 0, 0, 0, 0, 0, 0};
    RayState rs;
    Best64 best;
    best.face = -1;
    best.inst = -1;
    best.t = 0.0;
    if (trace) {
        f3 o, d;
        gen_ray<MODEL>(a, id, o, d);
        Cold cold;
        cold.p = &s_cold[0][threadIdx.x];
        cold.bt = &s_best_t[threadIdx.x];
        rs.init(o, d, a.max_range, cold);
        cold.i(C_COL) = id.col;
        cold.i(C_ROW) = id.row;
        cold.i(C_IMG) = id.env * a.S + id.sensor;
        const CastArgs* ap = &a;
        auto res = [ap](int inst, int leaf, Best64& b) { resolve_leaf64<MODEL>(ap, inst, leaf, &b); };
        if (TRAV == 2) {
            auto leaf_fn = [&](int leaf) {
                if (COUNT) cnt.f64++;
                rs.resolve64(leaf, res);
            };
            traverse_lane<false, COUNT>(a.sv, id.env, rs, leaf_fn, cnt);
            best = cold.best();
        } else {
            auto leaf_fn = [&](int leaf) { rs.leaf_filter<COUNT>(a.sv, leaf, res, cnt); };
            if (TRAV == 1) {
                // whole warps share (env, sensor): pinhole / beams tiles
#if AGR_IPACKET
                if (WIDE)
                    traverse_ipacketw<Tile<MODEL>::CL, WIDE ? WIDE : 8, COUNT, AGR_POP_CULL && MODEL == 1>(
                        a.sv, id.env, rs, leaf_fn, s_stack[threadIdx.x >> 5], s_stackd[POPC ? threadIdx.x >> 5 : 0],
                        s_pslab[threadIdx.x >> 5][0],
                        s_pslab[threadIdx.x >> 5][1], cnt);
                else
                    traverse_ipacket<Tile<MODEL>::CL, COUNT>(a.sv, id.env, rs, leaf_fn, s_stack[threadIdx.x >> 5],
                                            s_pslab[threadIdx.x >> 5][0], s_pslab[threadIdx.x >> 5][1], cnt);
#else
                traverse_packet<Tile<MODEL>::CL, false, COUNT>(a.sv, id.env, rs, leaf_fn, s_stack[threadIdx.x >> 5], cnt);
#endif
            } else {
                traverse_lane<false, COUNT>(a.sv, id.env, rs, leaf_fn, cnt);
            }
            // final arbitration: one out-of-line call per lane that builds the
            // FP64 ray once for all of its surviving candidates
            best = cold.best();
            bool any = false;
#pragma unroll
            for (int k = 0; k < NSLOT; ++k) {
                const bool live = cold.f(C_TL0 + k) <= rs.U;
                if (COUNT && live) cnt.f64++;
                any |= live;
            }
            if (any) arbitrate64<MODEL>(&a, rs.U, &best);
        }
        if (cold.i(C_OVF)) {
            if (COUNT) cnt.overflow++;
            best.face = -1;
            brute64(a.sv, id.env, gen_ray64<MODEL>(a, id), (double)a.max_range, &best);
        }
    }
    // f2: stereo shadow mask -- an any-hit segment from the hit
    // point to the second sensor; every lane of the warp takes part.
    bool valid = true;
    if (STEREO && MODEL != 0 && id.env < a.env_end) {
        // recomputed (not kept live across the primary traversal)
        id = ray_id<MODEL>(a);
        id.col = min(id.col, a.W - 1);
        id.row = min(id.row, a.H - 1);
        float3 sp32, sd32;
        float seg_max = -1.0f;
        if (trace && best.face >= 0) seg_max = shadow_segment<MODEL>(&a, id.env, id.sensor, id.col, id.row, best.t, &sp32, &sd32);
        if (!(seg_max > a.stereo_eps)) { sp32 = make_float3(0.f, 0.f, 0.f); sd32 = make_float3(1.f, 0.f, 0.f); }
        Cold cold;
        cold.p = &s_cold[0][threadIdx.x];
        cold.bt = &s_best_t[threadIdx.x];
        RayState ss;
        ss.init(mk(sp32.x, sp32.y, sp32.z), mk(sd32.x, sd32.y, sd32.z), fmaxf(seg_max - a.stereo_eps, 0.0f), cold);
        ss.tmin = a.stereo_eps;
        const bool tested = seg_max > 2.0f * a.stereo_eps;
        if (!tested) ss.U = -1.0f;  // nothing to test: valid
        const CastArgs* ap = &a;
        const Best64 prim = best;
        auto sres = [ap, prim](int inst, int leaf) { return shadow_test64<MODEL>(ap, prim.t, inst, leaf); };
        auto leaf_fn = [&](int leaf) { ss.leaf_anyhit<COUNT>(a.sv, leaf, sres, cnt); };
        if (TRAV == 1) traverse_packet<Tile<MODEL>::CL, true, COUNT>(a.sv, id.env, ss, leaf_fn, s_stack[threadIdx.x >> 5], cnt);
        else traverse_lane<true, COUNT>(a.sv, id.env, ss, leaf_fn, cnt);
        valid = !tested || ss.U >= 0.0f;
        if (cold.i(C_OVF) && tested) valid = !shadow_brute64<MODEL>(&a, id.env, best.t);
    }
    if (COUNT) {
        unsigned v[7] = {cnt.nodes, cnt.leaves, cnt.insts, cnt.f64, cnt.overflow, cnt.tnodes, cnt.empty};
        unsigned rays = id.active ? 1u : 0u;
        for (int o2 = 16; o2 > 0; o2 >>= 1) {
            rays += __shfl_xor_sync(0xFFFFFFFFu, rays, o2);
            for (int k = 0; k < 7; ++k) v[k] += __shfl_xor_sync(0xFFFFFFFFu, v[k], o2);
        }
        if ((threadIdx.x & 31) == 0) {
            atomicAdd(a.counters + 0, (unsigned long long)rays);
            for (int k = 0; k < 7; ++k) atomicAdd(a.counters + 1 + k, (unsigned long long)v[k]);
        }
    }
    if (!id.active) return;
    const bool hit = best.face >= 0;
    // streaming stores: the images are written once and must not evict the
    // L2-resident BVH
    if (a.out_dist) __stcs(a.out_dist + id.out, hit ? (float)best.t : a.max_range);
    if (a.out_seg) __stcs(a.out_seg + id.out, hit ? __ldg(a.sv.inst_label + best.inst) : -1);
    if (a.out_face) __stcs(a.out_face + id.out, hit ? best.face : -1);
    if (a.out_normal || a.out_bary || a.out_point || a.out_annot) write_extra<MODEL>(&a, id, best);
    if (a.out_valid) __stcs(a.out_valid + id.out, valid ? 1 : 0);  // 1 without STEREO (explicit rays)
}

template <int MODEL>
cudaError_t launch_model(CastArgs a, cudaStream_t stream) {
    constexpr int TILE_W = Tile<MODEL>::W, TILE_H = Tile<MODEL>::H;
    int64_t blocks;
    int n_envs = a.env_end - a.env_begin;
    if (n_envs <= 0) return cudaSuccess;
    if (MODEL == 0) {
        blocks = (int64_t)n_envs * ((a.R + CAST_THREADS - 1) / CAST_THREADS);
    } else {
        const int64_t tiles_img = (int64_t)((a.W + TILE_W - 1) / TILE_W) * ((a.H + TILE_H - 1) / TILE_H);
        if (tiles_img > 0x7FFFFFFF) return cudaErrorInvalidValue;  // ray_id's 32-bit math
        int64_t tiles = tiles_img * n_envs * a.S;
        if (tiles > 0x7FFFFFFF) return cudaErrorInvalidValue;  // fast_div needs warp < 2^31
        blocks = (tiles + CAST_THREADS / 32 - 1) / (CAST_THREADS / 32);
    }
    if (blocks <= 0) return cudaSuccess;
    if (blocks > 0x7FFFFFFF) return cudaErrorInvalidValue;
    const int trav = a.exact ? 2 : (MODEL != 0 && a.packet ? 1 : 0);
    const unsigned g = (unsigned)blocks;
    if (MODEL != 0) {
        const unsigned tiles_x = (unsigned)(a.W + TILE_W - 1) / TILE_W;
        const unsigned ds[3] = {tiles_x * (unsigned)((a.H + TILE_H - 1) / TILE_H), tiles_x, (unsigned)a.S};
        for (int k = 0; k < 3; ++k) {
            int l = 0;
            while ((1ull << l) < ds[k]) ++l;
            a.div_m[k] = (unsigned)((1ull << (31 + l)) / ds[k] + 1);
            a.div_s[k] = 31 + l;
        }
    }
    const bool stereo = MODEL != 0 && a.out_valid != nullptr;
#define AGR_LAUNCH(T, C, S, W) k_cast<MODEL, T, C, S, W><<<g, CAST_THREADS, 0, stream>>>(a)
#define AGR_LAUNCH_TRAV(C, S)                                   \
    do {                                                        \
        if (trav == 2) AGR_LAUNCH(2, C, S, 0);                  \
        else if (trav == 0) AGR_LAUNCH(0, C, S, 0);             \
        else if (wide == 32) AGR_LAUNCH(1, C, S, 32);           \
        else if (wide == 16) AGR_LAUNCH(1, C, S, 16);           \
        else if (wide == 8) AGR_LAUNCH(1, C, S, 8);             \
        else AGR_LAUNCH(1, C, S, 0);                            \
    } while (0)
    const int wide = a.wide ? a.sv.wide_w : 0;
    if (a.counters) {
        if (stereo) AGR_LAUNCH_TRAV(true, true);
        else AGR_LAUNCH_TRAV(true, false);
    } else {
        if (stereo) AGR_LAUNCH_TRAV(false, true);
        else AGR_LAUNCH_TRAV(false, false);
    }
#undef AGR_LAUNCH_TRAV
#undef AGR_LAUNCH
    return cudaGetLastError();
}

}  // namespace

cudaError_t cast_launch(const CastArgs& a, cudaStream_t stream) {
    switch (a.model) {
        case 0: return launch_model<0>(a, stream);
        case 1: return launch_model<1>(a, stream);
        case 2: return launch_model<2>(a, stream);
    }
    return cudaErrorInvalidValue;
}

}  // namespace agr
