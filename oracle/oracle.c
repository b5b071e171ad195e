/*
 * oracle.c -- CPU brute-force ray-casting ORACLE.  TEST INFRASTRUCTURE ONLY
 * (see oracle.h for who may call it and for the definition it implements).
 *
 * Plain, slow and obviously correct: for each queried ray, every triangle of
 * the ray's environment is tested in double precision.  No BVH, no blocking,
 * no reordering beyond the plain definition of SURVEY.md §8(c).
 *
 * Paper passages followed (§III.D.1 "Exteroceptive Sensors"):
 *   l.226  M^base_i = {M_j}; M_{i,t} = T_{i,t} o M^base_i -- every vertex of
 *          sub-mesh j is transformed by T_{j,t}  -> world_triangles()
 *   l.228  "individual rays are cast outwards per-pixel to evaluate
 *          intersection with M_{i,t}"            -> make_ray(), cast_one()
 *   l.228  range for ToF/LiDAR, depth = distance from the image plane
 *                                                 -> make_ray() direction scaling
 *   l.218  depth / segmentation / face-index images -> outputs
 * Readings of silent or garbled points are DESIGN.md §"Readings" R1-R18.
 */
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

static int64_t g_last_tests = 0;

int64_t oracle_last_tests(void) { return g_last_tests; }

/* ---- small FP64 vector helpers ---------------------------------------- */
typedef struct { double x, y, z; } v3;

static v3 vsub(v3 a, v3 b) { v3 r = {a.x - b.x, a.y - b.y, a.z - b.z}; return r; }
static double vdot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static v3 vcross(v3 a, v3 b) {
    v3 r = {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
    return r;
}
static double vnorm(v3 a) { return sqrt(vdot(a, a)); }

/* ---- the env's merged mesh M_{e,t} in FP64 -------------- */
typedef struct {
    int64_t n_tri;
    v3* v;          /* [n_tri][3] world (env-local) vertices */
    int32_t* label; /* [n_tri] label of the owning instance  */
    int64_t* vid;   /* [n_tri][3] scene-global vertex ids (annotations) */
    int64_t cap;
} world_mesh;

static int64_t env_tri_count(const oracle_scene* sc, int32_t e) {
    int64_t n = 0;
    for (int64_t j = sc->env_off[e]; j < sc->env_off[e + 1]; ++j) {
        int32_t a = sc->inst_asset[j];
        n += sc->face_off[a + 1] - sc->face_off[a];
    }
    return n;
}

/* Transform every vertex of every sub-mesh of env e: x' = A x + b, with the
 * FP32 inputs promoted to double.  Triangles are laid out in the per-env face
 * numbering of DESIGN.md reading R2: instances in creation order, faces in
 * asset order, so triangle k of this array has face index k. */
static int world_triangles(const oracle_scene* sc, int32_t e, world_mesh* w) {
    int64_t n = env_tri_count(sc, e);
    if (n > w->cap) {
        free(w->v);
        free(w->label);
        free(w->vid);
        w->v = (v3*)malloc(sizeof(v3) * 3 * (size_t)(n > 0 ? n : 1));
        w->label = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
        w->vid = (int64_t*)malloc(sizeof(int64_t) * 3 * (size_t)(n > 0 ? n : 1));
        if (!w->v || !w->label || !w->vid) return -1;
        w->cap = n;
    }
    int64_t k = 0;
    for (int64_t j = sc->env_off[e]; j < sc->env_off[e + 1]; ++j) {
        int32_t a = sc->inst_asset[j];
        const float* T = sc->inst_T + 12 * j;
        for (int64_t f = sc->face_off[a]; f < sc->face_off[a + 1]; ++f, ++k) {
            for (int c = 0; c < 3; ++c) {
                int64_t vi = sc->vert_off[a] + sc->faces[3 * f + c];
                w->vid[3 * k + c] = vi;
                const float* p = sc->verts + 3 * vi;
                double x = p[0], y = p[1], z = p[2];
                v3 q;
                q.x = (double)T[0] * x + (double)T[1] * y + (double)T[2] * z + (double)T[3];
                q.y = (double)T[4] * x + (double)T[5] * y + (double)T[6] * z + (double)T[7];
                q.z = (double)T[8] * x + (double)T[9] * y + (double)T[10] * z + (double)T[11];
                w->v[3 * k + c] = q;
            }
            w->label[k] = sc->inst_label[j];
        }
    }
    w->n_tri = n;
    return 0;
}

/* ---- ray generation (readings R6-R9) ----- */
static int64_t query_env(const oracle_rays* r, int64_t id) {
    if (r->model == ORACLE_RAYS) return id / r->R;
    if (r->model == ORACLE_PINHOLE) return id / ((int64_t)r->S * r->H * r->W);
    return id / ((int64_t)r->S * r->C * r->K);
}

static void make_ray(const oracle_rays* r, int64_t id, v3* o, v3* d) {
    if (r->model == ORACLE_RAYS) {
        const float* po = r->orig + 3 * id;
        const float* pd = r->dir + 3 * id;
        o->x = po[0]; o->y = po[1]; o->z = po[2];
        d->x = pd[0]; d->y = pd[1]; d->z = pd[2];
        return;
    }
    v3 ds;
    int64_t es; /* flat (env, sensor) index */
    if (r->model == ORACLE_PINHOLE) {
        int64_t u = id % r->W;
        int64_t v = (id / r->W) % r->H;
        es = id / ((int64_t)r->W * r->H);
        /* pixel centre (u+0.5, v+0.5); x forward, y left (u right), z up (v down) */
        double xs = ((double)u + 0.5 - (double)r->cx) / (double)r->fx;
        double ys = ((double)v + 0.5 - (double)r->cy) / (double)r->fy;
        ds.x = 1.0; ds.y = -xs; ds.z = -ys;
        if (r->kind == ORACLE_RANGE) {
            double n = vnorm(ds);
            ds.x /= n; ds.y /= n; ds.z /= n;
        }
    } else {
        int64_t k = id % r->K;
        int64_t c = (id / r->K) % r->C;
        es = id / ((int64_t)r->K * r->C);
        const float* b = r->beams + 3 * (c * r->K + k);
        ds.x = b[0]; ds.y = b[1]; ds.z = b[2];
        double n = vnorm(ds);
        ds.x /= n; ds.y /= n; ds.z /= n;
    }
    const float* P = r->poses + 12 * es; /* columns = sensor axes in env frame */
    d->x = (double)P[0] * ds.x + (double)P[1] * ds.y + (double)P[2] * ds.z;
    d->y = (double)P[4] * ds.x + (double)P[5] * ds.y + (double)P[6] * ds.z;
    d->z = (double)P[8] * ds.x + (double)P[9] * ds.y + (double)P[10] * ds.z;
    o->x = P[3]; o->y = P[7]; o->z = P[11];
}

/* ---- one ray against every triangle of the env ------------------------- */
typedef struct {
    double t;
    int32_t seg, face, amb;
    double t2, graze;
    double normal[3], bary[2], point[3];
} ray_result;

/* Near candidates (reading R24).  A ray through a shared edge or
 * vertex hits both triangles geometrically, but an FP64 edge test of the
 * rounded hit point (this file's edge functions, the GPU's FP64
 * Moller-Trumbore) can exclude either of them by rounding.  Both computations
 * start from the same FP32 inputs promoted to double; every quantity they
 * form (world vertices A v + b, the hit point o + t d, edge and cross
 * products) carries a relative error of a few tens of units of 2^-53 of the
 * largest coordinate magnitude M involved.  A plane hit whose in-plane
 * distance outside its triangle is at most
 *     nu = ORACLE_NEAR_REL * M,   M = |o|_inf + |t| |d|_inf + max_vertex |v|_inf,
 * (2^-40: ~2^8 times that rounding) is therefore a candidate hit that either
 * FP64 implementation may accept. */
#define ORACLE_NEAR_REL 9.094947017729282e-13 /* 2^-40 */

static double vmaxabs(v3 a) {
    double m = fabs(a.x);
    if (fabs(a.y) > m) m = fabs(a.y);
    if (fabs(a.z) > m) m = fabs(a.z);
    return m;
}

/* Plane hit of ray (o, d) with triangle (a, b, c): t, and whether the hit
 * point lies inside (inclusive edges) or, for 0 < t <= near_tmax only,
 * outside by at most nu (near). */
typedef struct { int parallel, inside, near; double t; } plane_hit;

static plane_hit hit_plane(v3 o, v3 d, v3 a, v3 b, v3 c, double near_tmax) {
    plane_hit h = {0, 0, 0, 0.0};
    v3 n = vcross(vsub(b, a), vsub(c, a));
    double denom = vdot(n, d);
    if (denom == 0.0) { h.parallel = 1; return h; } /* parallel ray or zero-area triangle */
    h.t = vdot(n, vsub(a, o)) / denom;
    v3 p = {o.x + h.t * d.x, o.y + h.t * d.y, o.z + h.t * d.z};
    /* edge function e_i = ((v_{i+1} - v_i) x (p - v_i)) . n = |edge_i| |n| times
     * the signed in-plane distance of p to edge i (>= 0 on the inner side) */
    double e0 = vdot(vcross(vsub(b, a), vsub(p, a)), n);
    double e1 = vdot(vcross(vsub(c, b), vsub(p, b)), n);
    double e2 = vdot(vcross(vsub(a, c), vsub(p, c)), n);
    h.inside = e0 >= 0.0 && e1 >= 0.0 && e2 >= 0.0;
    if (!h.inside && h.t > 0.0 && h.t <= near_tmax) {
        double M = vmaxabs(o) + fabs(h.t) * vmaxabs(d);
        double mv = vmaxabs(a);
        if (vmaxabs(b) > mv) mv = vmaxabs(b);
        if (vmaxabs(c) > mv) mv = vmaxabs(c);
        double nu = ORACLE_NEAR_REL * (M + mv);
        const double lim = nu * nu * vdot(n, n);
        int near = 1;
        if (e0 < 0.0) { v3 ab = vsub(b, a); near = e0 * e0 <= lim * vdot(ab, ab); }
        if (near && e1 < 0.0) { v3 bc = vsub(c, b); near = e1 * e1 <= lim * vdot(bc, bc); }
        if (near && e2 < 0.0) { v3 ca = vsub(a, c); near = e2 * e2 <= lim * vdot(ca, ca); }
        h.near = near;
    }
    return h;
}

static void cast_one(const world_mesh* w, v3 o, v3 d, double max_range,
                     double eps, int want_graze, ray_result* out, int64_t* tests) {
    double best_t = INFINITY, second_t = INFINITY, graze = INFINITY;
    int64_t best_f = -1;
    int near_zero = 0, any_near = 0;
    /* candidates within eps of max_range, kept to decide AMB_RANGE at the end */
    double range_cand = INFINITY;
    for (int64_t k = 0; k < w->n_tri; ++k) {
        /* a near candidate behind the best hit so far (+ eps) can never be
         * within eps of, or in front of, the final winner: not examined */
        plane_hit h = hit_plane(o, d, w->v[3 * k], w->v[3 * k + 1], w->v[3 * k + 2],
                                (best_t < max_range ? best_t : max_range) + eps);
        if (h.parallel) continue;
        double t = h.t;
        if (h.inside) {
            if (fabs(t) <= eps) near_zero = 1;
            if (fabs(t - max_range) <= eps && t < range_cand) range_cand = t;
            if (t > 0.0 && t <= max_range) {
                if (t < best_t || (t == best_t && k < best_f)) {
                    second_t = best_t;
                    best_t = t;
                    best_f = k;
                } else if (t < second_t) {
                    second_t = t;
                }
            }
        } else if (h.near) {
            any_near = 1;
        }
    }
    /* near candidates against the winner (second pass, only on the rare rays
     * that have one): one within eps of the winner is a tie (AMB_TIE, t2 is
     * its t); one more than eps in front of it -- or on a ray that otherwise
     * misses -- is a silhouette graze (AMB_GRAZE: hit it or pass it, t2 is
     * the nearest such t) */
    double tie_near = INFINITY, graze_near = INFINITY;
    if (any_near) {
        for (int64_t k = 0; k < w->n_tri; ++k) {
            plane_hit h = hit_plane(o, d, w->v[3 * k], w->v[3 * k + 1], w->v[3 * k + 2], max_range + eps);
            if (h.parallel || h.inside || !h.near) continue;
            if (best_f >= 0 && fabs(h.t - best_t) <= eps) {
                if (fabs(h.t - best_t) < fabs(tie_near - best_t)) tie_near = h.t;
            } else if (best_f < 0 || h.t < best_t - eps) {
                if (h.t < graze_near) graze_near = h.t;
            }
        }
    }
    *tests += w->n_tri;
    if (want_graze) {
        /* diagnostic second pass: how far outside its triangle the plane hit
         * of any triangle in front of the winner lies (metres) */
        double t_lim = best_f >= 0 ? best_t : max_range;
        for (int64_t k = 0; k < w->n_tri; ++k) {
            v3 a = w->v[3 * k], b = w->v[3 * k + 1], c = w->v[3 * k + 2];
            v3 n = vcross(vsub(b, a), vsub(c, a));
            double denom = vdot(n, d);
            if (denom == 0.0) continue;
            double t = vdot(n, vsub(a, o)) / denom;
            if (!(t > 0.0 && t <= t_lim) || k == best_f) continue;
            v3 p = {o.x + t * d.x, o.y + t * d.y, o.z + t * d.z};
            double nn = vnorm(n), out_d = 0.0, s;
            s = -vdot(vcross(vsub(b, a), vsub(p, a)), n) / (nn * vnorm(vsub(b, a))); if (s > out_d) out_d = s;
            s = -vdot(vcross(vsub(c, b), vsub(p, b)), n) / (nn * vnorm(vsub(c, b))); if (s > out_d) out_d = s;
            s = -vdot(vcross(vsub(a, c), vsub(p, c)), n) / (nn * vnorm(vsub(a, c))); if (s > out_d) out_d = s;
            if (out_d > 0.0 && out_d < graze) graze = out_d;
        }
    }
    int amb = 0;
    if (second_t - best_t <= eps) amb |= ORACLE_AMB_TIE;
    if (tie_near < INFINITY) amb |= ORACLE_AMB_TIE;
    if (graze_near < INFINITY) amb |= ORACLE_AMB_GRAZE;
    if (range_cand < INFINITY && range_cand <= best_t) amb |= ORACLE_AMB_RANGE;
    if (near_zero) amb |= ORACLE_AMB_ZERO;
    if (best_f >= 0) {
        out->t = best_t;
        out->seg = w->label[best_f];
        out->face = (int32_t)best_f;
    } else {
        out->t = max_range;
        out->seg = -1;
        out->face = -1;
    }
    out->amb = amb;
    /* the other candidate: a graze in front of the winner first (its t is
     * the alternative distance), else the closer of the second-best hit and
     * a tied near candidate (both within eps of the winner when flagged) */
    if (graze_near < INFINITY) out->t2 = graze_near;
    else out->t2 = tie_near < second_t ? tie_near : second_t;
    out->graze = graze;
    /* per-hit channels of the winning face */
    out->point[0] = o.x + out->t * d.x;
    out->point[1] = o.y + out->t * d.y;
    out->point[2] = o.z + out->t * d.z;
    if (best_f >= 0) {
        v3 a = w->v[3 * best_f], b = w->v[3 * best_f + 1], c = w->v[3 * best_f + 2];
        v3 n = vcross(vsub(b, a), vsub(c, a));
        double nn = vdot(n, n);
        double s = 1.0 / sqrt(nn);
        if (vdot(n, d) > 0.0) s = -s;
        out->normal[0] = n.x * s; out->normal[1] = n.y * s; out->normal[2] = n.z * s;
        v3 p = {out->point[0], out->point[1], out->point[2]};
        /* p = a + b1 (b - a) + b2 (c - a): cross with (c - a), resp. (b - a) */
        out->bary[0] = vdot(vcross(vsub(p, a), vsub(c, a)), n) / nn;
        out->bary[1] = vdot(vcross(vsub(b, a), vsub(p, a)), n) / nn;
    } else {
        out->normal[0] = out->normal[1] = out->normal[2] = 0.0;
        out->bary[0] = out->bary[1] = -1.0;
    }
}

/* ---- stereo shadow mask --------------------------------- */
/* "Shadows observed in stereo-camera systems are simulated by projecting
 * rays back from the points-of-intersection towards the second sensor and
 * marking pixels corresponding to the rays that intersect with the
 * environment as invalid."  Segment from the FP64 hit point p to the second
 * sensor's origin o2; invalid if any closed triangle meets it at a distance
 * in (eps, L - eps) from p (reading R21). */
static int32_t stereo_valid(const oracle_rays* r, int64_t id, const world_mesh* w,
                            const ray_result* rr, v3 o, v3 d, double amb_eps, int* amb) {
    *amb = 0;
    if (r->model == ORACLE_RAYS || rr->face < 0) return 1;
    int64_t es = r->model == ORACLE_PINHOLE ? id / ((int64_t)r->W * r->H)
                                            : id / ((int64_t)r->K * r->C);
    const float* P = r->poses + 12 * es;
    double ox = r->stereo[0], oy = r->stereo[1], oz = r->stereo[2];
    v3 o2 = {(double)P[0] * ox + (double)P[1] * oy + (double)P[2] * oz + (double)P[3],
             (double)P[4] * ox + (double)P[5] * oy + (double)P[6] * oz + (double)P[7],
             (double)P[8] * ox + (double)P[9] * oy + (double)P[10] * oz + (double)P[11]};
    v3 p = {o.x + rr->t * d.x, o.y + rr->t * d.y, o.z + rr->t * d.z};
    v3 v = vsub(o2, p);
    double L = vnorm(v);
    double eps = (double)r->stereo_eps;
    if (!(L > 2.0 * eps)) return 1;
    v3 u = {v.x / L, v.y / L, v.z / L};
    int32_t valid = 1;
    for (int64_t k = 0; k < w->n_tri; ++k) {
        v3 a = w->v[3 * k], b = w->v[3 * k + 1], c = w->v[3 * k + 2];
        v3 n = vcross(vsub(b, a), vsub(c, a));
        double denom = vdot(n, u);
        if (denom == 0.0) continue;
        double t = vdot(n, vsub(a, p)) / denom;
        v3 q = {p.x + t * u.x, p.y + t * u.y, p.z + t * u.z};
        if (vdot(vcross(vsub(b, a), vsub(q, a)), n) >= 0.0 &&
            vdot(vcross(vsub(c, b), vsub(q, b)), n) >= 0.0 &&
            vdot(vcross(vsub(a, c), vsub(q, c)), n) >= 0.0) {
            if (fabs(t - eps) <= amb_eps || fabs(t - (L - eps)) <= amb_eps) *amb = ORACLE_AMB_SHADOW;
            if (t > eps && t < L - eps) valid = 0;
        }
    }
    return valid;
}

/* ---- threading over the (env-sorted) query list ------------------------ */
typedef struct {
    const oracle_scene* sc;
    const oracle_rays* r;
    const int64_t* query;
    const int64_t* order; /* query positions sorted by env */
    int64_t lo, hi;
    double eps;
    double* t64; float* dist; int32_t* seg; int32_t* face; int32_t* amb;
    double* t2; double* graze;
    double* normal; double* bary; double* point; int32_t* valid; double* annot;
    int64_t tests;
    int status;
} job;

static void* worker(void* arg) {
    job* jb = (job*)arg;
    world_mesh w = {0, NULL, NULL, NULL, 0};
    int64_t cur_env = -1;
    jb->tests = 0;
    jb->status = 0;
    for (int64_t i = jb->lo; i < jb->hi; ++i) {
        int64_t q = jb->order[i];
        int64_t id = jb->query[q];
        int64_t e = query_env(jb->r, id);
        if (e != cur_env) {
            if (world_triangles(jb->sc, (int32_t)e, &w) != 0) { jb->status = -1; break; }
            cur_env = e;
        }
        v3 o, d;
        make_ray(jb->r, id, &o, &d);
        ray_result rr;
        cast_one(&w, o, d, (double)jb->r->max_range, jb->eps, jb->graze != NULL, &rr, &jb->tests);
        jb->t64[q] = rr.t;
        jb->dist[q] = (float)rr.t;
        jb->seg[q] = rr.seg;
        jb->face[q] = rr.face;
        jb->amb[q] = rr.amb;
        if (jb->t2) jb->t2[q] = rr.t2;
        if (jb->graze) jb->graze[q] = rr.graze;
        for (int k = 0; k < 3; ++k) {
            if (jb->normal) jb->normal[3 * q + k] = rr.normal[k];
            if (jb->point) jb->point[3 * q + k] = rr.point[k];
        }
        if (jb->bary) { jb->bary[2 * q] = rr.bary[0]; jb->bary[2 * q + 1] = rr.bary[1]; }
        if (jb->annot) {
            /* PAPER.md:228 vertex-level annotations, interpolated with the
             * winning face's barycentrics (SPEC S:550 query_annotation) */
            const int32_t K = jb->sc->annot_k;
            for (int32_t k = 0; k < K; ++k) {
                double val = NAN;
                if (rr.face >= 0) {
                    const int64_t* vi = w.vid + 3 * (int64_t)rr.face;
                    const float* A = jb->sc->annot;
                    val = (1.0 - rr.bary[0] - rr.bary[1]) * (double)A[vi[0] * K + k] +
                          rr.bary[0] * (double)A[vi[1] * K + k] + rr.bary[1] * (double)A[vi[2] * K + k];
                }
                jb->annot[(int64_t)K * q + k] = val;
            }
        }
        if (jb->valid) {
            int shadow_amb = 0;
            jb->valid[q] = stereo_valid(jb->r, id, &w, &rr, o, d, jb->eps, &shadow_amb);
            jb->amb[q] |= shadow_amb;
        }
    }
    free(w.v);
    free(w.label);
    free(w.vid);
    return NULL;
}

static int validate(const oracle_scene* sc, const oracle_rays* r) {
    if (!sc || !r || sc->n_assets < 0 || sc->n_envs < 0) return -1;
    for (int32_t a = 0; a < sc->n_assets; ++a) {
        int64_t nv = sc->vert_off[a + 1] - sc->vert_off[a];
        for (int64_t f = sc->face_off[a]; f < sc->face_off[a + 1]; ++f)
            for (int c = 0; c < 3; ++c)
                if (sc->faces[3 * f + c] < 0 || sc->faces[3 * f + c] >= nv) return -1;
    }
    int64_t n_inst = sc->env_off[sc->n_envs];
    for (int64_t j = 0; j < n_inst; ++j)
        if (sc->inst_asset[j] < 0 || sc->inst_asset[j] >= sc->n_assets) return -1;
    if (r->model == ORACLE_RAYS && r->R <= 0) return -1;
    if (r->model == ORACLE_PINHOLE && (r->W <= 0 || r->H <= 0 || r->S <= 0)) return -1;
    if (r->model == ORACLE_BEAMS && (r->C <= 0 || r->K <= 0 || r->S <= 0)) return -1;
    if (r->model < 0 || r->model > 2) return -1;
    return 0;
}

int oracle_cast(const oracle_scene* sc, const oracle_rays* r,
                const int64_t* query, int64_t n_query, double eps,
                int32_t n_threads, double* t64, float* dist, int32_t* seg,
                int32_t* face, int32_t* amb, double* t2, double* graze,
                double* normal, double* bary, double* point, int32_t* valid, double* annot) {
    if (validate(sc, r) != 0) return -1;
    if (annot && (!sc->annot || sc->annot_k <= 0)) return -1;
    int64_t n_rays_total;
    if (r->model == ORACLE_RAYS) n_rays_total = (int64_t)sc->n_envs * r->R;
    else if (r->model == ORACLE_PINHOLE) n_rays_total = (int64_t)sc->n_envs * r->S * r->H * r->W;
    else n_rays_total = (int64_t)sc->n_envs * r->S * r->C * r->K;
    for (int64_t q = 0; q < n_query; ++q)
        if (query[q] < 0 || query[q] >= n_rays_total) return -1;

    /* counting sort of query positions by env, so each env's mesh is
     * transformed once per thread */
    int64_t* count = (int64_t*)calloc((size_t)sc->n_envs + 1, sizeof(int64_t));
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_query > 0 ? n_query : 1));
    if (!count || !order) { free(count); free(order); return -1; }
    for (int64_t q = 0; q < n_query; ++q) count[query_env(r, query[q]) + 1]++;
    for (int32_t e = 0; e < sc->n_envs; ++e) count[e + 1] += count[e];
    for (int64_t q = 0; q < n_query; ++q) order[count[query_env(r, query[q])]++] = q;

    if (n_threads <= 0) n_threads = (int32_t)sysconf(_SC_NPROCESSORS_ONLN);
    if (n_threads < 1) n_threads = 1;
    if (n_threads > n_query) n_threads = (int32_t)(n_query > 0 ? n_query : 1);
    job* jobs = (job*)calloc((size_t)n_threads, sizeof(job));
    pthread_t* th = (pthread_t*)calloc((size_t)n_threads, sizeof(pthread_t));
    int status = 0;
    for (int32_t i = 0; i < n_threads; ++i) {
        job* jb = &jobs[i];
        jb->sc = sc; jb->r = r; jb->query = query; jb->order = order;
        jb->lo = n_query * i / n_threads;
        jb->hi = n_query * (i + 1) / n_threads;
        jb->eps = eps;
        jb->t64 = t64; jb->dist = dist; jb->seg = seg; jb->face = face;
        jb->amb = amb; jb->t2 = t2; jb->graze = graze;
        jb->normal = normal; jb->bary = bary; jb->point = point; jb->valid = valid; jb->annot = annot;
        if (n_threads == 1) worker(jb);
        else if (pthread_create(&th[i], NULL, worker, jb) != 0) { jb->status = -1; th[i] = 0; }
    }
    int64_t tests = 0;
    for (int32_t i = 0; i < n_threads; ++i) {
        if (n_threads > 1 && th[i]) pthread_join(th[i], NULL);
        if (jobs[i].status != 0) status = -1;
        tests += jobs[i].tests;
    }
    g_last_tests = tests;
    free(jobs); free(th); free(count); free(order);
    return status;
}

/* ---- certificate of a reported face (SURVEY.md §8(c) "Full-scale
 * certificate"): for ray id query[q] and the face reported for it, the FP64
 * plane-hit t of that face of M_{e,t}, how far (scene units)
 * the plane hit lies outside the face (<= 0: inside), and the face's label.
 * Costs one triangle per ray, so it runs on every ray of a full-size cast. */
typedef struct {
    const oracle_scene* sc;
    const oracle_rays* r;
    const int64_t* query;
    const int64_t* order;
    const int32_t* face;
    int64_t lo, hi;
    double* t_face; double* outside; int32_t* label;
    int status;
} cert_job;

static void* cert_worker(void* arg) {
    cert_job* jb = (cert_job*)arg;
    world_mesh w = {0, NULL, NULL, NULL, 0};
    int64_t cur_env = -1;
    jb->status = 0;
    for (int64_t i = jb->lo; i < jb->hi; ++i) {
        int64_t q = jb->order[i];
        int64_t id = jb->query[q];
        int32_t f = jb->face[q];
        jb->t_face[q] = NAN;
        jb->outside[q] = INFINITY;
        jb->label[q] = -1;
        if (f < 0) continue;
        int64_t e = query_env(jb->r, id);
        if (e != cur_env) {
            if (world_triangles(jb->sc, (int32_t)e, &w) != 0) { jb->status = -1; break; }
            cur_env = e;
        }
        if (f >= w.n_tri) continue;
        v3 o, d;
        make_ray(jb->r, id, &o, &d);
        v3 a = w.v[3 * f], b = w.v[3 * f + 1], c = w.v[3 * f + 2];
        v3 n = vcross(vsub(b, a), vsub(c, a));
        double denom = vdot(n, d);
        jb->label[q] = w.label[f];
        if (denom == 0.0) continue;
        double t = vdot(n, vsub(a, o)) / denom;
        v3 p = {o.x + t * d.x, o.y + t * d.y, o.z + t * d.z};
        double nn = vnorm(n), out_d = -INFINITY, s;
        s = -vdot(vcross(vsub(b, a), vsub(p, a)), n) / (nn * vnorm(vsub(b, a))); if (s > out_d) out_d = s;
        s = -vdot(vcross(vsub(c, b), vsub(p, b)), n) / (nn * vnorm(vsub(c, b))); if (s > out_d) out_d = s;
        s = -vdot(vcross(vsub(a, c), vsub(p, c)), n) / (nn * vnorm(vsub(a, c))); if (s > out_d) out_d = s;
        jb->t_face[q] = t;
        jb->outside[q] = out_d;
    }
    free(w.v);
    free(w.label);
    free(w.vid);
    return NULL;
}

int oracle_certify(const oracle_scene* sc, const oracle_rays* r, const int64_t* query,
                   int64_t n_query, const int32_t* face, int32_t n_threads,
                   double* t_face, double* outside, int32_t* label) {
    if (validate(sc, r) != 0) return -1;
    int64_t n_rays_total;
    if (r->model == ORACLE_RAYS) n_rays_total = (int64_t)sc->n_envs * r->R;
    else if (r->model == ORACLE_PINHOLE) n_rays_total = (int64_t)sc->n_envs * r->S * r->H * r->W;
    else n_rays_total = (int64_t)sc->n_envs * r->S * r->C * r->K;
    for (int64_t q = 0; q < n_query; ++q)
        if (query[q] < 0 || query[q] >= n_rays_total) return -1;
    int64_t* count = (int64_t*)calloc((size_t)sc->n_envs + 1, sizeof(int64_t));
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_query > 0 ? n_query : 1));
    if (!count || !order) { free(count); free(order); return -1; }
    for (int64_t q = 0; q < n_query; ++q) count[query_env(r, query[q]) + 1]++;
    for (int32_t e = 0; e < sc->n_envs; ++e) count[e + 1] += count[e];
    for (int64_t q = 0; q < n_query; ++q) order[count[query_env(r, query[q])]++] = q;
    if (n_threads <= 0) n_threads = (int32_t)sysconf(_SC_NPROCESSORS_ONLN);
    if (n_threads < 1) n_threads = 1;
    if (n_threads > n_query) n_threads = (int32_t)(n_query > 0 ? n_query : 1);
    cert_job* jobs = (cert_job*)calloc((size_t)n_threads, sizeof(cert_job));
    pthread_t* th = (pthread_t*)calloc((size_t)n_threads, sizeof(pthread_t));
    int status = 0;
    for (int32_t i = 0; i < n_threads; ++i) {
        cert_job* jb = &jobs[i];
        jb->sc = sc; jb->r = r; jb->query = query; jb->order = order; jb->face = face;
        jb->lo = n_query * i / n_threads;
        jb->hi = n_query * (i + 1) / n_threads;
        jb->t_face = t_face; jb->outside = outside; jb->label = label;
        if (n_threads == 1) cert_worker(jb);
        else if (pthread_create(&th[i], NULL, cert_worker, jb) != 0) { jb->status = -1; th[i] = 0; }
    }
    for (int32_t i = 0; i < n_threads; ++i) {
        if (n_threads > 1 && th[i]) pthread_join(th[i], NULL);
        if (jobs[i].status != 0) status = -1;
    }
    free(jobs); free(th); free(count); free(order);
    return status;
}
