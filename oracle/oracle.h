/*
 * oracle.h -- CPU brute-force ray-casting ORACLE (test infrastructure only).
 *
 * THIS IS TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load or call it.  The
 * product path (paper_2503_01471_b200/, libagr.so) never links, imports or
 * executes anything under oracle/, and this file shares no code, header,
 * table or constant with it.
 *
 * What it computes (the plain definition):
 *   For environment e the scene is the merged mesh M_{e,t} = T_{e,t} o M^base_e
 *   ("The vertices of the mesh are transformed to match the obstacles in the
 *   simulator at time t", §III.D.1).  Every instance j of env e
 *   is an asset mesh whose vertices are mapped x_env = A_j x + b_j (DESIGN.md
 *   reading R1) in FP64 from the FP32 inputs.  "Individual rays are cast
 *   outwards per-pixel to evaluate intersection with M_{i,t}":
 *   for every ray the result is the smallest t with 0 < t <= max_range such
 *   that o + t d lies on a closed, double-sided triangle of the env; equal t
 *   goes to the lowest per-env face index.  The distance reported is "range
 *   for ToF sensors and LiDARs" and "the distance of this point from the image
 *   plane ... as depth": depth rays use the unnormalised
 *   direction d_s = (1, -x', -y') so t is the depth; range rays use the unit
 *   direction so t is the Euclidean range.  Misses report max_range, seg -1,
 *   face -1 (readings R4, R5).
 *
 * Every ray is tested against every triangle of its env (no acceleration
 * structure), in double precision.  The ray/triangle test is a plane
 * intersection followed by an inclusive edge-function inside test; it is
 * deliberately a different formula from the GPU's Moller-Trumbore test.
 */
#ifndef AGR_ORACLE_H
#define AGR_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Scene description (all host memory, borrowed for the duration of a call). */
typedef struct {
    int32_t n_assets;
    const float*   verts;      /* all assets' vertices, [sum V][3]            */
    const int64_t* vert_off;   /* [n_assets+1] CSR into verts (in vertices)   */
    const int32_t* faces;      /* all assets' faces, [sum F][3], asset-local  */
    const int64_t* face_off;   /* [n_assets+1] CSR into faces (in faces)      */
    int32_t n_envs;
    const int64_t* env_off;    /* [n_envs+1] CSR of instances per env         */
    const int32_t* inst_asset; /* [n_inst]                                    */
    const int32_t* inst_label; /* [n_inst]                                    */
    const float*   inst_T;     /* [n_inst][3][4] row-major: x' = A x + b      */
    /* optional per-vertex annotations ("embed vertex-level
     * annotations that can be queried"): [sum V][annot_k], indexed like
     * verts; NaN rows = asset without annotations.  NULL / 0 = none.        */
    const float*   annot;
    int32_t        annot_k;
} oracle_scene;

/* Ray models. */
enum { ORACLE_RAYS = 0, ORACLE_PINHOLE = 1, ORACLE_BEAMS = 2 };
enum { ORACLE_DEPTH = 0, ORACLE_RANGE = 1 };

typedef struct {
    int32_t model;        /* ORACLE_RAYS / ORACLE_PINHOLE / ORACLE_BEAMS      */
    /* ORACLE_RAYS: orig, dir [n_envs][R][3] env-local, t in units of |dir|.  */
    const float* orig;
    const float* dir;
    int32_t R;
    /* ORACLE_PINHOLE: W, H, fx, fy, cx, cy, kind; poses [n_envs][S][3][4].   */
    int32_t W, H;
    float fx, fy, cx, cy;
    int32_t kind;
    /* ORACLE_BEAMS: beam table [C][K][3] (sensor frame), poses.             */
    const float* beams;
    int32_t C, K;
    const float* poses;   /* [n_envs][S][3][4] sensor -> env                 */
    int32_t S;
    float max_range;
    /* stereo shadow mask: second sensor origin in the sensor
     * frame and the self-hit guard (metres); used when `valid` is requested */
    float stereo[3];
    float stereo_eps;
} oracle_rays;

/* Ambiguity bits (SURVEY.md §8(c) parity rules; reading R24). */
enum {
    ORACLE_AMB_TIE   = 1, /* best and second-best candidate t within amb_eps, or a
                             near candidate (a plane hit outside its triangle by
                             at most nu = 2^-40 M, the FP64 rounding band of
                             hit_plane()) within amb_eps of the best t
                             (shared edges / vertices)                       */
    ORACLE_AMB_RANGE = 2, /* a candidate within amb_eps of max_range         */
    ORACLE_AMB_ZERO  = 4, /* a candidate within amb_eps of t = 0             */
    ORACLE_AMB_SHADOW = 8, /* a shadow-segment candidate within amb_eps of eps
                             or of L - eps                                   */
    ORACLE_AMB_GRAZE = 16 /* a near candidate more than amb_eps in front of the
                             best hit, or on a ray that otherwise misses: a
                             silhouette graze within FP64 rounding (hit it or
                             pass it; t2 = its t)                            */
};

/*
 * Cast the rays named by `query` (flat ray ids: for RAYS  id = e*R + r; for
 * PINHOLE id = ((e*S + s)*H + v)*W + u; for BEAMS id = ((e*S + s)*C + c)*K + k).
 * Per query it writes:
 *   t64[q]   the winning t in double (max_range on a miss)
 *   dist[q]  (float)t64[q]
 *   seg[q]   instance label or -1;  face[q] per-env face index or -1
 *   amb[q]   ORACLE_AMB_* bits computed with tolerance amb_eps (metres)
 *   t2[q]    the other candidate: on an AMB_GRAZE ray the nearest grazing
 *            near candidate's t; otherwise the second-best hit t or a tied
 *            near candidate's t, whichever is closer (within amb_eps of
 *            t64 when AMB_TIE is set; R24); +inf if none [may be NULL]
 *   graze[q] smallest distance (scene units) by which the plane hit of a
 *            triangle closer than the winner lies outside that triangle
 *            (diagnostic for silhouette rays; +inf if none)     [may be NULL]
 *   normal[3q..] unit geometric normal of the winning face, oriented so
 *            that n . d < 0 (towards the ray origin); 0 on a miss [may be NULL]
 *   bary[2q..] (b1, b2) with hit = (1-b1-b2) v0 + b1 v1 + b2 v2 over the
 *            face's vertices, from the plane hit point by cross-product
 *            area ratios; -1 on a miss                          [may be NULL]
 *   point[3q..] o + t d (t = the reported distance)             [may be NULL]
 *   annot[K q..] barycentric interpolation (1-b1-b2) A(v0) + b1 A(v1) +
 *            b2 A(v2) of the winning face's vertex annotations (scene
 *            annot, K = annot_k); NaN on a miss              [may be NULL]
 *   valid[q] stereo shadow mask: 0 if the segment from the hit point p to
 *            the second sensor o2 = P (stereo) hits a triangle at a distance
 *            in (eps, |o2 - p| - eps) from p, else 1 (1 on a miss; PINHOLE
 *            and BEAMS only)                                    [may be NULL]
 * (PAPER.md:218 surface normals; :228 "barycentric coordinates of
 * intersecting rays", "point clouds and surface normals".)
 * n_threads <= 0 uses all online cores.  Returns 0, or -1 on bad input.
 */
int oracle_cast(const oracle_scene* scene, const oracle_rays* rays,
                const int64_t* query, int64_t n_query, double amb_eps,
                int32_t n_threads,
                double* t64, float* dist, int32_t* seg, int32_t* face,
                int32_t* amb, double* t2, double* graze,
                double* normal, double* bary, double* point, int32_t* valid,
                double* annot);

/*
 * Certificate of a reported face (SURVEY.md §8(c) "Full-scale certificate",
 * one triangle per ray, so it covers every ray of a full-size cast): for ray
 * query[q] and face[q] (per-env face index, -1 = miss), writes
 *   t_face[q]  FP64 plane-hit t of that face (NaN on a miss or when the ray
 *              is parallel to the face's plane)
 *   outside[q] how far (scene units) that plane hit lies outside the face:
 *              max over the three edges of the signed distance, <= 0 inside
 *              (+inf on a miss)
 *   label[q]   label of the face's instance (-1 on a miss)
 * It proves the hit is real and its distance right; optimality (no closer
 * face) is oracle_cast's job on samples.  Returns 0, or -1 on bad input.
 */
int oracle_certify(const oracle_scene* scene, const oracle_rays* rays,
                   const int64_t* query, int64_t n_query, const int32_t* face,
                   int32_t n_threads, double* t_face, double* outside, int32_t* label);

/* Number of triangle tests the last oracle_cast call performed (for the
 * cpu_baseline report: ray-triangle tests/s). */
int64_t oracle_last_tests(void);

#ifdef __cplusplus
}
#endif
#endif
