/*
 * agr_sim.h -- kinematic env-step stand-in for the simulator around the
 * renderer (part of libagr.so, NOT part of the paper's rendering API).
 *
 * PAPER.md Table II (lines 276-304, §IV "Rendering Throughput Comparison")
 * measures the renderer "with controller-in-the-loop (to emulate practical
 * use-cases)" in "a room-like static environment consisting of 15 floating
 * obstacles": every step the robots move (physics + controller), then each
 * env's camera renders depth + segmentation.  Physics and controllers are
 * out of scope here, so this call advances a
 * kinematic stand-in on the device -- one robot per env flying towards
 * random goals under a first-order velocity controller, and optionally the
 * floating obstacles drifting (yaw rotation + vertical bobbing) -- and
 * writes the per-env sensor poses and obstacle transforms that the
 * renderer's agr_set_instance_transforms / agr_cast_pinhole calls consume.
 * It exists so that the Table-II-shaped env-step benchmark (bench.py
 * --table2) has an on-device pose update in its loop; it carries none of
 * the renderer's arithmetic.
 *
 * One launch per call, async on `stream`, no allocation and no host
 * synchronisation (capturable into a CUDA graph).  Every record is owned by
 * exactly one thread, so the step is deterministic.
 */
#ifndef AGR_SIM_H
#define AGR_SIM_H

#include <stdint.h>

#include "agr.h"

#ifdef __cplusplus
extern "C" {
#endif

/* One robot (device memory, 48 B, one per env). */
typedef struct {
    float p[3];        /* position, env frame (m)                            */
    float v[3];        /* velocity (m/s)                                     */
    float goal[3];     /* current goal position                              */
    float yaw;         /* heading about +z (rad); the body x axis is forward */
    int32_t n_goals;   /* goals drawn so far (0: draw the first one)         */
    int32_t pad;
} agr_sim_robot;

/* One obstacle instance (device memory, 80 B, one per scene instance). */
typedef struct {
    float T0[12];      /* base transform [3][4] (object -> env-local)        */
    float omega;       /* yaw rate about the instance's own position (rad/s) */
    float amp;         /* vertical bobbing amplitude (m)                     */
    float freq;        /* bobbing angular frequency (rad/s)                  */
    float angle;       /* accumulated yaw (state)                            */
    float phase;       /* accumulated bobbing phase (state)                  */
    float pad[3];
} agr_sim_obstacle;

/* Step parameters (host struct, read before return). */
typedef struct {
    float dt;             /* step (s), > 0                                   */
    float v_max;          /* speed limit of the velocity command (m/s)       */
    float tau;            /* velocity time constant (s), >= dt               */
    float yaw_rate_max;   /* heading rate limit (rad/s)                      */
    float goal_radius;    /* a goal closer than this is replaced (m)         */
    float lo[3], hi[3];   /* goal sampling box and position clamp (env frame)*/
    uint32_t seed;        /* goal stream seed (counter-based: goal k of env e
                             depends only on seed, env_base + e and k)       */
    int32_t env_base;     /* global index of env 0 (multi-GPU shards)        */
} agr_sim_params;

/*
 * Advance every robot by one step and write its sensor pose
 *   poses[e] = [Rz(yaw) | p]  (device float [n_envs][3][4]; one sensor per
 *   env, sensor frame = body frame: x forward, y left, z up)
 * and, if n_obst > 0, advance every obstacle and write
 *   obst_T[i] = [Rz(angle) A0 | b0 + (0, 0, amp sin(phase))]
 *   (device float [n_obst][3][4], the layout agr_set_instance_transforms
 *   takes; an obstacle with omega = amp = 0 keeps T0 exactly).
 * EINVAL on a NULL pointer with a positive count, n_envs < 0, n_obst < 0,
 * dt <= 0 or tau < dt.
 */
agr_status agr_sim_kinematic_step(agr_sim_robot* robots, int32_t n_envs, float* poses,
                                  agr_sim_obstacle* obst, int64_t n_obst, float* obst_T,
                                  const agr_sim_params* params, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* AGR_SIM_H */
