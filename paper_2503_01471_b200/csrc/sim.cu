// sim.cu -- kinematic env-step stand-in for the simulator around the
// renderer (include/agr_sim.h): robots flying to random goals under a
// first-order velocity controller, floating obstacles drifting.  It only
// produces the per-step sensor poses and instance transforms that the
// Table-II-shaped env-step benchmark ("controller-in-the-
// loop") feeds to the renderer; none of the renderer's arithmetic is here.
#include "../../include/agr_sim.h"

#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <string>

namespace {

__device__ __forceinline__ unsigned long long sim_mix64(unsigned long long x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}

// Uniform in [0, 1) from (seed, env, goal k, axis): counter-based, so goal
// k of env e does not depend on the launch shape or on the GPU count.
__device__ __forceinline__ float sim_uniform(uint32_t seed, int64_t env, int k, int axis) {
    unsigned long long h = sim_mix64(((unsigned long long)seed << 32) ^ (unsigned long long)env);
    h = sim_mix64(h ^ ((unsigned long long)(uint32_t)k << 2 | (unsigned long long)axis));
    return (float)(h >> 40) * (1.0f / 16777216.0f);
}

__global__ void k_sim_step(agr_sim_robot* __restrict__ robots, int n_envs, float* __restrict__ poses,
                           agr_sim_obstacle* __restrict__ obst, int64_t n_obst, float* __restrict__ obst_T,
                           agr_sim_params P) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n_envs) {
        agr_sim_robot r = robots[i];
        float dx = r.goal[0] - r.p[0], dy = r.goal[1] - r.p[1], dz = r.goal[2] - r.p[2];
        if (r.n_goals == 0 || dx * dx + dy * dy + dz * dz < P.goal_radius * P.goal_radius) {
            for (int a = 0; a < 3; ++a)
                r.goal[a] = P.lo[a] + (P.hi[a] - P.lo[a]) * sim_uniform(P.seed, P.env_base + i, r.n_goals, a);
            r.n_goals += 1;
            dx = r.goal[0] - r.p[0];
            dy = r.goal[1] - r.p[1];
            dz = r.goal[2] - r.p[2];
        }
        // velocity command towards the goal (gain 1/s), speed-limited
        const float n = sqrtf(dx * dx + dy * dy + dz * dz);
        const float s = n > P.v_max ? P.v_max / n : 1.0f;
        const float a = P.dt / P.tau;
        const float cmd[3] = {dx * s, dy * s, dz * s};
        for (int k = 0; k < 3; ++k) {
            r.v[k] += (cmd[k] - r.v[k]) * a;
            r.p[k] = fminf(fmaxf(r.p[k] + r.v[k] * P.dt, P.lo[k]), P.hi[k]);
        }
        // heading towards the goal, rate-limited
        if (dx * dx + dy * dy > 1e-6f) {
            float d = atan2f(dy, dx) - r.yaw;
            d = d - 6.2831853f * rintf(d * 0.15915494f);
            const float m = P.yaw_rate_max * P.dt;
            r.yaw += fminf(fmaxf(d, -m), m);
            r.yaw = r.yaw - 6.2831853f * rintf(r.yaw * 0.15915494f);
        }
        robots[i] = r;
        float c, sn;
        sincosf(r.yaw, &sn, &c);
        float* o = poses + 12 * i;
        o[0] = c;  o[1] = -sn; o[2] = 0.0f;  o[3] = r.p[0];
        o[4] = sn; o[5] = c;   o[6] = 0.0f;  o[7] = r.p[1];
        o[8] = 0.0f; o[9] = 0.0f; o[10] = 1.0f; o[11] = r.p[2];
    }
    if (i < n_obst) {
        agr_sim_obstacle b = obst[i];
        float* o = obst_T + 12 * i;
        if (b.omega == 0.0f && b.amp == 0.0f) {
            for (int k = 0; k < 12; ++k) o[k] = b.T0[k];
            return;
        }
        b.angle += b.omega * P.dt;
        b.phase += b.freq * P.dt;
        b.angle -= 6.2831853f * rintf(b.angle * 0.15915494f);
        b.phase -= 6.2831853f * rintf(b.phase * 0.15915494f);
        obst[i].angle = b.angle;
        obst[i].phase = b.phase;
        float c, sn;
        sincosf(b.angle, &sn, &c);
        // rows of Rz(angle) A0
        for (int col = 0; col < 3; ++col) {
            const float a0 = b.T0[0 + col], a1 = b.T0[4 + col], a2 = b.T0[8 + col];
            o[0 + col] = c * a0 - sn * a1;
            o[4 + col] = sn * a0 + c * a1;
            o[8 + col] = a2;
        }
        o[3] = b.T0[3];
        o[7] = b.T0[7];
        o[11] = b.T0[11] + b.amp * sinf(b.phase);
    }
}

}  // namespace

// error reporting shares agr_last_error's thread-local message (abi.cu)
namespace agr {
agr_status set_error(agr_status s, const char* msg);
}

extern "C" agr_status agr_sim_kinematic_step(agr_sim_robot* robots, int32_t n_envs, float* poses,
                                             agr_sim_obstacle* obst, int64_t n_obst, float* obst_T,
                                             const agr_sim_params* params, void* stream) {
    if (!params) return agr::set_error(AGR_EINVAL, "params is NULL");
    if (n_envs < 0 || n_obst < 0) return agr::set_error(AGR_EINVAL, "negative count");
    if (n_envs > 0 && (!robots || !poses)) return agr::set_error(AGR_EINVAL, "robots / poses is NULL");
    if (n_obst > 0 && (!obst || !obst_T)) return agr::set_error(AGR_EINVAL, "obst / obst_T is NULL");
    if (!(params->dt > 0.0f) || !(params->tau >= params->dt))
        return agr::set_error(AGR_EINVAL, "need dt > 0 and tau >= dt");
    const int64_t n = n_envs > n_obst ? (int64_t)n_envs : n_obst;
    if (n == 0) return agr::set_error(AGR_OK, "");
    const int threads = 128;
    k_sim_step<<<(unsigned)((n + threads - 1) / threads), threads, 0, (cudaStream_t)stream>>>(
        robots, n_envs, poses, obst, n_obst, obst_T, *params);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return agr::set_error(AGR_ECUDA, cudaGetErrorString(e));
    return agr::set_error(AGR_OK, "");
}
