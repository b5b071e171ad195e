// checksum.cu -- K11: per-env order-independent 64-bit checksums of the
// output images: lets 1-GPU and n-GPU runs be
// compared bitwise without moving images between GPUs or to the host.
#include "agr_internal.cuh"

namespace agr {
namespace {

__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
    // splitmix64 finaliser
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    x ^= x >> 31;
    return x;
}

__global__ void k_checksum(const float* __restrict__ dist, const int* __restrict__ seg,
                           const int* __restrict__ face, int64_t per_env,
                           unsigned long long* sums) {
    const int e = blockIdx.x;
    const int64_t base = (int64_t)e * per_env;
    unsigned long long acc = 0;
    for (int64_t i = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; i < per_env;
         i += (int64_t)gridDim.y * blockDim.x) {
        unsigned long long h = mix64((unsigned long long)i + 0x9E3779B97F4A7C15ull);
        if (dist) h = mix64(h ^ (unsigned long long)__float_as_uint(dist[base + i]));
        if (seg) h = mix64(h ^ ((unsigned long long)(unsigned)seg[base + i] << 1));
        if (face) h = mix64(h ^ ((unsigned long long)(unsigned)face[base + i] << 2));
        acc += h;
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(sums + e, acc);
}

}  // namespace

cudaError_t checksum_launch(const float* dist, const int* seg, const int* face, int64_t per_env,
                            int n_envs, unsigned long long* sums, cudaStream_t stream) {
    cudaError_t err = cudaMemsetAsync(sums, 0, sizeof(unsigned long long) * n_envs, stream);
    if (err != cudaSuccess) return err;
    if (n_envs <= 0 || per_env <= 0) return cudaSuccess;
    int bx = (int)((per_env + 256 * 8 - 1) / (256 * 8));
    if (bx > 64) bx = 64;
    dim3 grid(n_envs, bx);
    k_checksum<<<grid, 256, 0, stream>>>(dist, seg, face, per_env, sums);
    return cudaGetLastError();
}

}  // namespace agr
