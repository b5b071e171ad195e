// fma_peak.cu -- issue-rate microbenchmark behind the "alu" roofline peak
// of bench.py: 148 SMs x 128 lanes x SM clock thread-
// instructions per second.  Times long dependent-chain-free loops of FP32
// FFMA (FMA pipe) and FMNMX (ALU pipe) instructions, 8 independent chains
// per thread, a few blocks per SM, CUDA events; prints one JSON object.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fma_peak tools/fma_peak.cu
#include <cuda_runtime.h>
#include <cstdio>

constexpr int ITERS = 1 << 14;

__global__ void k_ffma(float* out, float a, float b) {
    float x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3f + k;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fmaf(x[k], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 1234.5f) out[threadIdx.x] = s;
}

__global__ void k_fmnmx(float* out, float a, float b) {
    float x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3f + k;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fminf(fmaxf(x[k], a), b);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 1234.5f) out[threadIdx.x] = s;
}

template <class K>
double rate(K kern, int sms, int& clk_khz) {
    float* out;
    cudaMalloc(&out, 4096);
    const int threads = 256, blocks = sms * 8;
    kern<<<blocks, threads>>>(out, 0.999f, 0.001f);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        kern<<<blocks, threads>>>(out, 0.999f, 0.001f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    cudaFree(out);
    // one FFMA / FMNMX pair counts as one / two instructions per chain step
    return (double)blocks * threads * ITERS * 8 / (best * 1e-3);
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    int dummy = 0;
    double ffma = rate(k_ffma, p.multiProcessorCount, dummy);
    double mnmx = 2.0 * rate(k_fmnmx, p.multiProcessorCount, dummy);
    double peak = (double)p.multiProcessorCount * 128 * clk * 1e3;
    printf("{\"gpu\": \"%s\", \"sms\": %d, \"max_clock_mhz\": %.0f, "
           "\"ffma_thread_inst_per_s\": %.4e, \"fmnmx_thread_inst_per_s\": %.4e, "
           "\"model_peak_at_max_clock\": %.4e, \"ffma_frac_of_model\": %.4f, \"fmnmx_frac_of_model\": %.4f}\n",
           p.name, p.multiProcessorCount, clk / 1e3, ffma, mnmx, peak, ffma / peak, mnmx / peak);
    return 0;
}
