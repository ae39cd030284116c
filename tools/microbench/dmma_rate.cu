// DMMA (mma.sync.m8n8k4.f64) issue-rate probe: one CTA per SM, W warps, each
// warp running C independent accumulator chains for N iterations (registers
// only), plus an optional LDS.64 per DMMA from shared memory. Prints DMMA per
// clock per SM for each (W, C, lds) so kernels can be sized against it.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int C, int LDS>
__global__ void probe(int iters, double* out) {
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1e-3 * i;
    __syncthreads();
    double acc[C][2];
    for (int c = 0; c < C; ++c) acc[c][0] = acc[c][1] = 0.0;
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
    const int lane = threadIdx.x & 31;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            double bb = b;
            if (LDS) bb = sm[(lane * 2 + c * 64 + it) & 1023];
            dmma(acc[c][0], acc[c][1], a, bb);
        }
    }
    double s = 0;
    for (int c = 0; c < C; ++c) s += acc[c][0] + acc[c][1];
    if (s == 12345.678) out[0] = s;
}

template <int C, int LDS>
void run(int warps, int sms) {
    double* d;
    cudaMalloc(&d, 8);
    const int iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    probe<C, LDS><<<sms, warps * 32>>>(iters, d);
    cudaEventRecord(e0);
    probe<C, LDS><<<sms, warps * 32>>>(iters, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double dmmas_per_sm = static_cast<double>(warps) * iters * C;
    const double cycles = ms * 1e-3 * clk * 1e3;
    printf("warps %2d chains %2d lds %d: %.3f DMMA/clk/SM (%.1f TF/s)\n", warps, C, LDS, dmmas_per_sm / cycles,
           dmmas_per_sm * sms * 512 / (ms * 1e-3) / 1e12);
    cudaFree(d);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int w : {4, 8, 12, 16, 24, 32}) {
        run<1, 0>(w, sms);
        run<2, 0>(w, sms);
        run<4, 0>(w, sms);
        run<8, 0>(w, sms);
        run<4, 1>(w, sms);
    }
    return 0;
}
