// Replica of vf_residue_tma_kernel's consumer loop with no memory traffic:
// 12 consumer warps per CTA (one 8-row m-tile x 32 channels each), 148 CTAs,
// T tiles of SPS k-steps (4 DMMA per step), A fragments in registers, B
// fragments from shared memory at the kernel's addresses. Variants isolate what
// costs DMMA issue rate: A register array vs constant, step grouping, tile overhead.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
constexpr int kRow = 136;

template <int SP, int MODE>
__global__ void __launch_bounds__(384, 1) rep(int tiles, int steps, double* out) {
    extern __shared__ double ring[];
    for (int i = threadIdx.x; i < 40 * kRow; i += blockDim.x) ring[i] = 1e-3 * (i & 255);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, half = warp & 1;
    const int q_l = lane & 3, n_l = lane >> 2, j0 = q_l >> 1, part = q_l & 1;
    double fa[SP];
#pragma unroll
    for (int st = 0; st < SP; ++st) fa[st] = 1.0 + 1e-3 * (st + lane);
    const double* st_base = ring + (half * 32 + n_l) * 2 + part;
    const int J = 2 * steps;
    double tot = 0.0;
    for (int t = 0; t < tiles; ++t) {
        double acc[4][2];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
        if (MODE == 0) {  // per-step branch (kernel PIPE 0)
#pragma unroll
            for (int st = 0; st < SP; ++st) {
                if (st < steps) {
                    const double* b = st_base + min(2 * st + j0, J - 1) * kRow;
                    double fb[4];
#pragma unroll
                    for (int nt = 0; nt < 4; ++nt) fb[nt] = b[nt * 16];
#pragma unroll
                    for (int nt = 0; nt < 4; ++nt) dmma(acc[nt][0], acc[nt][1], fa[st], fb[nt]);
                }
            }
        } else if (MODE == 1) {  // groups of 4 steps (kernel PIPE 3)
#pragma unroll
            for (int g = 0; g < SP / 4; ++g) {
                if (g < (steps + 3) / 4) {
                    double fb[4][4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const double* b = st_base + min(2 * (4 * g + u) + j0, J - 1) * kRow;
#pragma unroll
                        for (int nt = 0; nt < 4; ++nt) fb[u][nt] = b[nt * 16];
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int nt = 0; nt < 4; ++nt) dmma(acc[nt][0], acc[nt][1], fa[4 * g + u], fb[u][nt]);
                }
            }
        } else if (MODE == 2) {  // compile-time step count, no branches at all
#pragma unroll
            for (int st = 0; st < 20; ++st) {
                const double* b = st_base + (2 * st + j0) * kRow;
                double fb[4];
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) fb[nt] = b[nt * 16];
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) dmma(acc[nt][0], acc[nt][1], fa[st], fb[nt]);
            }
        } else {  // MODE 3: registers only (no LDS), compile-time 20 steps
#pragma unroll
            for (int st = 0; st < 20; ++st)
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) dmma(acc[nt][0], acc[nt][1], fa[st], fa[(st + nt + 1) % SP]);
        }
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) tot += acc[nt][0] - acc[nt][1];
    }
    if (tot == 1.2345e-300) out[0] = tot;
}

template <int SP, int MODE>
void run(int warps, int sms, int tiles) {
    double* d;
    cudaMalloc(&d, 8);
    const size_t smem = 40 * kRow * sizeof(double);
    cudaFuncSetAttribute(rep<SP, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    rep<SP, MODE><<<sms, warps * 32, smem>>>(tiles, 20, d);
    cudaEventRecord(e0);
    rep<SP, MODE><<<sms, warps * 32, smem>>>(tiles, 20, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double dm = (double)warps * tiles * 80;
    const double ideal_us = dm * 16 / 4 / 1.965e3;
    printf("mode %d warps %2d: %.1f us (ideal %.1f at 1.965 GHz) -> %.1f%%\n", MODE, warps, ms * 1e3, ideal_us,
           100 * ideal_us / (ms * 1e3));
    cudaFree(d);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int w : {8, 12}) {
        run<24, 0>(w, sms, 32);
        run<24, 1>(w, sms, 32);
        run<24, 2>(w, sms, 32);
        run<24, 3>(w, sms, 32);
        run<24, 2>(w, sms, 320);
    }
    return 0;
}
