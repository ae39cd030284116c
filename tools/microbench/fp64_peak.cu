// FP64 throughput microbenchmark on sm_100a: DFMA pipe vs legacy DMMA (mma.sync f64).
// Used once to pin the FP64 roofline denominator (MEASURED_FP64.json).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, a2 = a0 + 2e-9, a3 = a0 + 3e-9;
  double a4 = a0 + 4e-9, a5 = a0 + 5e-9, a6 = a0 + 6e-9, a7 = a0 + 7e-9;
  const double b = 0.999999, c = 1e-12;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void dmma_m8n8k4_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[u][0]), "+d"(c[u][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0; for (int u = 0; u < 8; ++u) s += c[u][0] + c[u][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma_m16n8k16_kernel(double* out, int iters) {
  double a[8], b[4];
  for (int q = 0; q < 8; ++q) a[q] = (threadIdx.x + q) * 1e-3;
  for (int q = 0; q < 4; ++q) b[q] = 1.0 + (threadIdx.x + q) * 1e-4;
  double c[4][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[u][0]), "+d"(c[u][1]), "+d"(c[u][2]), "+d"(c[u][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0; for (int u = 0; u < 4; ++u) s += c[u][0] + c[u][1] + c[u][2] + c[u][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("{\"gpu\": \"%s\", \"sms\": %d", p.name, p.multiProcessorCount);
  double* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = p.multiProcessorCount * 8, threads = 256;
  for (int kind = 0; kind < 3; ++kind) {
    int iters = kind == 0 ? 4096 : 4096;
    double best = 1e30;
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(e0);
      if (kind == 0) dfma_kernel<<<blocks, threads>>>(out, iters);
      else if (kind == 1) dmma_m8n8k4_kernel<<<blocks, threads>>>(out, iters);
      else dmma_m16n8k16_kernel<<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (rep > 0 && ms < best) best = ms;
    }
    double flops;
    if (kind == 0) flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    else if (kind == 1) flops = 2.0 * 8 * 8 * 4 * 8 * (double)iters * blocks * (threads / 32);
    else flops = 2.0 * 16 * 8 * 16 * 4 * (double)iters * blocks * (threads / 32);
    const char* nm[3] = {"dfma", "dmma_m8n8k4", "dmma_m16n8k16"};
    printf(", \"%s_tflops\": %.3f", nm[kind], flops / (best * 1e-3) / 1e12);
  }
  printf(", \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
