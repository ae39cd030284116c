// FP64 mma.sync shape probe: m8n8k4 against the sm_90+ shapes m16n8k4 / k8 / k16.
// One CTA per SM, W warps, C independent accumulator chains per warp, registers
// only. Prints FP64 TF/s per shape so the trailing GEMM can pick the shape with
// the best issue efficiency. SASS (cuobjdump) shows what each shape lowers to.
#include <cstdio>
#include <cuda_runtime.h>

template <int S> struct Acc { double v[S == 0 ? 2 : 4]; };

template <int S>
__device__ __forceinline__ void mma(Acc<S>& c, const double* a, const double* b) {
    if constexpr (S == 0) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c.v[0]), "+d"(c.v[1]) : "d"(a[0]), "d"(b[0]));
    } else if constexpr (S == 1) {
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+d"(c.v[0]), "+d"(c.v[1]), "+d"(c.v[2]), "+d"(c.v[3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
    } else if constexpr (S == 2) {
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+d"(c.v[0]), "+d"(c.v[1]), "+d"(c.v[2]), "+d"(c.v[3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
    } else {
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                     : "+d"(c.v[0]), "+d"(c.v[1]), "+d"(c.v[2]), "+d"(c.v[3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                       "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
}

template <int S, int C>
__global__ void probe(int iters, double* out) {
    Acc<S> acc[C];
    for (int c = 0; c < C; ++c)
        for (double& x : acc[c].v) x = 0.0;
    double a[8], b[4];
    for (int i = 0; i < 8; ++i) a[i] = 1.0 + threadIdx.x * 1e-9 + i;
    for (int i = 0; i < 4; ++i) b[i] = 0.5 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < C; ++c) mma<S>(acc[c], a, b);
    }
    double s = 0;
    for (int c = 0; c < C; ++c)
        for (double x : acc[c].v) s += x;
    if (s == 12345.678) out[0] = s;
}

template <int S, int C>
void run(int warps, int sms) {
    static const char* names[] = {"m8n8k4", "m16n8k4", "m16n8k8", "m16n8k16"};
    static const double flops[] = {512, 1024, 2048, 4096};
    double* d;
    cudaMalloc(&d, 8);
    const int iters = 16384 >> S;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    probe<S, C><<<sms, warps * 32>>>(iters, d);
    cudaEventRecord(e0);
    probe<S, C><<<sms, warps * 32>>>(iters, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-9s warps %2d chains %d: %.2f TF/s\n", names[S], warps, C,
           static_cast<double>(warps) * iters * C * sms * flops[S] / (ms * 1e-3) / 1e12);
    cudaFree(d);
}

template <int S>
void shape(int sms) {
    for (int w : {4, 8, 16}) {
        run<S, 1>(w, sms);
        run<S, 2>(w, sms);
        run<S, 4>(w, sms);
    }
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    shape<0>(sms);
    shape<1>(sms);
    shape<2>(sms);
    shape<3>(sms);
    return 0;
}
