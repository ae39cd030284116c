// Right-looking blocked complex LU with partial pivoting, batched over
// independent frequency systems, for sm_100a (FP64).
//
// The reference has no BEM/LU; this is the solve inside the new
// FrequencySystem::evaluate (systems.hpp:34-42). Per 64-column panel:
//   panel                16-wide sub-panels (lu_panel_cluster_kernel: the rows
//                        of one matrix across a thread-block cluster, pivot
//                        candidates exchanged through distributed shared
//                        memory, one cluster barrier per column; LAPACK izamax
//                        rule, first max wins), lu_sub_swap_trsm_kernel and
//                        lu_window_update_kernel between sub-panels;
//                        lu_panel_kernel (global slots + atomic barrier) when a
//                        matrix needs more than 16 CTAs.
//   swap + TRSM          lu_l11_inverse_kernel (L11^{-1} and the panel's swaps
//                        as one gather map) + lu_swap_apply_kernel (32-column
//                        strips: gather, then L11^{-1} X on DMMA).
//   trailing update      lu_gemm3m_tma_kernel (default): A22 -= L21 U12 as a
//                        complex GEMM on the FP64 tensor pipe with three real
//                        mma.sync.m8n8k4.f64 products per complex MAC (3M),
//                        64x32 tiles, operand sum planes from lu_g3_prep_kernel,
//                        TMA-fed double buffer refilled by the last warp out;
//                        lu_gemm_tma_kernel (FDSWEEP_GEMM=4m): four products,
//                        64x64 tiles.
// Batches go two panels at a time (super_panel_step): one rank-128 trailing
// update per 128 columns, interchanges in LAPACK order inside the super-panel.
// Single matrices use a look-ahead schedule (the next panel on a side stream).
// Across panels / super-panels the row swaps are LINPACK-style (earlier L
// columns are not permuted); lu_solve follows the same interchange groups.
#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>

#include <climits>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>
#include <cstdlib>
#include <string>

#include "lu.cuh"

namespace fdsb {

namespace {

constexpr int kPanelThreads = 256;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void group_barrier(unsigned* ctr, unsigned target) {
    fds_jitter(target);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1u);
        while (ld_acquire(ctr) < target) __nanosleep(20);
    }
    __syncthreads();
}

}  // namespace

template <int NB>
__global__ void __launch_bounds__(kPanelThreads)
lu_panel_kernel(double* A, size_t mstride, size_t plane, int n, int ld, int batch, int k, int w,
                int P, int R, int G, int* ipiv, int* info, double* slots, unsigned* counters) {
    // One thread per panel row (R <= kPanelThreads): a thread owns its row in
    // shared memory for all w columns, so scaling / rank-1 updates need no
    // intra-CTA synchronisation; only the pivot choice crosses threads / CTAs.
    extern __shared__ double sm[];
    double* tre = sm;             // [NB][R]
    double* tim = tre + NB * R;   // [NB][R]
    double* urow = tim + NB * R;  // [2NB] pivot row (new row c)
    double* drow = urow + 2 * NB; // [2NB] old row c (moves to the pivot row)
    __shared__ double red_v[kPanelThreads / 32];
    __shared__ int red_i[kPanelThreads / 32];
    __shared__ int s_lrow, s_piv;
    __shared__ double s_best;

    const int g = blockIdx.x / P, p = blockIdx.x % P;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    unsigned* ctr = counters + g;
    unsigned step = 0;
    const size_t sstride = 2 + 2 * NB;
    double* gslots = slots + static_cast<size_t>(g) * 2 * (P + 1) * sstride;
    // compact (value, row) keys of the P candidates per parity, after all groups' rows
    double2* gkeys = reinterpret_cast<double2*>(slots + static_cast<size_t>(G) * 2 * (P + 1) * sstride) +
                     static_cast<size_t>(g) * 2 * P;

    for (int b = g; b < batch; b += G) {
        double* Are = A + static_cast<size_t>(b) * mstride;
        double* Aim = Are + plane;
        const int r0 = k + p * R;
        const int r1 = min(r0 + R, n);
        const int nr = max(0, r1 - r0);
        const int myrow = r0 + tid;
        const bool own = tid < nr;
        if (own)
            for (int j = 0; j < w; ++j) {
                const size_t gi = static_cast<size_t>(k + j) * ld + myrow;
                tre[j * R + tid] = Are[gi];
                tim[j * R + tid] = Aim[gi];
            }
        for (int j = 0; j < w; ++j) {
            const int c = k + j;
            // (a) CTA-local argmax of |re|+|im| (LAPACK izamax: first maximum)
            double best = -1.0;
            int bi = INT_MAX;
            if (own && myrow >= c) {
                best = fabs(tre[j * R + tid]) + fabs(tim[j * R + tid]);
                bi = myrow;
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, best, off);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
                if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
            }
            if (lane == 0) { red_v[wid] = best; red_i[wid] = bi; }
            __syncthreads();
            const int par = step & 1;
            double* myslot = gslots + (static_cast<size_t>(par) * (P + 1) + p) * sstride;
            double* dslot = gslots + (static_cast<size_t>(par) * (P + 1) + P) * sstride;
            if (wid == 0) {
                double v = lane < kPanelThreads / 32 ? red_v[lane] : -1.0;
                int ri = lane < kPanelThreads / 32 ? red_i[lane] : INT_MAX;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    const double ov = __shfl_xor_sync(0xffffffffu, v, off);
                    const int oi = __shfl_xor_sync(0xffffffffu, ri, off);
                    if (ov > v || (ov == v && oi < ri)) { v = ov; ri = oi; }
                }
                if (lane == 0) {
                    gkeys[par * P + p] = make_double2(v, static_cast<double>(ri));
                    s_lrow = ri;
                }
                __syncwarp();
                const int lr = s_lrow;
                if (lr != INT_MAX)
                    for (int jj = lane; jj < 2 * NB; jj += 32) {
                        const int col = jj % NB;
                        myslot[2 + jj] = col < w ? (jj < NB ? tre[col * R + lr - r0] : tim[col * R + lr - r0]) : 0.0;
                    }
            } else if (wid == 1 && c >= r0 && c < r1) {
                for (int jj = lane; jj < 2 * NB; jj += 32) {
                    const int col = jj % NB;
                    dslot[2 + jj] = col < w ? (jj < NB ? tre[col * R + c - r0] : tim[col * R + c - r0]) : 0.0;
                }
            }
            ++step;
            group_barrier(ctr, step * static_cast<unsigned>(P));
            // (b) winner among the P candidates; stage pivot row + old row c
            if (wid == 0) {
                double bv = -1.0;
                int bidx = INT_MAX, bw = 0;
                for (int q = lane; q < P; q += 32) {
                    const double2 kv = __ldcg(&gkeys[par * P + q]);
                    const int ri = static_cast<int>(kv.y);
                    if (kv.x > bv || (kv.x == bv && ri < bidx)) { bv = kv.x; bidx = ri; bw = q; }
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
                    const int oi = __shfl_xor_sync(0xffffffffu, bidx, off);
                    const int ow = __shfl_xor_sync(0xffffffffu, bw, off);
                    if (ov > bv || (ov == bv && oi < bidx)) { bv = ov; bidx = oi; bw = ow; }
                }
                const double* ws = gslots + (static_cast<size_t>(par) * (P + 1) + bw) * sstride;
                for (int jj = lane; jj < 2 * NB; jj += 32) {
                    urow[jj] = __ldcg(ws + 2 + jj);
                    drow[jj] = __ldcg(dslot + 2 + jj);
                }
                if (lane == 0) {
                    s_piv = bidx;
                    s_best = bv;
                    if (p == 0) {
                        ipiv[static_cast<size_t>(b) * n + c] = bidx;
                        if (!(bv > 0.0) && info[b] == 0) info[b] = c + 1;
                    }
                }
            }
            __syncthreads();
            // (c) swap, scale, rank-1 update of the own row
            const int piv = s_piv;
            if (own) {
                if (myrow == c && piv != c) {
                    for (int jj = 0; jj < w; ++jj) { tre[jj * R + tid] = urow[jj]; tim[jj * R + tid] = urow[NB + jj]; }
                } else if (myrow == piv && piv != c) {
                    for (int jj = 0; jj < w; ++jj) { tre[jj * R + tid] = drow[jj]; tim[jj * R + tid] = drow[NB + jj]; }
                }
                if (myrow > c) {
                    const cplx u = mk(urow[j], urow[NB + j]);
                    if (u.re != 0.0 || u.im != 0.0) {
                        const cplx l = mk(tre[j * R + tid], tim[j * R + tid]) * crecip(u);
                        tre[j * R + tid] = l.re;
                        tim[j * R + tid] = l.im;
                        for (int jj = j + 1; jj < w; ++jj) {
                            const double ur = urow[jj], ui = urow[NB + jj];
                            tre[jj * R + tid] -= l.re * ur - l.im * ui;
                            tim[jj * R + tid] -= l.re * ui + l.im * ur;
                        }
                    }
                }
            }
        }
        if (own)
            for (int j = 0; j < w; ++j) {
                const size_t gi = static_cast<size_t>(k + j) * ld + myrow;
                Are[gi] = tre[j * R + tid];
                Aim[gi] = tim[j * R + tid];
            }
        __syncthreads();
    }
}

// Cluster variant for batches of moderate N: the P CTAs of one matrix form a
// thread-block cluster, so the per-column pivot exchange runs through
// distributed shared memory — every CTA publishes its candidate (|a|, row, row
// values) in its own smem, one hardware cluster barrier, then each CTA reads
// the P keys and the winning row straight from the peers' smem (mapa /
// ld.shared::cluster) instead of a global-memory slot + atomic-counter barrier.
// Candidate slots are double-buffered by column parity, so a single barrier per
// column suffices (a slot is rewritten two columns later, after every CTA has
// passed the intervening barrier).
template <int NB>
__global__ void __launch_bounds__(kPanelThreads)
lu_panel_cluster_kernel(double* A, size_t mstride, size_t plane, int n, int ld, int batch, int k, int w, int R,
                        int G, int* ipiv, int* info) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ double sm[];
    double* tre = sm;             // [NB][R]
    double* tim = tre + NB * R;   // [NB][R]
    double* urow = tim + NB * R;  // [2NB] pivot row (new row c)
    double* drow = urow + 2 * NB; // [2NB] old row c (moves to the pivot row)
    // published per parity: [0] |a|, [1] row, [2 .. 2+2NB) candidate row, [2+2NB .. 2+4NB) old row c
    __shared__ double pub[2][2 + 4 * NB];
    __shared__ double red_v[kPanelThreads / 32];
    __shared__ int red_i[kPanelThreads / 32];
    __shared__ int s_piv;
    __shared__ double s_best;

    const int P = static_cast<int>(cluster.num_blocks());
    const int p = static_cast<int>(cluster.block_rank());
    const int g = blockIdx.x / P;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    unsigned step = 0;
    for (int b = g; b < batch; b += G) {
        double* Are = A + static_cast<size_t>(b) * mstride;
        double* Aim = Are + plane;
        const int r0 = k + p * R;
        const int r1 = min(r0 + R, n);
        const int nr = max(0, r1 - r0);
        const int myrow = r0 + tid;
        const bool own = tid < nr;
        if (own)
            for (int j = 0; j < w; ++j) {
                const size_t gi = static_cast<size_t>(k + j) * ld + myrow;
                tre[j * R + tid] = Are[gi];
                tim[j * R + tid] = Aim[gi];
            }
        for (int j = 0; j < w; ++j) {
            const int c = k + j;
            const int par = step & 1;
            double best = -1.0;
            int bi = INT_MAX;
            if (own && myrow >= c) {
                best = fabs(tre[j * R + tid]) + fabs(tim[j * R + tid]);
                bi = myrow;
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, best, off);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
                if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
            }
            if (lane == 0) { red_v[wid] = best; red_i[wid] = bi; }
            __syncthreads();
            if (wid == 0) {
                double v = lane < kPanelThreads / 32 ? red_v[lane] : -1.0;
                int ri = lane < kPanelThreads / 32 ? red_i[lane] : INT_MAX;
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    const double ov = __shfl_xor_sync(0xffffffffu, v, off);
                    const int oi = __shfl_xor_sync(0xffffffffu, ri, off);
                    if (ov > v || (ov == v && oi < ri)) { v = ov; ri = oi; }
                }
                if (lane == 0) {
                    pub[par][0] = v;
                    pub[par][1] = static_cast<double>(ri);
                }
                if (ri != INT_MAX)
                    for (int jj = lane; jj < 2 * NB; jj += 32) {
                        const int col = jj % NB;
                        pub[par][2 + jj] = col < w ? (jj < NB ? tre[col * R + ri - r0] : tim[col * R + ri - r0]) : 0.0;
                    }
            } else if (wid == 1 && c >= r0 && c < r1) {
                for (int jj = lane; jj < 2 * NB; jj += 32) {
                    const int col = jj % NB;
                    pub[par][2 + 2 * NB + jj] = col < w ? (jj < NB ? tre[col * R + c - r0] : tim[col * R + c - r0]) : 0.0;
                }
            }
            ++step;
            fds_jitter(step);
            cluster.sync();
            // winner among the P candidates (peers' smem), pivot row + old row c
            if (wid == 0) {
                double bv = -1.0;
                int bidx = INT_MAX, bw = 0;
                for (int q = lane; q < P; q += 32) {
                    const double* rp = cluster.map_shared_rank(&pub[par][0], q);
                    const double kv = rp[0];
                    const int ri = static_cast<int>(rp[1]);
                    if (kv > bv || (kv == bv && ri < bidx)) { bv = kv; bidx = ri; bw = q; }
                }
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
                    const int oi = __shfl_xor_sync(0xffffffffu, bidx, off);
                    const int ow = __shfl_xor_sync(0xffffffffu, bw, off);
                    if (ov > bv || (ov == bv && oi < bidx)) { bv = ov; bidx = oi; bw = ow; }
                }
                const int owner = (c - k) / R;  // CTA holding row c
                const double* wp = cluster.map_shared_rank(&pub[par][2], bw);
                const double* op = cluster.map_shared_rank(&pub[par][2 + 2 * NB], owner);
                for (int jj = lane; jj < 2 * NB; jj += 32) {
                    urow[jj] = wp[jj];
                    drow[jj] = op[jj];
                }
                if (lane == 0) {
                    s_piv = bidx;
                    s_best = bv;
                    if (p == 0) {
                        ipiv[static_cast<size_t>(b) * n + c] = bidx;
                        if (!(bv > 0.0) && info[b] == 0) info[b] = c + 1;
                    }
                }
            }
            __syncthreads();
            const int piv = s_piv;
            if (own) {
                if (myrow == c && piv != c) {
                    for (int jj = 0; jj < w; ++jj) { tre[jj * R + tid] = urow[jj]; tim[jj * R + tid] = urow[NB + jj]; }
                } else if (myrow == piv && piv != c) {
                    for (int jj = 0; jj < w; ++jj) { tre[jj * R + tid] = drow[jj]; tim[jj * R + tid] = drow[NB + jj]; }
                }
                if (myrow > c) {
                    const cplx u = mk(urow[j], urow[NB + j]);
                    if (u.re != 0.0 || u.im != 0.0) {
                        const cplx l = mk(tre[j * R + tid], tim[j * R + tid]) * crecip(u);
                        tre[j * R + tid] = l.re;
                        tim[j * R + tid] = l.im;
                        for (int jj = j + 1; jj < w; ++jj) {
                            const double ur = urow[jj], ui = urow[NB + jj];
                            tre[jj * R + tid] -= l.re * ur - l.im * ui;
                            tim[jj * R + tid] -= l.re * ui + l.im * ur;
                        }
                    }
                }
            }
        }
        if (own)
            for (int j = 0; j < w; ++j) {
                const size_t gi = static_cast<size_t>(k + j) * ld + myrow;
                Are[gi] = tre[j * R + tid];
                Aim[gi] = tim[j * R + tid];
            }
        __syncthreads();
    }
    cluster.sync();  // peers may still read this CTA's published slots
}

// ------------------------------------------------------------------ swaps + TRSM
constexpr int kTrsmCols = 128;
constexpr int kTrsmThreads = 512;

template <int NB>
__global__ void __launch_bounds__(kTrsmThreads)
lu_swap_trsm_kernel(double* A, size_t mstride, size_t plane, int n, int ld, int k, int w,
                    const int* ipiv) {
    extern __shared__ double sm[];
    double* Lre = sm;                    // [NB][NB], L[j*NB+i]
    double* Lim = Lre + NB * NB;
    double* Xre = Lim + NB * NB;         // [kTrsmCols][NB], X[t*NB+i]
    double* Xim = Xre + kTrsmCols * NB;
    const int b = blockIdx.y;
    double* Are = A + static_cast<size_t>(b) * mstride;
    double* Aim = Are + plane;
    const int col0 = k + w + blockIdx.x * kTrsmCols;
    const int ncols = min(kTrsmCols, n - col0);
    const int tid = threadIdx.x;
    for (int idx = tid; idx < w * w; idx += blockDim.x) {
        const int j = idx / w, i = idx % w;
        const size_t gi = static_cast<size_t>(k + j) * ld + k + i;
        Lre[j * NB + i] = Are[gi];
        Lim[j * NB + i] = Aim[gi];
    }
    for (int idx = tid; idx < ncols * w; idx += blockDim.x) {
        const int t = idx / w, i = idx % w;
        const size_t gi = static_cast<size_t>(col0 + t) * ld + k + i;
        Xre[t * NB + i] = Are[gi];
        Xim[t * NB + i] = Aim[gi];
    }
    __syncthreads();
    if (tid < ncols) {
        const size_t colbase = static_cast<size_t>(col0 + tid) * ld;
        const int* pv = ipiv + static_cast<size_t>(b) * n;
        for (int c = k; c < k + w; ++c) {
            const int r = pv[c];
            if (r == c) continue;
            const int lc = c - k;
            if (r < k + w) {
                const int lr = r - k;
                double t0 = Xre[tid * NB + lc], t1 = Xim[tid * NB + lc];
                Xre[tid * NB + lc] = Xre[tid * NB + lr];
                Xim[tid * NB + lc] = Xim[tid * NB + lr];
                Xre[tid * NB + lr] = t0;
                Xim[tid * NB + lr] = t1;
            } else {
                const double gr = Are[colbase + r], gi = Aim[colbase + r];
                Are[colbase + r] = Xre[tid * NB + lc];
                Aim[colbase + r] = Xim[tid * NB + lc];
                Xre[tid * NB + lc] = gr;
                Xim[tid * NB + lc] = gi;
            }
        }
    }
    __syncthreads();
    for (int j = 0; j < w - 1; ++j) {
        const int rows = w - j - 1;
        for (int idx = tid; idx < ncols * rows; idx += blockDim.x) {
            const int t = idx / rows, i = j + 1 + idx % rows;
            const double lr = Lre[j * NB + i], li = Lim[j * NB + i];
            const double xr = Xre[t * NB + j], xi = Xim[t * NB + j];
            Xre[t * NB + i] -= lr * xr - li * xi;
            Xim[t * NB + i] -= lr * xi + li * xr;
        }
        __syncthreads();
    }
    for (int idx = tid; idx < ncols * w; idx += blockDim.x) {
        const int t = idx / w, i = idx % w;
        const size_t gi = static_cast<size_t>(col0 + t) * ld + k + i;
        Are[gi] = Xre[t * NB + i];
        Aim[gi] = Xim[t * NB + i];
    }
}

// ------------------------------------------------------------------ DMMA GEMM
constexpr int GBM = 64, GBN = 64, GBK = 16, GSTAGES = 2;
constexpr int kG3W = 256;      // deepest trailing update (256-column super-panels)
constexpr int kG3Rows = kG3W + 8;  // U12 sum-plane column length: update depth + TMA over-read
constexpr int GAS = GBM + 4;  // A tile row stride (doubles) ≡ 4 (mod 16): conflict-free fragments
constexpr int GBS = GBK + 4;  // B tile row stride
constexpr int kGemmThreads = 256;
constexpr int GWM = 2, GWN = 4;                      // warp grid over the 64x64 tile
constexpr int GMI = GBM / GWM / 8, GNI = GBN / GWN / 8;  // 8x8 DMMA tiles per warp
constexpr int kGemmSmemDoubles = GSTAGES * 2 * (GBK * GAS + GBN * GBS);

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(kGemmThreads, 2)
lu_gemm_kernel(double* A, size_t mstride, size_t plane, int n, int ld, int k, int w, int c0, int c1) {
    extern __shared__ __align__(16) double gsm[];
    const int b = blockIdx.z;
    double* Are = A + static_cast<size_t>(b) * mstride;
    double* Aim = Are + plane;
    const int m0 = k + w + blockIdx.x * GBM;  // first row of this tile
    const int n0 = c0 + blockIdx.y * GBN;  // first column (c0 >= k + w)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp % GWM, wn = warp / GWM;
    auto As = [&](int st, int pl) { return gsm + (st * 2 + pl) * (GBK * GAS); };
    auto Bs = [&](int st, int pl) { return gsm + GSTAGES * 2 * (GBK * GAS) + (st * 2 + pl) * (GBN * GBS); };

    auto load_stage = [&](int st, int kc) {
        const int kk0 = kc * GBK;
        // A tile: L21[m0..m0+64)[k+kk0 .. +16): per (plane, kk) 64 contiguous doubles = 32 chunks
        for (int q = tid; q < 2 * GBK * (GBM / 2); q += kGemmThreads) {
            const int pl = q / (GBK * (GBM / 2));
            const int rem = q % (GBK * (GBM / 2));
            const int kk = rem / (GBM / 2), ch = rem % (GBM / 2);
            const double* src = (pl ? Aim : Are) + static_cast<size_t>(k + kk0 + kk) * ld + m0 + 2 * ch;
            const int bytes = (kk0 + kk < w && m0 + 2 * ch < ld) ? 16 : 0;  // rows past ld: sub-panel windows
            cp_async16(As(st, pl) + kk * GAS + 2 * ch, bytes ? src : Are, bytes);
        }
        // B tile: U12[k+kk0 .. +16)[n0..n0+64): per (plane, column) 16 contiguous doubles = 8 chunks
        for (int q = tid; q < 2 * GBN * (GBK / 2); q += kGemmThreads) {
            const int pl = q / (GBN * (GBK / 2));
            const int rem = q % (GBN * (GBK / 2));
            const int nn = rem / (GBK / 2), ch = rem % (GBK / 2);
            const int kk = kk0 + 2 * ch;
            const double* src = (pl ? Aim : Are) + static_cast<size_t>(n0 + nn) * ld + k + kk;
            const int bytes = n0 + nn >= c1 ? 0 : (kk + 2 <= w ? 16 : (kk < w ? 8 : 0));  // window [c0, c1)
            cp_async16(Bs(st, pl) + nn * GBS + 2 * ch, bytes ? src : Are, bytes);
        }
    };

    const int nk = (w + GBK - 1) / GBK;
    load_stage(0, 0);
    cp_async_commit();
    // Accumulators start from C (loads overlap the first A/B stage); the
    // mainloop subtracts L21 U12 and the epilogue is a plain store.
    double acr[GMI][GNI][2], aci[GMI][GNI][2];
#pragma unroll
    for (int mi = 0; mi < GMI; ++mi) {
        const int row = m0 + wm * (GBM / GWM) + mi * 8 + (lane >> 2);
#pragma unroll
        for (int ni = 0; ni < GNI; ++ni)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = n0 + wn * (GBN / GWN) + ni * 8 + 2 * (lane & 3) + e;
                const size_t gi = static_cast<size_t>(col) * ld + row;
                // column window [c0, c1) (sub-panel updates stop at the panel edge); rows of a
                // sub-panel window's last tile can pass n (and ld): never read past the matrix
                const bool in = col < c1 && row < n;
                acr[mi][ni][e] = in ? Are[gi] : 0.0;
                aci[mi][ni][e] = in ? Aim[gi] : 0.0;
            }
    }
    for (int kc = 0; kc < nk; ++kc) {
        if (kc + 1 < nk) load_stage((kc + 1) % GSTAGES, kc + 1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        const int st = kc % GSTAGES;
        const double* ar = As(st, 0);
        const double* ai = As(st, 1);
        const double* br = Bs(st, 0);
        const double* bi = Bs(st, 1);
#pragma unroll
        for (int k4 = 0; k4 < GBK; k4 += 4) {
            double na_r[GMI], fa_i[GMI], na_i[GMI], fb_r[GNI], fb_i[GNI];
            const int kr = k4 + (lane & 3);
#pragma unroll
            for (int mi = 0; mi < GMI; ++mi) {
                const int m = wm * (GBM / GWM) + mi * 8 + (lane >> 2);
                na_r[mi] = -ar[kr * GAS + m];
                fa_i[mi] = ai[kr * GAS + m];
                na_i[mi] = -fa_i[mi];
            }
#pragma unroll
            for (int ni = 0; ni < GNI; ++ni) {
                const int nn = wn * (GBN / GWN) + ni * 8 + (lane >> 2);
                fb_r[ni] = br[nn * GBS + kr];
                fb_i[ni] = bi[nn * GBS + kr];
            }
            // C - (ar + i ai)(br + i bi): two passes over the 16 tiles so that the
            // two products accumulated into one register pair are 32 DMMAs apart.
#pragma unroll
            for (int mi = 0; mi < GMI; ++mi)
#pragma unroll
                for (int ni = 0; ni < GNI; ++ni) {
                    dmma(acr[mi][ni][0], acr[mi][ni][1], na_r[mi], fb_r[ni]);
                    dmma(aci[mi][ni][0], aci[mi][ni][1], na_r[mi], fb_i[ni]);
                }
#pragma unroll
            for (int mi = 0; mi < GMI; ++mi)
#pragma unroll
                for (int ni = 0; ni < GNI; ++ni) {
                    dmma(acr[mi][ni][0], acr[mi][ni][1], fa_i[mi], fb_i[ni]);
                    dmma(aci[mi][ni][0], aci[mi][ni][1], na_i[mi], fb_r[ni]);
                }
        }
        __syncthreads();
    }
    // epilogue: store C - L21 U12
#pragma unroll
    for (int mi = 0; mi < GMI; ++mi) {
        const int row = m0 + wm * (GBM / GWM) + mi * 8 + (lane >> 2);
#pragma unroll
        for (int ni = 0; ni < GNI; ++ni) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = n0 + wn * (GBN / GWN) + ni * 8 + 2 * (lane & 3) + e;
                if (row < n && col < c1) {
                    const size_t gi = static_cast<size_t>(col) * ld + row;
                    Are[gi] = acr[mi][ni][e];
                    Aim[gi] = aci[mi][ni][e];
                }
            }
        }
    }
}

// ------------------------------------------------------------------ TMA-fed trailing GEMM
// Same tile, warp layout and DMMA schedule as lu_gemm_kernel, for full 64-wide
// panels: one thread issues cp.async.bulk.tensor loads of the L21 / U12 k-chunks
// (both planes) into the double buffer and the CTA waits on an mbarrier with
// the transaction byte count. The TMA boxes over-read 4 rows (A: 68 x 16) and
// 4 k-rows (B: 20 x 64) so that the dense box lands in exactly the padded,
// bank-conflict-free layouts of the cp.async kernel (strides 68 and 20).
constexpr int kTmaABox0 = GAS, kTmaBBox0 = GBS;
constexpr unsigned kTmaStageBytes = 2u * (GBK * GAS + GBN * GBS) * sizeof(double);
constexpr size_t kTmaSmemPad = 128 + GSTAGES * sizeof(uint64_t);

template <int W>
__global__ void __launch_bounds__(kGemmThreads, 2)
lu_gemm_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, double* A,
                   size_t mstride, size_t plane, int n, int ld, int k, int c0) {
    // TMA destinations need 128 B alignment: round the dynamic base up (the
    // launch requests kTmaSmemPad extra bytes); the mbarriers sit after the tiles
    extern __shared__ double gsm_raw[];
    const unsigned raw = static_cast<unsigned>(__cvta_generic_to_shared(gsm_raw));
    double* gsm = gsm_raw + ((128u - (raw & 127u)) & 127u) / sizeof(double);
    uint64_t* bar = reinterpret_cast<uint64_t*>(gsm + kGemmSmemDoubles);
    constexpr int w = W, nk = w / GBK;
    const int b = blockIdx.z;
    double* Are = A + static_cast<size_t>(b) * mstride;
    double* Aim = Are + plane;
    const int m0 = k + w + blockIdx.x * GBM;
    const int n0 = c0 + blockIdx.y * GBN;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp % GWM, wn = warp / GWM;
    auto As = [&](int st, int pl) { return gsm + (st * 2 + pl) * (GBK * GAS); };
    auto Bs = [&](int st, int pl) { return gsm + GSTAGES * 2 * (GBK * GAS) + (st * 2 + pl) * (GBN * GBS); };
    if (tid == 0) {
#pragma unroll
        for (int st = 0; st < GSTAGES; ++st) mbar_init(&bar[st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int st, int kc) {  // thread 0 only
        mbar_expect_tx(&bar[st], kTmaStageBytes);
#pragma unroll
        for (int pl = 0; pl < 2; ++pl) {
            tma_load_3d(As(st, pl), &tmA, &bar[st], m0, k + kc * GBK, 2 * b + pl);
            tma_load_3d(Bs(st, pl), &tmB, &bar[st], k + kc * GBK, n0, 2 * b + pl);
        }
    };
    if (tid == 0) issue(0, 0);
    double acr[GMI][GNI][2], aci[GMI][GNI][2];
#pragma unroll
    for (int mi = 0; mi < GMI; ++mi) {
        const int row = m0 + wm * (GBM / GWM) + mi * 8 + (lane >> 2);
#pragma unroll
        for (int ni = 0; ni < GNI; ++ni)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = n0 + wn * (GBN / GWN) + ni * 8 + 2 * (lane & 3) + e;
                const size_t gi = static_cast<size_t>(col) * ld + row;
                acr[mi][ni][e] = Are[gi];
                aci[mi][ni][e] = Aim[gi];
            }
    }
#pragma unroll 1
    for (int kc = 0; kc < nk; ++kc) {
        if (tid == 0 && kc + 1 < nk) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // prior generic reads of the slot
            issue((kc + 1) % GSTAGES, kc + 1);
        }
        const int st = kc % GSTAGES;
        mbar_wait(&bar[st], (kc / GSTAGES) & 1);
        const double* ar = As(st, 0);
        const double* ai = As(st, 1);
        const double* br = Bs(st, 0);
        const double* bi = Bs(st, 1);
#pragma unroll
        for (int k4 = 0; k4 < GBK; k4 += 4) {
            double na_r[GMI], fa_i[GMI], na_i[GMI], fb_r[GNI], fb_i[GNI];
            const int kr = k4 + (lane & 3);
#pragma unroll
            for (int mi = 0; mi < GMI; ++mi) {
                const int m = wm * (GBM / GWM) + mi * 8 + (lane >> 2);
                na_r[mi] = -ar[kr * GAS + m];
                fa_i[mi] = ai[kr * GAS + m];
                na_i[mi] = -fa_i[mi];
            }
#pragma unroll
            for (int ni = 0; ni < GNI; ++ni) {
                const int nn = wn * (GBN / GWN) + ni * 8 + (lane >> 2);
                fb_r[ni] = br[nn * GBS + kr];
                fb_i[ni] = bi[nn * GBS + kr];
            }
#pragma unroll
            for (int mi = 0; mi < GMI; ++mi)
#pragma unroll
                for (int ni = 0; ni < GNI; ++ni) {
                    dmma(acr[mi][ni][0], acr[mi][ni][1], na_r[mi], fb_r[ni]);
                    dmma(aci[mi][ni][0], aci[mi][ni][1], na_r[mi], fb_i[ni]);
                }
#pragma unroll
            for (int mi = 0; mi < GMI; ++mi)
#pragma unroll
                for (int ni = 0; ni < GNI; ++ni) {
                    dmma(acr[mi][ni][0], acr[mi][ni][1], fa_i[mi], fb_i[ni]);
                    dmma(aci[mi][ni][0], aci[mi][ni][1], na_i[mi], fb_r[ni]);
                }
        }
        __syncthreads();
    }
#pragma unroll
    for (int mi = 0; mi < GMI; ++mi) {
        const int row = m0 + wm * (GBM / GWM) + mi * 8 + (lane >> 2);
#pragma unroll
        for (int ni = 0; ni < GNI; ++ni) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = n0 + wn * (GBN / GWN) + ni * 8 + 2 * (lane & 3) + e;
                if (row < n && col < n) {
                    const size_t gi = static_cast<size_t>(col) * ld + row;
                    Are[gi] = acr[mi][ni][e];
                    Aim[gi] = aci[mi][ni][e];
                }
            }
        }
    }
}

// ------------------------------------------------------------------ 3M (three real products) trailing GEMM
// The same update with three real DMMA products per complex MAC instead of four:
//   t1 = Ar (Br + Bi),  t2 = (Ar + Ai) Bi,  t3 = (Ai - Ar) Br
//   Re(A B) = t1 - t2,  Im(A B) = t1 + t3
// so C - A B = (Cre + t2 - t1, Cim - t3 - t1): accumulators Q = Cre (preloaded)
// += t2, R = Cim (preloaded) -= t3 and P = t1 from zero, stored as Q - P, R - P.
// The operand sums come pre-formed from lu_g3_prep_kernel (three TMA planes
// per operand); in-register sums stalled the DMMA stream (shared FP64 pipe). Three accumulators per output need 1.5x the registers of the
// four-product kernel, so the tile is BN = 32 columns wide with 16x16 warp
// tiles (2 CTAs/SM) — or 64 wide at 1 CTA/SM. Error: normwise like ZGEMM
// (Higham, "Stability of a method for multiplying complex matrices with three
// real matrix multiplications"), componentwise slightly weaker in Im.
template <int BN, int KC = GBK, int NS = GSTAGES>
constexpr int g3_smem_doubles() { return NS * 3 * (KC * GAS + BN * (KC + 4)); }

// Operand planes of one trailing update, formed once per (panel, matrix) so the
// GEMM's inner loop is DMMA-only (FP64 adds there contend with DMMA for the
// same pipe): L21 planes Re+Im, Re-Im at [b][p][kk][m] (absolute row m, panel
// column kk, ld rows per column), U12 plane Re+Im at [b][c][kk] (kG3Rows per column).
// Grid: x = [L column blocks (one per panel column kk, lblocks = w or 0 when the
// L planes are current)] + [U blocks striding over (column, k-pair)], y = matrix.
// 16-byte accesses throughout (k, w, ld and kG3Rows are even), no divisions.
__global__ void __launch_bounds__(256) lu_g3_prep_kernel(const double* __restrict__ A, size_t mstride, size_t plane,
                                                         int n, int ld, int k, int w, int c0, int c1,
                                                         double* __restrict__ g3, int lblocks) {
    const int b = blockIdx.y;
    const double* Are = A + static_cast<size_t>(b) * mstride;
    const double* Aim = Are + plane;
    if (static_cast<int>(blockIdx.x) < lblocks) {
        const int kk = blockIdx.x;
        double* L = g3 + static_cast<size_t>(b) * 2 * kG3W * ld;
        const double2* xr = reinterpret_cast<const double2*>(Are + static_cast<size_t>(k + kk) * ld);
        const double2* xi = reinterpret_cast<const double2*>(Aim + static_cast<size_t>(k + kk) * ld);
        double2* ls = reinterpret_cast<double2*>(L + static_cast<size_t>(kk) * ld);
        double2* ld2 = reinterpret_cast<double2*>(L + static_cast<size_t>(kG3W + kk) * ld);
        for (int m2 = (k + w) / 2 + threadIdx.x; 2 * m2 < n; m2 += blockDim.x) {
            const double2 x = xr[m2], y = xi[m2];
            ls[m2] = make_double2(x.x + y.x, x.y + y.y);
            ld2[m2] = make_double2(x.x - y.x, x.y - y.y);
        }
        return;
    }
    double* U = g3 + static_cast<size_t>(gridDim.y) * 2 * kG3W * ld + static_cast<size_t>(b) * ld * kG3Rows;
    const int sh = __ffs(w) - 2;  // log2(w / 2): w is 64, 128 or 256
    const int total = (c1 - c0) << sh;
    const int nub = gridDim.x - lblocks;
    for (int idx = (blockIdx.x - lblocks) * blockDim.x + threadIdx.x; idx < total; idx += nub * blockDim.x) {
        const int c = c0 + (idx >> sh), k2 = idx & ((1 << sh) - 1);
        const size_t gi = static_cast<size_t>(c) * ld + k + 2 * k2;
        const double2 x = *reinterpret_cast<const double2*>(Are + gi);
        const double2 y = *reinterpret_cast<const double2*>(Aim + gi);
        *reinterpret_cast<double2*>(U + static_cast<size_t>(c) * kG3Rows + 2 * k2) = make_double2(x.x + y.x, x.y + y.y);
    }
}

// Fragment mapping: a lane's two row fragments are rows 2j, 2j+1 of its warp's
// 16 (j = lane / 4), so A fragments arrive by one 16-byte LDS and the C tile
// moves in 16-byte accesses (a store instruction writes whole 128-byte lines).
// (Measured: 16-byte B fragments through a permuted k order inside the chunk,
// 8 instead of 12 shared loads per pass and chunk, gave no gain.)
template <int W, int BN, int WGM, int MINB, int NT = kGemmThreads, int PFIRST = 0, int KC = GBK, int NS = GSTAGES>
__global__ void __launch_bounds__(NT, MINB)
lu_gemm3m_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmL, const __grid_constant__ CUtensorMap tmU, double* A,
                     size_t mstride, size_t plane, int n, int ld, int k, int c0, int band) {
    constexpr int WGN = (NT / 32) / WGM;
    constexpr int MI = GBM / WGM / 8, NI = BN / WGN / 8;
    static_assert(MI == 2, "row-pair fragments");
    // KC-deep k-chunks in an NS-stage ring (measured: KC = 8 with 4 or 5 stages,
    // more latency slack but twice the per-chunk hand-offs, 6.5-9 % slower)
    constexpr int AS = GAS, BS = KC + 4;  // KC + 4: conflict-free 8-byte B fragments for KC = 8, 16
    constexpr int nk = W / KC;
    constexpr unsigned kStageBytes = 3u * (KC * AS + BN * BS) * sizeof(double);
    extern __shared__ double gsm_raw[];
    const unsigned raw = static_cast<unsigned>(__cvta_generic_to_shared(gsm_raw));
    double* gsm = gsm_raw + ((128u - (raw & 127u)) & 127u) / sizeof(double);
    uint64_t* bar = reinterpret_cast<uint64_t*>(gsm + g3_smem_doubles<BN, KC, NS>());
    unsigned* freed = reinterpret_cast<unsigned*>(bar + NS);  // per stage: warps done with it
    const int b = blockIdx.z;
    double* Are = A + static_cast<size_t>(b) * mstride;
    double* Aim = Are + plane;
    // Tile order: launch order runs down the rows of one column block (x fastest);
    // with band > 0 it runs through bands of `band` row tiles across every
    // column block, so a band's L21 rows stay in L2 while the U12 column blocks
    // stream (a 128-deep L21 panel of N = 36864 is 113 MB, beyond the L2).
    int tx = blockIdx.x, ty = blockIdx.y;
    if (band > 0) {
        const int ntx = gridDim.x, nty = gridDim.y;
        const int lin = blockIdx.x + ntx * blockIdx.y;
        const int bi = lin / (band * nty);
        const int b0 = bi * band;
        const int hb = min(band, ntx - b0);
        const int rem = lin - bi * band * nty;
        ty = rem / hb;
        tx = b0 + rem % hb;
    }
    const int m0 = k + W + tx * GBM;
    const int n0 = c0 + ty * BN;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp % WGM, wn = warp / WGM;
    const int r0 = wm * (GBM / WGM) + 2 * (lane >> 2);  // this lane's row pair in the tile
    // A planes: Re L21, Re+Im, Re-Im; B planes: Re U12, Im U12, Re+Im
    auto As = [&](int st, int pl) { return gsm + (st * 3 + pl) * (KC * AS); };
    auto Bs = [&](int st, int pl) { return gsm + NS * 3 * (KC * AS) + (st * 3 + pl) * (BN * BS); };
    if (tid == 0) {
#pragma unroll
        for (int st = 0; st < NS; ++st) {
            mbar_init(&bar[st], 1);
            freed[st] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int st, int kc) {  // thread 0 only
        mbar_expect_tx(&bar[st], kStageBytes);
        tma_load_3d(As(st, 0), &tmA, &bar[st], m0, k + kc * KC, 2 * b);
        tma_load_3d(As(st, 1), &tmL, &bar[st], m0, kc * KC, 2 * b);
        tma_load_3d(As(st, 2), &tmL, &bar[st], m0, kc * KC, 2 * b + 1);
        tma_load_3d(Bs(st, 0), &tmB, &bar[st], k + kc * KC, n0, 2 * b);
        tma_load_3d(Bs(st, 1), &tmB, &bar[st], k + kc * KC, n0, 2 * b + 1);
        tma_load_3d(Bs(st, 2), &tmU, &bar[st], kc * KC, n0, b);
    };
    if (tid == 0)
        for (int st = 0; st < NS && st < nk; ++st) issue(st, st);
    double q[MI][NI][2], r[MI][NI][2], p[MI][NI][2];
#pragma unroll
    for (int ni = 0; ni < NI; ++ni)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int col = n0 + wn * (BN / WGN) + ni * 8 + 2 * (lane & 3) + e;
            const size_t gi = static_cast<size_t>(col) * ld + m0 + r0;  // even: 16-byte aligned
            const double2 cr = *reinterpret_cast<const double2*>(Are + gi);
            const double2 ci = *reinterpret_cast<const double2*>(Aim + gi);
            q[0][ni][e] = cr.x;
            q[1][ni][e] = cr.y;
            r[0][ni][e] = ci.x;
            r[1][ni][e] = ci.y;
            p[0][ni][e] = 0.0;
            p[1][ni][e] = 0.0;
        }
    // passes [p0, p1) of chunk kc (P: Re A x (Re+Im) B, Q: (Re+Im) A x Im B,
    // R: (Re-Im) A x Re B), each holding only its own fragments
    auto compute = [&](int st, int p0, int p1) {
        const double* ar = As(st, 0);
        const double* as = As(st, 1);
        const double* ad = As(st, 2);
        const double* br = Bs(st, 0);
        const double* bi = Bs(st, 1);
        const double* bs = Bs(st, 2);
        const int qk = lane & 3;
#pragma unroll
        for (int k8 = 0; k8 < KC; k8 += 8) {
#pragma unroll
            for (int pass = 0; pass < 3; ++pass) {
                if (pass < p0 || pass >= p1) continue;
                const double* pa = pass == 0 ? ar : (pass == 1 ? as : ad);
                const double* pb = pass == 0 ? bs : (pass == 1 ? bi : br);
                double(&acc)[MI][NI][2] = pass == 0 ? p : (pass == 1 ? q : r);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int kr = k8 + 4 * h + qk;
                    const double2 fa = *reinterpret_cast<const double2*>(pa + kr * AS + r0);
                    double fb[NI];
#pragma unroll
                    for (int ni = 0; ni < NI; ++ni) fb[ni] = pb[(wn * (BN / WGN) + ni * 8 + (lane >> 2)) * BS + kr];
#pragma unroll
                    for (int ni = 0; ni < NI; ++ni) {
                        dmma(acc[0][ni][0], acc[0][ni][1], fa.x, fb[ni]);
                        dmma(acc[1][ni][0], acc[1][ni][1], fa.y, fb[ni]);
                    }
                }
            }
        }
    };
    // P-first prologue (PFIRST chunks): the C-independent product runs while the
    // C tile loads into the Q / R accumulators are still in flight
#pragma unroll 1
    for (int kc = 0; kc < PFIRST && kc < nk; ++kc) {
        mbar_wait(&bar[kc % NS], (kc / NS) & 1);
        compute(kc % NS, 0, 1);
    }
    // No CTA barrier per k-chunk: each warp's lane 0 counts itself out of a stage
    // once its fragment loads have been consumed, and the last warp out refills the
    // stage with chunk kc + NS (fast warps never wait for slow ones).
#pragma unroll 1
    for (int kc = 0; kc < nk; ++kc) {
        const int st = kc % NS;
        if (kc < PFIRST) {
            compute(st, 1, 3);
        } else {
            mbar_wait(&bar[st], (kc / NS) & 1);
            compute(st, 0, 3);
        }
        fds_jitter(kc);
        if (kc + NS < nk) {
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                const unsigned old = atomicAdd(&freed[st], 1u);
                if (old % (NT / 32) == NT / 32 - 1) {
                    __threadfence_block();
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    issue(st, kc + NS);
                }
            }
        }
    }
    const int row = m0 + r0;
#pragma unroll
    for (int ni = 0; ni < NI; ++ni)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int col = n0 + wn * (BN / WGN) + ni * 8 + 2 * (lane & 3) + e;
            if (col >= n) continue;
            const size_t gi = static_cast<size_t>(col) * ld + row;
            if (row + 1 < n) {
                *reinterpret_cast<double2*>(Are + gi) = make_double2(q[0][ni][e] - p[0][ni][e], q[1][ni][e] - p[1][ni][e]);
                *reinterpret_cast<double2*>(Aim + gi) = make_double2(r[0][ni][e] - p[0][ni][e], r[1][ni][e] - p[1][ni][e]);
            } else if (row < n) {
                Are[gi] = q[0][ni][e] - p[0][ni][e];
                Aim[gi] = r[0][ni][e] - p[0][ni][e];
            }
        }
}

// ------------------------------------------------------------------ TRSM via L11^{-1} (DMMA)
// U12 = L11^{-1} P A12: per panel and matrix, lu_l11_inverse_kernel forms the
// unit-lower 64x64 inverse and resolves the panel's 64 sequential row swaps
// into one gather (source row of every panel row and of every outside row a
// pivot names); lu_swap_apply_kernel then permutes each 32-column strip with
// independent loads and multiplies by L11^{-1} on the FP64 tensor pipe.
constexpr size_t kLinvStride = 2 * 64 * 64 + 128;  // doubles per matrix: Linv planes + swap map (ints)
constexpr int kInvThreads = 256;

// Sources are "virtual" indices into V = [panel rows k..k+63, erow[0..next)]:
// v < 64 is panel row k + v, v >= 64 is outside row erow[v - 64].
struct SwapMap {  // lives in the int tail of a matrix's kLinvStride record
    int psrc[64];     // source (virtual) of panel row k + c
    int next;         // outside rows touched
    int erow[64];     // those rows
    int esrc[64];     // and their sources (virtual)
};
static_assert(sizeof(SwapMap) <= 128 * sizeof(double), "swap map record");

__global__ void __launch_bounds__(kInvThreads)
lu_l11_inverse_kernel(const double* A, size_t mstride, size_t plane, int n, int ld, int k, const int* ipiv,
                      double* linv) {
    extern __shared__ double ism[];
    double (*lre)[65] = reinterpret_cast<double (*)[65]>(ism);             // L[i][m]
    double (*lim)[65] = reinterpret_cast<double (*)[65]>(ism + 64 * 65);
    double (*xre)[65] = reinterpret_cast<double (*)[65]>(ism + 2 * 64 * 65);  // published rows of X = L^{-1}
    double (*xim)[65] = reinterpret_cast<double (*)[65]>(ism + 3 * 64 * 65);
    const int b = blockIdx.x, t = threadIdx.x;
    const double* Are = A + static_cast<size_t>(b) * mstride;
    const double* Aim = Are + plane;
    for (int q = t; q < 64 * 64; q += kInvThreads) {
        const int m = q / 64, i = q % 64;
        const size_t gi = static_cast<size_t>(k + m) * ld + k + i;
        lre[i][m] = Are[gi];
        lim[i][m] = Aim[gi];
    }
    double* rec = linv + static_cast<size_t>(b) * kLinvStride;
    __shared__ int pvs[64], psrc[64];
    if (t < 64) {
        pvs[t] = ipiv[static_cast<size_t>(b) * n + k + t];
        psrc[t] = k + t;
    }
    __syncthreads();
    if (t < 32) {  // warp 0: sequential LAPACK swaps -> gather map (outside rows held by lanes)
        int er0 = -1, er1 = -1, es0 = 0, es1 = 0, ne = 0;
        for (int c = 0; c < 64; ++c) {
            const int r = pvs[c];
            if (r == k + c) continue;
            if (r < k + 64) {
                if (t == 0) { const int tmp = psrc[c]; psrc[c] = psrc[r - k]; psrc[r - k] = tmp; }
            } else {
                const unsigned lo = __ballot_sync(0xffffffffu, er0 == r), hi = __ballot_sync(0xffffffffu, er1 == r);
                int j = lo ? __ffs(lo) - 1 : (hi ? 32 + __ffs(hi) - 1 : ne);
                if (j == ne) {  // first time this row is named
                    if (t == (j & 31)) { if (j < 32) { er0 = r; es0 = r; } else { er1 = r; es1 = r; } }
                    ++ne;
                }
                if (t == (j & 31)) {
                    int& es = j < 32 ? es0 : es1;
                    const int tmp = psrc[c]; psrc[c] = es; es = tmp;
                }
            }
            __syncwarp();
        }
        // rows -> virtual indices (outside rows by their slot)
        __shared__ int erow_s[64];
        if (t < ne) erow_s[t] = er0;
        if (t + 32 < ne) erow_s[t + 32] = er1;
        __syncwarp();
        auto virt = [&](int row) {
            if (row < k + 64) return row - k;
            int j = 0;
            while (erow_s[j] != row) ++j;
            return 64 + j;
        };
        SwapMap* sm = reinterpret_cast<SwapMap*>(rec + 2 * 64 * 64);
        sm->psrc[t] = virt(psrc[t]);
        sm->psrc[t + 32] = virt(psrc[t + 32]);
        if (t == 0) sm->next = ne;
        if (t < ne) { sm->erow[t] = er0; sm->esrc[t] = virt(es0); }
        if (t + 32 < ne) { sm->erow[t + 32] = er1; sm->esrc[t + 32] = virt(es1); }
    }
    // blocked inverse, 16x16 blocks D_I on the diagonal:
    //   X_II = D_I^{-1} (warp I, lane = column, in registers)
    //   X_IJ = -X_II sum_{K=J}^{I-1} L_IK X_KJ   for I = 1..3, J < I (block rows in order)
    double (*tre)[17] = reinterpret_cast<double (*)[17]>(ism + 4 * 64 * 65);  // [3 * 16][17] scratch
    double (*tim)[17] = reinterpret_cast<double (*)[17]>(ism + 4 * 64 * 65 + 48 * 17);
    const int warp = t >> 5, lane = t & 31;
    for (int q = t; q < 64 * 64; q += kInvThreads) {  // X = 0 (upper blocks stay zero)
        xre[q / 64][q % 64] = 0.0;
        xim[q / 64][q % 64] = 0.0;
    }
    __syncthreads();
    if (warp < 4 && lane < 16) {
        const int o = 16 * warp, c = lane;
        double xr[16], xi[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            double sr = 0.0, si = 0.0;
#pragma unroll
            for (int m = 0; m < i; ++m) {
                if (m >= c) {
                    const double a = lre[o + i][o + m], bb = lim[o + i][o + m];
                    sr += a * xr[m] - bb * xi[m];
                    si += a * xi[m] + bb * xr[m];
                }
            }
            xr[i] = i < c ? 0.0 : (i == c ? 1.0 : -sr);
            xi[i] = i <= c ? 0.0 : -si;
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            xre[o + i][o + c] = xr[i];
            xim[o + i][o + c] = xi[i];
        }
    }
    __syncthreads();
    const int r = t >> 4, c = t & 15;
    for (int I = 1; I < 4; ++I) {
        for (int J = 0; J < I; ++J) {  // T_J = sum_K L_IK X_KJ
            double sr = 0.0, si = 0.0;
            for (int kk = 16 * J; kk < 16 * I; ++kk) {
                const double a = lre[16 * I + r][kk], bb = lim[16 * I + r][kk];
                const double yr = xre[kk][16 * J + c], yi = xim[kk][16 * J + c];
                sr += a * yr - bb * yi;
                si += a * yi + bb * yr;
            }
            tre[16 * J + r][c] = sr;
            tim[16 * J + r][c] = si;
        }
        __syncthreads();
        for (int J = 0; J < I; ++J) {  // X_IJ = -X_II T_J
            double sr = 0.0, si = 0.0;
#pragma unroll
            for (int kk = 0; kk < 16; ++kk) {
                const double a = xre[16 * I + r][16 * I + kk], bb = xim[16 * I + r][16 * I + kk];
                const double yr = tre[16 * J + kk][c], yi = tim[16 * J + kk][c];
                sr += a * yr - bb * yi;
                si += a * yi + bb * yr;
            }
            xre[16 * I + r][16 * J + c] = -sr;
            xim[16 * I + r][16 * J + c] = -si;
        }
        __syncthreads();
    }
    // Linv stored [col c][row i]
    for (int q = t; q < 64 * 64; q += kInvThreads) {
        const int cc = q / 64, i = q % 64;
        rec[cc * 64 + i] = xre[i][cc];
        rec[64 * 64 + cc * 64 + i] = xim[i][cc];
    }
}

constexpr int SAS = 68;  // padded smem stride (≡ 4 mod 16 doubles)
constexpr int kApplyThreads = 256;
constexpr int kApplyCols = 32;  // strip width: L11^{-1} + one strip = 104 KB smem, 2 CTAs per SM

// One CTA per 32-column strip of the trailing columns: the panel rows of the
// strip are permuted through registers (sources in smem, or straight from HBM
// for the few outside rows a pivot names — every outside row receives a panel
// row, so no staging buffer is needed), the outside rows are written from the
// untouched strip, and U12 = L11^{-1} (P A12) runs on DMMA.
// mode 0: swap + TRSM; 1: swap only (the panel's interchanges applied to a
// column range, e.g. an earlier panel's L columns); 2: TRSM only (rows already
// in place); 3: swap, then the rank-rlen update from the earlier panels of the
// super-panel, columns [kp, kp + rlen) (X -= L[k.., kp..] U[kp.., strip],
// operands straight from L2 / HBM), then TRSM — panels 2..4 of a super-panel
// (rlen = 64, 128, 192). Columns [cb, ce).
__global__ void __launch_bounds__(kApplyThreads, 2)
lu_swap_apply_kernel(double* A, size_t mstride, size_t plane, int n, int ld, int k, const double* linv, int cb, int ce,
                     int mode, int kp, int rlen) {
    extern __shared__ __align__(16) double ssm[];
    double* Lr = ssm;                 // [kk][m] = Linv[m][kk]
    double* Li = Lr + 64 * SAS;
    double* Xr = Li + 64 * SAS;       // [n][kk], n < kApplyCols
    double* Xi = Xr + kApplyCols * SAS;
    __shared__ SwapMap map;
    const int b = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* Are = A + static_cast<size_t>(b) * mstride;
    double* Aim = Are + plane;
    const int col0 = cb + blockIdx.x * kApplyCols;
    const int ncols = min(kApplyCols, ce - col0);
    const double* rec = linv + static_cast<size_t>(b) * kLinvStride;
    const double* L = rec;
    {
        const int* src = reinterpret_cast<const int*>(rec + 2 * 64 * 64);
        int* dst = reinterpret_cast<int*>(&map);
        for (int q = tid; q < static_cast<int>(sizeof(SwapMap) / sizeof(int)); q += blockDim.x) dst[q] = src[q];
    }
    if (mode != 1)
        for (int q = tid; q < 64 * 64; q += blockDim.x) {
            const int kk = q / 64, m = q % 64;
            Lr[kk * SAS + m] = L[kk * 64 + m];
            Li[kk * SAS + m] = L[64 * 64 + kk * 64 + m];
        }
    // original panel rows of the strip (coalesced)
    for (int q = tid; q < kApplyCols * 64; q += blockDim.x) {
        const int nn = q / 64, kk = q % 64;
        double vr = 0.0, vi = 0.0;
        if (nn < ncols) {
            const size_t gi = static_cast<size_t>(col0 + nn) * ld + k + kk;
            vr = Are[gi];
            vi = Aim[gi];
        }
        Xr[nn * SAS + kk] = vr;
        Xi[nn * SAS + kk] = vi;
    }
    __syncthreads();
    const int ne = mode == 2 ? 0 : map.next;
    // permuted panel rows into registers: panel sources from smem, outside
    // sources (their original values) from HBM before any outside row is written
    constexpr int kPer = kApplyCols * 64 / kApplyThreads;
    double pr[kPer], pi[kPer];
#pragma unroll
    for (int p = 0; p < kPer; ++p) {
        const int q = tid + kApplyThreads * p, nn = q / 64, kk = q % 64;
        const int v = mode == 2 ? kk : map.psrc[kk];
        if (v < 64) {
            pr[p] = Xr[nn * SAS + v];
            pi[p] = Xi[nn * SAS + v];
        } else {
            pr[p] = pi[p] = 0.0;
            if (nn < ncols) {
                const size_t gi = static_cast<size_t>(col0 + nn) * ld + map.erow[v - 64];
                pr[p] = Are[gi];
                pi[p] = Aim[gi];
            }
        }
    }
    __syncthreads();
    // outside rows receive their (panel-row) sources from the untouched strip
    for (int q = tid; q < kApplyCols * ne; q += blockDim.x) {
        const int nn = q / ne, j = q % ne;
        if (nn < ncols) {
            const int v = map.esrc[j];
            const size_t gi = static_cast<size_t>(col0 + nn) * ld + map.erow[j];
            Are[gi] = Xr[nn * SAS + v];
            Aim[gi] = Xi[nn * SAS + v];
        }
    }
    __syncthreads();
    if (mode == 1) {  // permuted panel rows straight back
#pragma unroll
        for (int p = 0; p < kPer; ++p) {
            const int q = tid + kApplyThreads * p, nn = q / 64, kk = q % 64;
            if (nn < ncols) {
                const size_t gi = static_cast<size_t>(col0 + nn) * ld + k + kk;
                Are[gi] = pr[p];
                Aim[gi] = pi[p];
            }
        }
        return;
    }
#pragma unroll
    for (int p = 0; p < kPer; ++p) {
        const int q = tid + kApplyThreads * p, nn = q / 64, kk = q % 64;
        Xr[nn * SAS + kk] = pr[p];
        Xi[nn * SAS + kk] = pi[p];
    }
    __syncthreads();
    // 8 warps: 2 (rows of 32) x 4 (columns of 8)
    const int wm = warp & 1, wn = warp >> 1;
    if (mode == 3) {  // X -= L[k+m][kp+kk] U[kp+kk][col]: accumulators start from X
        double ur[4][2], ui[4][2];
        const int nn0 = wn * 8 + 2 * (lane & 3);
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
            const int m = wm * 32 + mi * 8 + (lane >> 2);
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                ur[mi][e] = Xr[(nn0 + e) * SAS + m];
                ui[mi][e] = Xi[(nn0 + e) * SAS + m];
            }
        }
        const int nb_col = col0 + wn * 8 + (lane >> 2);
        const bool bok = nb_col < ce;
#pragma unroll 4
        for (int k4 = 0; k4 < rlen; k4 += 4) {
            const int kk = kp + k4 + (lane & 3);
            double nar[4], fai[4], nai[4];
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) {
                const size_t gi = static_cast<size_t>(kk) * ld + k + wm * 32 + mi * 8 + (lane >> 2);
                nar[mi] = -Are[gi];
                fai[mi] = Aim[gi];
                nai[mi] = -fai[mi];
            }
            const size_t gb = static_cast<size_t>(nb_col) * ld + kk;
            const double br = bok ? Are[gb] : 0.0, bi = bok ? Aim[gb] : 0.0;
#pragma unroll
            for (int mi = 0; mi < 4; ++mi) {
                dmma(ur[mi][0], ur[mi][1], nar[mi], br);
                dmma(ur[mi][0], ur[mi][1], fai[mi], bi);
                dmma(ui[mi][0], ui[mi][1], nar[mi], bi);
                dmma(ui[mi][0], ui[mi][1], nai[mi], br);
            }
        }
        __syncthreads();  // every warp has read X
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
            const int m = wm * 32 + mi * 8 + (lane >> 2);
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                Xr[(nn0 + e) * SAS + m] = ur[mi][e];
                Xi[(nn0 + e) * SAS + m] = ui[mi][e];
            }
        }
        __syncthreads();
    }
    double acr[4][2] = {}, aci[4][2] = {};
#pragma unroll 4
    for (int k4 = 0; k4 < 64; k4 += 4) {
        const int kr = k4 + (lane & 3);
        double ar[4], ai[4], an[4];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
            const int m = wm * 32 + mi * 8 + (lane >> 2);
            ar[mi] = Lr[kr * SAS + m];
            ai[mi] = Li[kr * SAS + m];
            an[mi] = -ai[mi];
        }
        const int nn = wn * 8 + (lane >> 2);
        const double br = Xr[nn * SAS + kr], bi = Xi[nn * SAS + kr];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
            dmma(acr[mi][0], acr[mi][1], ar[mi], br);
            dmma(aci[mi][0], aci[mi][1], ar[mi], bi);
        }
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
            dmma(acr[mi][0], acr[mi][1], an[mi], bi);
            dmma(aci[mi][0], aci[mi][1], ai[mi], br);
        }
    }
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
        const int row = k + wm * 32 + mi * 8 + (lane >> 2);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int cl = wn * 8 + 2 * (lane & 3) + e;
            if (cl < ncols) {
                const size_t gi = static_cast<size_t>(col0 + cl) * ld + row;
                Are[gi] = acr[mi][e];
                Aim[gi] = aci[mi][e];
            }
        }
    }
}

// Rank-16 update of a sub-panel's window inside the 64-wide panel,
// A[r][c0:c1) -= L[r][ks:ks+16) U[ks:ks+16)[c0:c1) for rows r >= ks + 16,
// with the DMMA fragments loaded straight from HBM / L2 (sector-exact for the
// m8n8k4 layouts) and no shared memory, so four CTAs per SM keep the short
// load -> 16 DMMA -> store sequence of each tile overlapped.
constexpr int kWinThreads = 256;  // 8 warps x one 8-row m-tile each: 64 rows per CTA

__global__ void __launch_bounds__(kWinThreads, 4)
lu_window_update_kernel(double* A, size_t mstride, size_t plane, int n, int ld, int ks, int c0, int c1) {
    const int b = blockIdx.y, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* Are = A + static_cast<size_t>(b) * mstride;
    double* Aim = Are + plane;
    const int r = ks + 16 + blockIdx.x * 64 + warp * 8 + (lane >> 2);  // fragment row (A / C)
    const bool rok = r < n;
    const int q = lane & 3;
    // L fragments for the four k4 steps (negated: the update subtracts)
    double nar[4], ai[4], nai[4];
#pragma unroll
    for (int k4 = 0; k4 < 4; ++k4) {
        const size_t gi = static_cast<size_t>(ks + 4 * k4 + q) * ld + r;
        const double xr = rok ? Are[gi] : 0.0, xi = rok ? Aim[gi] : 0.0;
        nar[k4] = -xr;
        ai[k4] = xi;
        nai[k4] = -xi;
    }
    for (int n0 = c0; n0 < c1; n0 += 16) {  // two 8-column n-tiles per pass
        double acr[2][2], aci[2][2];
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = n0 + 8 * t + 2 * q + e;
                const size_t gi = static_cast<size_t>(col) * ld + r;
                const bool ok = rok && col < c1;
                acr[t][e] = ok ? Are[gi] : 0.0;
                aci[t][e] = ok ? Aim[gi] : 0.0;
            }
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4) {
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const int col = n0 + 8 * t + (lane >> 2);
                const size_t gi = static_cast<size_t>(col) * ld + ks + 4 * k4 + q;
                const double br = col < c1 ? Are[gi] : 0.0, bi = col < c1 ? Aim[gi] : 0.0;
                dmma(acr[t][0], acr[t][1], nar[k4], br);
                dmma(acr[t][0], acr[t][1], ai[k4], bi);
                dmma(aci[t][0], aci[t][1], nar[k4], bi);
                dmma(aci[t][0], aci[t][1], nai[k4], br);
            }
        }
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = n0 + 8 * t + 2 * q + e;
                if (rok && col < c1) {
                    const size_t gi = static_cast<size_t>(col) * ld + r;
                    Are[gi] = acr[t][e];
                    Aim[gi] = aci[t][e];
                }
            }
    }
}

// ------------------------------------------------------------------ 16-wide sub-panels
// For batches the 64-wide panel is factored as four 16-wide sub-panels: a
// 16-wide panel needs a quarter of the on-chip memory per matrix, so ~4x more
// matrices run their latency-bound column steps concurrently. Between
// sub-panels the remaining panel columns receive the sub-panel's row swaps, a
// 16x16 unit-lower solve and a rank-16 update; the 64-wide panel then leaves
// exactly the LAPACK-within-panel layout the trailing update and lu_solve use.
constexpr int kSub = 16;

__global__ void __launch_bounds__(64)
lu_sub_swap_trsm_kernel(double* A, size_t mstride, size_t plane, int n, int ld, int k, int w, int ks,
                        const int* ipiv) {
    // thread = one column c of the 64-panel outside the current sub-panel
    const int b = blockIdx.x;
    const int c = k + threadIdx.x;
    if (threadIdx.x >= w || (c >= ks && c < ks + kSub)) return;
    double* Are = A + static_cast<size_t>(b) * mstride;
    double* Aim = Are + plane;
    const size_t cb = static_cast<size_t>(c) * ld;
    const int* pv = ipiv + static_cast<size_t>(b) * n;
    for (int i = ks; i < ks + kSub; ++i) {
        const int r = pv[i];
        if (r == i) continue;
        const double tr = Are[cb + i], ti = Aim[cb + i];
        Are[cb + i] = Are[cb + r];
        Aim[cb + i] = Aim[cb + r];
        Are[cb + r] = tr;
        Aim[cb + r] = ti;
    }
    if (c < ks) return;  // columns left of the sub-panel hold L: swaps only
    // U = L11s^{-1} x on rows ks..ks+15 (unit lower, from columns ks..ks+15)
    double xr[kSub], xi[kSub];
#pragma unroll
    for (int i = 0; i < kSub; ++i) { xr[i] = Are[cb + ks + i]; xi[i] = Aim[cb + ks + i]; }
#pragma unroll
    for (int j = 0; j < kSub; ++j) {
#pragma unroll
        for (int i = j + 1; i < kSub; ++i) {
            const size_t li = static_cast<size_t>(ks + j) * ld + ks + i;
            const double lr = Are[li], lim = Aim[li];
            xr[i] -= lr * xr[j] - lim * xi[j];
            xi[i] -= lr * xi[j] + lim * xr[j];
        }
    }
#pragma unroll
    for (int i = 0; i < kSub; ++i) { Are[cb + ks + i] = xr[i]; Aim[cb + ks + i] = xi[i]; }
}


// ------------------------------------------------------------------ solves
// Blocked substitution, one 64-wide block column per step (the factor's panel
// width). Panel kernels: one CTA of 64 threads per matrix; thread i holds row i
// of the diagonal block in registers, so the serial triangular recurrence only
// waits on one barrier per column. GEMV kernels: 32-row slabs x 8 column
// groups per CTA, so even a single matrix puts ~25 warps of loads on every SM.
constexpr int kSolveW = 64;

__global__ void __launch_bounds__(kSolveW)
lu_fwd_panel_kernel(const double* A, size_t mstride, size_t plane, int n, int ld, int k, int w, const int* ipiv,
                    cplx* rhs, size_t rstride) {
    __shared__ cplx y[kSolveW], ext[kSolveW];
    __shared__ int pvs[kSolveW];
    const int b = blockIdx.x, tid = threadIdx.x;
    const double* Are = A + static_cast<size_t>(b) * mstride;
    const double* Aim = Are + plane;
    cplx* x = rhs + static_cast<size_t>(b) * rstride;
    const int* pv = ipiv + static_cast<size_t>(b) * n;
    // row tid of the unit-lower diagonal block, L[tid][j] for j < tid
    double lr[kSolveW - 1], li[kSolveW - 1];
#pragma unroll
    for (int j = 0; j < kSolveW - 1; ++j) {
        lr[j] = li[j] = 0.0;
        if (j < tid && tid < w) {
            const size_t gi = static_cast<size_t>(k + j) * ld + k + tid;
            lr[j] = Are[gi];
            li[j] = Aim[gi];
        }
    }
    // row interchanges of this block (LAPACK order): the block segment and the
    // rows below it that the pivots name are staged in smem, swapped by one
    // thread in order, and written back (each outside row by its first slot)
    int r = -1;
    if (tid < w) {
        r = pv[k + tid];
        pvs[tid] = r;
        y[tid] = x[k + tid];
        if (r >= k + w) ext[tid] = x[r];
    }
    __syncthreads();
    if (tid == 0) {
        for (int c = 0; c < w; ++c) {
            const int rc = pvs[c];
            if (rc == k + c) continue;
            if (rc < k + w) {
                const cplx t = y[c]; y[c] = y[rc - k]; y[rc - k] = t;
            } else {
                int slot = 0;
                while (pvs[slot] != rc) ++slot;
                const cplx t = y[c]; y[c] = ext[slot]; ext[slot] = t;
            }
        }
    }
    __syncthreads();
    if (tid < w && r >= k + w) {
        bool first = true;
        for (int c = 0; c < tid; ++c) first = first && pvs[c] != r;
        if (first) x[r] = ext[tid];
    }
    // unit-lower solve
    cplx yt = tid < w ? y[tid] : mk(0.0, 0.0);
#pragma unroll
    for (int j = 0; j < kSolveW - 1; ++j) {
        if (j >= w - 1) break;
        __syncthreads();
        const cplx yj = y[j];
        if (tid > j && tid < w) {
            yt = yt - mk(lr[j], li[j]) * yj;
            y[tid] = yt;
        }
    }
    if (tid < w) x[k + tid] = yt;
}

// x[r] -= A[r][k:k+w] y for a 32-row slab per CTA: warp g sums columns
// 8g..8g+7 for the slab's 32 consecutive rows (coalesced), then the 8 partial
// sums are reduced through smem in a fixed order.
constexpr int kGemvRows = 32, kGemvGroups = kSolveW / 8;

template <bool FWD>
__global__ void __launch_bounds__(kGemvRows * kGemvGroups)
lu_gemv_kernel(const double* A, size_t mstride, size_t plane, int n, int ld, int k, int w, cplx* rhs,
               size_t rstride) {
    __shared__ cplx y[kSolveW];
    __shared__ cplx part[kGemvGroups][kGemvRows];
    const int b = blockIdx.y;
    const double* Are = A + static_cast<size_t>(b) * mstride;
    const double* Aim = Are + plane;
    cplx* x = rhs + static_cast<size_t>(b) * rstride;
    const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
    if (threadIdx.x < kSolveW) y[threadIdx.x] = threadIdx.x < w ? x[k + threadIdx.x] : mk(0.0, 0.0);
    __syncthreads();
    const int r = (FWD ? k + w : 0) + blockIdx.x * kGemvRows + lane;
    const bool ok = FWD ? r < n : r < k;
    double ar = 0.0, ai = 0.0;
    if (ok) {
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
            const int j = 8 * g + jj;
            if (j < w) {
                const size_t gi = static_cast<size_t>(k + j) * ld + r;
                const double mr = Are[gi], mi = Aim[gi];
                ar += mr * y[j].re - mi * y[j].im;
                ai += mr * y[j].im + mi * y[j].re;
            }
        }
    }
    part[g][lane] = mk(ar, ai);
    __syncthreads();
    if (g == 0 && ok) {
        cplx acc = part[0][lane];
#pragma unroll
        for (int q = 1; q < kGemvGroups; ++q) acc = acc + part[q][lane];
        x[r] = x[r] - acc;
    }
}

__global__ void __launch_bounds__(kSolveW)
lu_bwd_panel_kernel(const double* A, size_t mstride, size_t plane, int n, int ld, int k, int w, cplx* rhs,
                    size_t rstride) {
    __shared__ cplx y[kSolveW];
    const int b = blockIdx.x, tid = threadIdx.x;
    const double* Are = A + static_cast<size_t>(b) * mstride;
    const double* Aim = Are + plane;
    cplx* x = rhs + static_cast<size_t>(b) * rstride;
    // row tid of the upper diagonal block, U[tid][j] for j >= tid
    double ur[kSolveW], ui[kSolveW];
#pragma unroll
    for (int j = 0; j < kSolveW; ++j) {
        ur[j] = ui[j] = 0.0;
        if (j >= tid && j < w) {
            const size_t gi = static_cast<size_t>(k + j) * ld + k + tid;
            ur[j] = Are[gi];
            ui[j] = Aim[gi];
        }
    }
    cplx diag = mk(1.0, 0.0);
#pragma unroll
    for (int j = 0; j < kSolveW; ++j)
        if (j == tid) diag = mk(ur[j], ui[j]);
    cplx yt = tid < w ? x[k + tid] : mk(0.0, 0.0);
    if (tid == w - 1) yt = cdiv(yt, diag);
    if (tid < w) y[tid] = yt;
    // column j final (divided) at the top of its step; row j-1 divides right after its last update
#pragma unroll
    for (int j = kSolveW - 1; j >= 1; --j) {
        if (j >= w) continue;
        __syncthreads();
        const cplx yj = y[j];
        if (tid < j) {
            yt = yt - mk(ur[j], ui[j]) * yj;
            if (tid == j - 1) yt = cdiv(yt, diag);
            y[tid] = yt;
        }
    }
    if (tid < w) x[k + tid] = yt;
}

// ------------------------------------------------------------------ dataflow solve
// Forward / backward substitution as a dataflow over row blocks of the
// factorization's panel width nb: one CTA per (block, matrix), handed out in
// dependency order through a ticket, so every block a CTA waits on
// already holds an SM or is done (no co-residency assumption). A block streams
// its L21 / U12 row blocks, multiplying each by an earlier solution block as
// soon as that block's flag is published (release / acquire), then finishes
// with one warp's substitution on its diagonal block staged in smem. The
// blocks progress as a wavefront instead of 2·n/nb dependent panel + GEMV
// launches, so a single system's solve runs at HBM speed.
//
// The factors keep each panel's row interchanges in the panel and the columns
// to its right only (the partial-pivoting schedule of lu_factor), so the L21
// rows that meet a given final row r sit at r's position at that panel's step:
// block m traces its rows back through panels m..0 (σ_{-1,m}, the position of
// r's right-hand-side entry) and forward again one panel per step. Panels with
// no interchange (pflag = 0, the usual case on BEM matrices) are skipped.
constexpr int kDfThreads = 256;  // 64 rows x 4 column groups

// poll a published flag with relaxed loads (an acquire per poll would
// invalidate L1 each time), then order the following loads with one fence
__device__ __forceinline__ void wait_flag(const int* p) {
    int v;
    do {
        asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
        if (v == 0) __nanosleep(32);
    } while (v == 0);
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

__device__ __forceinline__ int ld_relaxed_i(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Blocks publish in dependency order (block j's flag implies every block it
// depends on), so a warp that needs block j first looks at the last block it
// will ever need (`last`) and otherwise waits for j and scans on: it returns
// the furthest block known ready, fenced once, and polls again only past it.
// step = +1 (forward chain) or -1 (backward chain).
__device__ __forceinline__ int wait_ready(const int* fl, int j, int last, int step) {
    fds_jitter(j);
    int r = 0;
    if ((threadIdx.x & 31) == 0) {
        if (ld_relaxed_i(fl + last) != 0) {
            r = last;
        } else {
            wait_flag(fl + j);
            r = j;
            while (r != last && ld_relaxed_i(fl + r + step) != 0) r += step;
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    return __shfl_sync(0xffffffffu, r, 0);
}

__device__ __forceinline__ void st_release_i(int* p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int swap_forward(int q, const int* pv, int k, int w) {
    for (int i = 0; i < w; ++i) {
        const int a = k + i, b = __ldg(pv + a);
        q = q == a ? b : (q == b ? a : q);
    }
    return q;
}

__device__ __forceinline__ int swap_backward(int q, const int* pv, int k, int w) {
    for (int i = w - 1; i >= 0; --i) {
        const int a = k + i, b = __ldg(pv + a);
        q = q == a ? b : (q == b ? a : q);
    }
    return q;
}

// Interchange groups: 128-row super-panels below ks, nb-row panels from ks on.
// Interchange groups: 256-row super-panels below k1, 128-row super-panels in
// [k1, ks), nb-row panels from ks on.
struct SwapGroups {
    int n, nb, k1, ks;
    __host__ __device__ __forceinline__ int g1() const { return k1 >> 8; }
    __host__ __device__ __forceinline__ int g2() const { return g1() + ((ks - k1) >> 7); }
    __host__ __device__ __forceinline__ int count() const { return g2() + (n - ks + nb - 1) / nb; }
    __device__ __forceinline__ int of(int r) const {
        return r < k1 ? r >> 8 : (r < ks ? g1() + ((r - k1) >> 7) : g2() + (r - ks) / nb);
    }
    __device__ __forceinline__ int start(int g) const {
        return g < g1() ? g << 8 : (g < g2() ? k1 + ((g - g1()) << 7) : ks + (g - g2()) * nb);
    }
    __device__ __forceinline__ int size(int g) const {
        return min(g < g1() ? 256 : (g < g2() ? 128 : nb), n - start(g));
    }
};

// pflag[b][g] = interchange group g has an interchange (blockDim >= the largest group)
__global__ void __launch_bounds__(256)
lu_pivflag_kernel(SwapGroups sg, const int* ipiv, int* pflag) {
    const int b = blockIdx.y, g = blockIdx.x;
    const int r = sg.start(g) + threadIdx.x;
    const bool moved = threadIdx.x < sg.size(g) && ipiv[static_cast<size_t>(b) * sg.n + r] != r;
    const int any = __syncthreads_or(moved);
    if (threadIdx.x == 0) pflag[static_cast<size_t>(b) * sg.count() + g] = any;
}

// diagonal block rows/cols < w of matrix (Are, Aim) at (k, k) into smem, column-major [64][64] re then im
__device__ __forceinline__ void stage_diag(double* dsm, const double* Are, const double* Aim, int k, int w, int ld) {
#pragma unroll 4
    for (int e = threadIdx.x; e < 64 * 64; e += kDfThreads) {
        const int c = e >> 6, r = e & 63;
        double vr = 0.0, vi = 0.0;
        if (c < w && r < w) {
            const size_t gi = static_cast<size_t>(k + c) * ld + k + r;
            vr = Are[gi];
            vi = Aim[gi];
        }
        dsm[e] = vr;
        dsm[4096 + e] = vi;
    }
}

// In-place inverse of the staged diagonal block by all 256 threads, before
// the block's own wait: the unit-lower part (LOWER; X L = I, columns right to
// left) or the upper part (X U = I, columns left to right). The diagonal
// block's solve then becomes one parallel 64x64 product at the end of the
// dependency chain instead of 64 sequential substitution steps.
template <bool LOWER>
__device__ __forceinline__ void invert_diag(double* dsm, cplx (*red)[64], int w) {
    const int i = threadIdx.x & 63, g = threadIdx.x >> 6;
    auto S = [&](int r, int c) { return mk(dsm[c * 64 + r], dsm[4096 + c * 64 + r]); };
    if (LOWER) {
        for (int j = w - 2; j >= 0; --j) {
            cplx acc = mk(0.0, 0.0);
            if (i > j && i < w) {
                for (int k = j + 1 + g; k < i; k += 4) acc = acc + S(i, k) * S(k, j);
                if (g == 0) acc = acc + S(i, j);
            }
            red[g][i] = acc;
            __syncthreads();
            if (g == 0 && i > j && i < w) {
                const cplx x = red[0][i] + red[1][i] + red[2][i] + red[3][i];
                dsm[j * 64 + i] = -x.re;
                dsm[4096 + j * 64 + i] = -x.im;
            }
            __syncthreads();
        }
    } else {
        for (int j = 0; j < w; ++j) {
            cplx acc = mk(0.0, 0.0);
            if (i < j)
                for (int k = i + g; k < j; k += 4) acc = acc + S(i, k) * S(k, j);
            red[g][i] = acc;
            const cplx d = crecip(S(j, j));
            __syncthreads();
            if (g == 0 && i <= j) {
                const cplx x = i == j ? d : mk(0.0, 0.0) - (red[0][i] + red[1][i] + red[2][i] + red[3][i]) * d;
                dsm[j * 64 + i] = x.re;
                dsm[4096 + j * 64 + i] = x.im;
            }
            __syncthreads();
        }
    }
}

// v (smem, 64) -> X v with X the inverted diagonal block (unit lower: ones on
// the diagonal, zeros above; upper: zeros below). Returns row tr's value in
// threads g == 0.
template <bool LOWER>
__device__ __forceinline__ cplx apply_diag(const double* dsm, const cplx* v, cplx (*red)[64], int w) {
    const int tr = threadIdx.x & 63, g = threadIdx.x >> 6;
    double ar = 0.0, ai = 0.0;
#pragma unroll
    for (int cc = 0; cc < 16; ++cc) {
        const int c = g * 16 + cc;
        const bool on = LOWER ? c < tr : c >= tr;
        if (on && c < w) {
            const double xr = dsm[c * 64 + tr], xi = dsm[4096 + c * 64 + tr];
            ar += xr * v[c].re - xi * v[c].im;
            ai += xr * v[c].im + xi * v[c].re;
        }
    }
    red[g][tr] = mk(ar, ai);
    __syncthreads();
    cplx y = red[0][tr] + red[1][tr] + red[2][tr] + red[3][tr];
    if (LOWER) y = y + v[tr];
    return y;
}

template <int NB>
__global__ void __launch_bounds__(kDfThreads, 2)
lu_fwd_df_kernel(const double* A, size_t mstride, size_t plane, int n, int ld, int k1, int ks, const int* ipiv,
                 const int* pflag, const cplx* rhs, size_t rstride, cplx* ybuf, int* flags, int* tickets) {
    extern __shared__ double dsm[];  // unit-lower diagonal block
    __shared__ cplx part[4][64];
    __shared__ int s_m;
    const int tid = threadIdx.x, lane = tid & 31;
    constexpr int nb = NB, cpg = NB / 4;
    const int nblk = (n + nb - 1) / nb, batch = gridDim.x / nblk;
    if (tid == 0) s_m = atomicAdd(tickets, 1);
    __syncthreads();
    // tickets interleave the matrices (block-major), so every matrix's chain
    // advances in the same wave
    const int b = s_m % batch, m = s_m / batch, k = m * nb, w = min(nb, n - k);
    const double* Are = A + static_cast<size_t>(b) * mstride;
    const double* Aim = Are + plane;
    const int* pv = ipiv + static_cast<size_t>(b) * n;
    const SwapGroups sg{n, nb, k1, ks};
    const int* pf = pflag + static_cast<size_t>(b) * sg.count();
    int* fl = flags + static_cast<size_t>(b) * nblk;
    cplx* yb = ybuf + static_cast<size_t>(b) * n;
    __shared__ cplx vsm[64];
    stage_diag(dsm, Are, Aim, k, w, ld);
    __syncthreads();
    invert_diag<true>(dsm, part, w);
    const int tr = tid & 63, g = tid >> 6;
    const bool live = tr < w;
    int q = k + tr;
    if (live)
        for (int p = sg.of(k); p >= 0; --p)
            if (pf[p]) q = swap_backward(q, pv, sg.start(p), sg.size(p));
    double ar = 0.0, ai = 0.0;
    if (live && g == 0) {
        const cplx v = rhs[static_cast<size_t>(b) * rstride + q];
        ar = v.re;
        ai = v.im;
    }
    int ready = -1;  // furthest block known published (warp-uniform)
    for (int j = 0; j < m; ++j) {
        const int kj = j * nb;
        if (live) {
            const int gj = sg.of(kj);
            if (sg.start(gj) == kj && pf[gj]) q = swap_forward(q, pv, kj, sg.size(gj));
        }
        double lr[cpg], li[cpg];
        {
            const double* pr = Are + static_cast<size_t>(kj + g * cpg) * ld + q;
#pragma unroll
            for (int c = 0; c < cpg; ++c) {
                lr[c] = live ? __ldg(pr) : 0.0;
                li[c] = live ? __ldg(pr + plane) : 0.0;
                pr += ld;
            }
        }
        if (j > ready) ready = wait_ready(fl, j, m - 1, 1);
        __syncwarp();
#pragma unroll
        for (int c = 0; c < cpg; ++c) {
            const double2 y = __ldcg(reinterpret_cast<const double2*>(yb + kj + g * cpg + c));
            ar -= lr[c] * y.x - li[c] * y.y;
            ai -= lr[c] * y.y + li[c] * y.x;
        }
    }
    part[g][tr] = mk(ar, ai);
    __syncthreads();
    if (tid < 64) vsm[tid] = part[0][tid] + part[1][tid] + part[2][tid] + part[3][tid];
    __syncthreads();
    const cplx y = apply_diag<true>(dsm, vsm, part, w);
    if (g == 0 && live) yb[k + tr] = y;
    __threadfence();
    __syncthreads();
    fds_jitter(m);
    if (tid == 0) st_release_i(fl + m, 1);
}

template <int NB>
__global__ void __launch_bounds__(kDfThreads, 2)
lu_bwd_df_kernel(const double* A, size_t mstride, size_t plane, int n, int ld, const cplx* ybuf, cplx* rhs,
                 size_t rstride, int* flags, int* tickets) {
    extern __shared__ double dsm[];  // upper diagonal block
    __shared__ cplx part[4][64];
    __shared__ int s_m;
    const int tid = threadIdx.x, lane = tid & 31;
    constexpr int nb = NB, cpg = NB / 4;
    const int nblk = (n + nb - 1) / nb, batch = gridDim.x / nblk;
    if (tid == 0) s_m = atomicAdd(tickets, 1);
    __syncthreads();
    const int b = s_m % batch, m = nblk - 1 - s_m / batch, k = m * nb, w = min(nb, n - k);
    const double* Are = A + static_cast<size_t>(b) * mstride;
    const double* Aim = Are + plane;
    int* fl = flags + static_cast<size_t>(b) * nblk;
    cplx* x = rhs + static_cast<size_t>(b) * rstride;
    __shared__ cplx vsm[64];
    stage_diag(dsm, Are, Aim, k, w, ld);
    __syncthreads();
    invert_diag<false>(dsm, part, w);
    const int tr = tid & 63, g = tid >> 6;
    const bool live = tr < w;
    double ar = 0.0, ai = 0.0;
    int ready = nblk;  // furthest block known published (warp-uniform)
    for (int j = nblk - 1; j > m; --j) {
        const int kj = j * nb, wj = min(nb, n - kj);
        double ur[cpg], ui[cpg];
        {
            const double* pr = Are + static_cast<size_t>(kj + g * cpg) * ld + k + tr;
#pragma unroll
            for (int c = 0; c < cpg; ++c) {
                const bool on = live && g * cpg + c < wj;
                ur[c] = on ? __ldg(pr) : 0.0;
                ui[c] = on ? __ldg(pr + plane) : 0.0;
                pr += ld;
            }
        }
        if (j < ready) ready = wait_ready(fl, j, m + 1, -1);
        __syncwarp();
#pragma unroll
        for (int c = 0; c < cpg; ++c) {
            const int col = g * cpg + c;
            if (col < wj) {
                const double2 v = __ldcg(reinterpret_cast<const double2*>(x + kj + col));
                ar += ur[c] * v.x - ui[c] * v.y;
                ai += ur[c] * v.y + ui[c] * v.x;
            }
        }
    }
    part[g][tr] = mk(ar, ai);
    __syncthreads();
    if (tid < 64) {
        const cplx* yb = ybuf + static_cast<size_t>(b) * n;
        vsm[tid] = tid < w ? yb[k + tid] - (part[0][tid] + part[1][tid] + part[2][tid] + part[3][tid]) : mk(0.0, 0.0);
    }
    __syncthreads();
    const cplx xm = apply_diag<false>(dsm, vsm, part, w);
    if (g == 0 && live) x[k + tr] = xm;
    __threadfence();
    __syncthreads();
    fds_jitter(m);
    if (tid == 0) st_release_i(fl + m, 1);
}

// ------------------------------------------------------------------ host
void LuWorkspace::ensure(int groups, int P, int nb) {
    const size_t need = static_cast<size_t>(groups) * 2 * (P + 1) * (2 + 2 * nb) * sizeof(double) +
                        static_cast<size_t>(groups) * 2 * P * sizeof(double2);
    if (need > slot_bytes) {
        if (slots) cudaFree(slots);
        FDS_CUDA(cudaMalloc(&slots, need));
        slot_bytes = need;
    }
    if (groups > counter_count) {
        if (counters) cudaFree(counters);
        FDS_CUDA(cudaMalloc(&counters, groups * sizeof(unsigned)));
        counter_count = groups;
    }
}

void LuWorkspace::ensure_side() {
    if (side) return;
    int lo = 0, hi = 0;
    FDS_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    FDS_CUDA(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, hi));
    for (auto& e : ev) FDS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}

double* LuWorkspace::g3_planes(const LuProblem& pb) {
    const size_t need = static_cast<size_t>(pb.batch) * pb.ld * (2 * kG3W + kG3Rows);
    if (need > g3_cap) {
        if (g3) cudaFree(g3);
        FDS_CUDA(cudaMalloc(&g3, need * sizeof(double)));
        g3_cap = need;
    }
    return g3;
}

double* LuWorkspace::linv(int batch) {
    if (batch > linv_cap) {
        if (linv_buf) cudaFree(linv_buf);
        FDS_CUDA(cudaMalloc(&linv_buf, static_cast<size_t>(batch) * kLinvStride * sizeof(double)));
        linv_cap = batch;
    }
    return linv_buf;
}

void LuWorkspace::release() {
    if (g3) cudaFree(g3);
    g3 = nullptr;
    g3_cap = 0;
    if (ybuf) cudaFree(ybuf);
    if (sflags) cudaFree(sflags);
    ybuf = nullptr;
    sflags = nullptr;
    ybuf_cap = sflag_cap = 0;
    if (linv_buf) cudaFree(linv_buf);
    linv_buf = nullptr;
    linv_cap = 0;
    if (slots) cudaFree(slots);
    if (counters) cudaFree(counters);
    slots = nullptr;
    counters = nullptr;
    if (side) {
        cudaStreamSynchronize(side);
        cudaStreamDestroy(side);
    }
    for (auto& e : ev)
        if (e) cudaEventDestroy(e);
    side = nullptr;
    for (auto& e : ev) e = nullptr;
    slot_bytes = 0;
    counter_count = 0;
}

namespace {

size_t panel_smem(int nb, int R) { return (2 * static_cast<size_t>(nb) * R + 4 * nb) * sizeof(double); }

template <int NB>
int panel_rows_max() {
    const size_t budget = device_info().smem_optin - 8 * 1024;
    const int by_smem = static_cast<int>((budget / sizeof(double) - 4 * NB) / (2 * NB));
    return std::min(by_smem, kPanelThreads);  // one thread per row
}

// Co-resident CTAs of lu_panel_kernel<NB> at its largest row block (the group
// barrier needs a matrix's P CTAs on chip together): 16-wide sub-panels of 256
// rows take 66 KB, so three fit an SM and one matrix may have up to 3 x 148 x 256
// = 113 664 rows (N = 37 888 when it was one CTA per SM).
template <int NB>
int panel_ctas_max() {
    static std::mutex mu;
    static std::map<int, int> cache;
    int dev = 0;
    FDS_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    const size_t smem = panel_smem(NB, panel_rows_max<NB>());
    ensure_dynamic_smem(reinterpret_cast<const void*>(lu_panel_kernel<NB>), smem);
    int per_sm = 1;
    FDS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lu_panel_kernel<NB>, kPanelThreads, smem));
    return cache[dev] = device_info().sms * std::max(per_sm, 1);
}

bool use_cluster_panel() {
    static const bool on = [] {
        const char* e = std::getenv("FDSWEEP_PANEL_CLUSTER");
        return !(e && std::string(e) == "0");
    }();
    return on;
}

// One cluster of P CTAs per matrix (P <= 16, non-portable size), as many
// clusters as fit at once; each loops over matrices g, g+G, ...
template <int NB>
void panel_step_cluster(const LuProblem& pb, int k, int w, int P, int R, size_t smem, cudaStream_t st) {
    auto kern = lu_panel_cluster_kernel<NB>;
    ensure_dynamic_smem(reinterpret_cast<const void*>(kern), smem);
    once_per_device(reinterpret_cast<const void*>(kern), [&] {
        FDS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    });
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = P;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(kPanelThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(P);
    int clusters = 0;
    FDS_CUDA(cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg));
    const int G = std::max(1, std::min(pb.batch, clusters));
    cfg.gridDim = dim3(G * P);
    cudaEvent_t pe;
    profiler().begin(st, kProfLuPanel, 0.0, pe);
    FDS_CUDA(cudaLaunchKernelEx(&cfg, kern, pb.A, pb.mstride, pb.plane, pb.n, pb.ld, pb.batch, k, w, R, G, pb.ipiv,
                                pb.info));
    profiler().end(st, pe, kProfLuPanel, 8.0 * (pb.n - k) * w * w / 2.0 * pb.batch);
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

template <int NB>
void panel_step(const LuProblem& pb, LuWorkspace& ws, int k, int w, cudaStream_t st, bool coop = true) {
    const int sms = device_info().sms;
    const int rows = pb.n - k;
    const int rmax = panel_rows_max<NB>();
    int P = ceil_div(rows, rmax);
    if (P > panel_ctas_max<NB>()) throw NumericError("lu: panel does not fit in on-chip memory");
    const int R = ceil_div(rows, P);
    const size_t smem = panel_smem(NB, R);
    ensure_dynamic_smem(reinterpret_cast<const void*>(lu_panel_kernel<NB>), smem);
    if (NB == kSub && P <= 16 && use_cluster_panel()) {
        panel_step_cluster<NB>(pb, k, w, P, R, smem, st);
        return;
    }
    int per_sm = 1;
    FDS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lu_panel_kernel<NB>, kPanelThreads, smem));
    per_sm = std::max(per_sm, 1);
    const int G = std::max(1, std::min(pb.batch, (sms * per_sm) / P));
    ws.ensure(G, P, NB);
    FDS_CUDA(cudaMemsetAsync(ws.counters, 0, G * sizeof(unsigned), st));
    double* A = pb.A;
    size_t mstride = pb.mstride, plane = pb.plane;
    int n = pb.n, ld = pb.ld, batch = pb.batch;
    int* ipiv = pb.ipiv;
    int* info = pb.info;
    double* slots = ws.slots;
    unsigned* counters = ws.counters;
    int kk = k, ww = w, PP = P, RR = R, GG = G;
    void* args[] = {&A, &mstride, &plane, &n, &ld, &batch, &kk, &ww, &PP, &RR, &GG, &ipiv, &info, &slots, &counters};
    cudaEvent_t pe;
    profiler().begin(st, kProfLuPanel, 0.0, pe);
    if (coop) {
        FDS_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(lu_panel_kernel<NB>), dim3(G * P),
                                             dim3(kPanelThreads), args, smem, st));
    } else {
        // Pipelined mode: launched next to the other half-batch's GEMM on a
        // high-priority stream. G*P never exceeds what an idle GPU holds, and the
        // concurrent GEMM CTAs always retire, so every group's CTAs become
        // resident eventually; the CTA scheduler places these first.
        lu_panel_kernel<NB><<<G * P, kPanelThreads, smem, st>>>(A, mstride, plane, n, ld, batch, kk, ww, PP, RR, GG,
                                                                ipiv, info, slots, counters);
        FDS_CUDA(cudaGetLastError());
    }
    profiler().end(st, pe, kProfLuPanel, 8.0 * rows * w * w / 2.0 * pb.batch);
    g_launches.fetch_add(1, std::memory_order_relaxed);
}

constexpr size_t kInvSmem = (4 * 64 * 65 + 2 * 48 * 17) * sizeof(double);

// L11^{-1} and the swap map of the 64-wide panel at k (lu_l11_inverse_kernel)
void l11_inverse_step(const LuProblem& pb, int k, cudaStream_t st, double* linv) {
    ensure_dynamic_smem(reinterpret_cast<const void*>(lu_l11_inverse_kernel), kInvSmem);
    FDS_LAUNCH(lu_l11_inverse_kernel, pb.batch, kInvThreads, kInvSmem, st, pb.A, pb.mstride, pb.plane, pb.n, pb.ld, k,
               pb.ipiv, linv);
}

// inverse_ready: the look-ahead schedule already formed L11^{-1} on its side stream
template <int NB>
void trsm_step(const LuProblem& pb, int k, int w, cudaStream_t st, double* linv, bool inverse_ready = false) {
    const int rest = pb.n - k - w;
    if (rest <= 0) return;
    const size_t smem = (2 * NB * NB + 2 * kTrsmCols * NB) * sizeof(double);
    ensure_dynamic_smem(reinterpret_cast<const void*>(lu_swap_trsm_kernel<NB>), smem);
    cudaEvent_t te;
    profiler().begin(st, kProfLuTrsm, 0.0, te);
    if (NB == 64 && w == 64) {
        const size_t asmem = (2 * 64 * SAS + 2 * kApplyCols * SAS) * sizeof(double);
        ensure_dynamic_smem(reinterpret_cast<const void*>(lu_swap_apply_kernel), asmem);
        if (!inverse_ready) l11_inverse_step(pb, k, st, linv);
        FDS_LAUNCH(lu_swap_apply_kernel, dim3(ceil_div(rest, kApplyCols), pb.batch), kApplyThreads, asmem, st, pb.A,
                   pb.mstride, pb.plane, pb.n, pb.ld, k, linv, k + 64, pb.n, 0, 0, 64);
    } else {
        dim3 gt(ceil_div(rest, kTrsmCols), pb.batch);
        FDS_LAUNCH(lu_swap_trsm_kernel<NB>, gt, kTrsmThreads, smem, st, pb.A, pb.mstride, pb.plane, pb.n, pb.ld, k,
                   w, pb.ipiv);
    }
    profiler().end(st, te, kProfLuTrsm, 4.0 * w * w * rest * pb.batch);
}

// Tensor maps of a batch (rows x columns x planes, planes = 2 per matrix), cached
// per (base pointer, ld, batch): the box of A (L21 chunk) and of B (U12 chunk).
struct TmaMaps {
    CUtensorMap a, b, b32;  // b32: 32-column U12 boxes of the 3M kernel's narrow tiles
};

// Trailing-update kernel: 3M with 64x32 tiles, 2 CTAs/SM (default), or the
// four-product kernel (FDSWEEP_GEMM=4m: bit-identical results across batch
// sizes / schedules). 64x64 3M tiles at 1 CTA/SM, with 16 warps, or at 2
// CTAs/SM with spills, and a cp.async (non-TMA) operand feed were measured
// slower on B200 and removed.
bool gemm_3m() {
    static const bool v = [] {
        const char* e = std::getenv("FDSWEEP_GEMM");
        return !(e && std::string(e) == "4m");
    }();
    return v;
}

const TmaMaps& tma_maps(const LuProblem& pb) {
    static std::mutex mu;
    static std::map<std::tuple<const void*, int, int, size_t>, TmaMaps> cache;
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_tuple(static_cast<const void*>(pb.A), pb.ld, pb.batch, pb.plane);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    PFN_cuTensorMapEncodeTiled_v12000 encode = tensor_map_encoder();
    if (pb.mstride != 2 * pb.plane) throw ValidationError("lu: TMA path needs re/im planes back to back");
    TmaMaps m{};
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(pb.ld), static_cast<cuuint64_t>(pb.ld),
                                static_cast<cuuint64_t>(2) * pb.batch};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(pb.ld) * sizeof(double), pb.plane * sizeof(double)};
    const cuuint32_t estr[3] = {1, 1, 1};
    const cuuint32_t boxa[3] = {static_cast<cuuint32_t>(kTmaABox0), GBK, 1};
    const cuuint32_t boxb[3] = {static_cast<cuuint32_t>(kTmaBBox0), GBN, 1};
    auto enc = [&](CUtensorMap* t, const cuuint32_t* box) {
        const CUresult r = encode(t, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, pb.A, dims, strides, box, estr,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
    };
    const cuuint32_t boxb32[3] = {static_cast<cuuint32_t>(kTmaBBox0), 32, 1};
    enc(&m.a, boxa);
    enc(&m.b, boxb);
    enc(&m.b32, boxb32);
    return cache.emplace(key, m).first->second;
}

// The 3M kernel's pre-formed operand planes (LuWorkspace::g3): L21 sums as a
// [2 batch][kG3W][ld] tensor (boxes 68 x 16 like tmA), U12 sums as [batch][ld][kG3Rows]
// (boxes 20 x BN like tmB).
struct G3Maps {
    double* base = nullptr;
    CUtensorMap l, u32;
};

// set by lu_factor for the schedules whose updates run in stream order on one
// workspace (not the opt-in half-batch pipeline): enables the 3M update
thread_local LuWorkspace* t_g3_ws = nullptr;

const G3Maps& g3_maps(const LuProblem& pb, LuWorkspace& ws) {
    static std::mutex mu;
    static std::map<std::tuple<const void*, int, int>, G3Maps> cache;
    double* base = ws.g3_planes(pb);
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_tuple(static_cast<const void*>(base), pb.ld, pb.batch);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    G3Maps m{};
    m.base = base;
    const cuuint32_t estr[3] = {1, 1, 1};
    auto enc = [&](CUtensorMap* t, void* ptr, const cuuint64_t* dims, const cuuint64_t* strides, const cuuint32_t* box) {
        const CUresult r = tensor_map_encoder()(t, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, ptr, dims, strides, box, estr,
                                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
    };
    const cuuint64_t ldims[3] = {static_cast<cuuint64_t>(pb.ld), kG3W, static_cast<cuuint64_t>(2) * pb.batch};
    const cuuint64_t lstr[2] = {static_cast<cuuint64_t>(pb.ld) * sizeof(double),
                                static_cast<cuuint64_t>(pb.ld) * kG3W * sizeof(double)};
    const cuuint32_t lbox[3] = {static_cast<cuuint32_t>(kTmaABox0), GBK, 1};
    enc(&m.l, base, ldims, lstr, lbox);
    double* ubase = base + static_cast<size_t>(pb.batch) * 2 * kG3W * pb.ld;
    const cuuint64_t udims[3] = {kG3Rows, static_cast<cuuint64_t>(pb.ld), static_cast<cuuint64_t>(pb.batch)};
    const cuuint64_t ustr[2] = {kG3Rows * sizeof(double), static_cast<cuuint64_t>(pb.ld) * kG3Rows * sizeof(double)};
    const cuuint32_t ubox32[3] = {static_cast<cuuint32_t>(kTmaBBox0), 32, 1};
    enc(&m.u32, ubase, udims, ustr, ubox32);
    return cache.emplace(key, m).first->second;
}

// A22[:, c0:c1) -= L21 U12[:, c0:c1) for the rows below the panel (c0 >= k + w).
// A[k+w : r1)[c0 : c1) -= L U with the panel's w columns / rows (defaults: the
// whole trailing matrix)
// allow3m = false forces the four-product kernel: it needs no operand-plane
// workspace, so it can run on a side stream next to a 3M update.
void gemm_step(const LuProblem& pb, int k, int w, cudaStream_t st, int c0 = -1, int c1 = -1, int r1 = -1,
               bool allow3m = true) {
    if (r1 < 0) r1 = pb.n;
    const int rest = r1 - k - w;
    if (rest <= 0) return;
    if (c0 < 0) c0 = k + w;
    if (c1 < 0) c1 = pb.n;
    if (c1 <= c0) return;
    ensure_dynamic_smem(reinterpret_cast<const void*>(lu_gemm_kernel), kGemmSmemDoubles * sizeof(double));
    dim3 gg(ceil_div(rest, GBM), ceil_div(c1 - c0, GBN), pb.batch);
    cudaEvent_t ge;
    profiler().begin(st, kProfLuGemm, 0.0, ge);
    if (w == 256 && !(gemm_3m() && t_g3_ws && allow3m)) throw CudaError("lu: rank-256 updates need the 3M kernel");
    if (w == 64 || w == 128 || w == 256) {
        ensure_dynamic_smem(reinterpret_cast<const void*>(lu_gemm_tma_kernel<64>),
                            kGemmSmemDoubles * sizeof(double) + kTmaSmemPad);
        ensure_dynamic_smem(reinterpret_cast<const void*>(lu_gemm_tma_kernel<128>),
                            kGemmSmemDoubles * sizeof(double) + kTmaSmemPad);
        const TmaMaps& tm = tma_maps(pb);
        if (gemm_3m() && t_g3_ws && allow3m) {
            const G3Maps& gm = g3_maps(pb, *t_g3_ws);
            // operand planes: L21 once per (A, k, w) (the look-ahead window and the rest
            // share it; both run on this stream), U12 for this call's columns
            const bool do_l = !(t_g3_ws->g3_key_A == pb.A && t_g3_ws->g3_key_k == k && t_g3_ws->g3_key_w == w);
            t_g3_ws->g3_key_A = pb.A;
            t_g3_ws->g3_key_k = k;
            t_g3_ws->g3_key_w = w;
            if (w != 64 && w != 128 && w != 256) throw CudaError("lu: 3M operand planes need w = 64, 128 or 256");
            const int ublocks = static_cast<int>(std::min<long long>(
                ceil_div(static_cast<long long>(c1 - c0) * (w / 2), 256LL), 2LL * device_info().sms));
            FDS_LAUNCH(lu_g3_prep_kernel, dim3(static_cast<unsigned>((do_l ? w : 0) + ublocks), pb.batch), 256, 0, st,
                       pb.A, pb.mstride, pb.plane, pb.n, pb.ld, k, w, c0, c1, gm.base, do_l ? w : 0);
            constexpr size_t sm = g3_smem_doubles<32>() * sizeof(double) + 128 +
                                  GSTAGES * (sizeof(uint64_t) + sizeof(unsigned));
            // banded tile order once the L21 panel (3 planes, w deep) is a sizeable
            // part of the L2 (FDSWEEP_GEMM_BAND_MB, default 24 MB; FDSWEEP_GEMM_BAND
            // forces a band height in row tiles, 0 = off)
            static const int band_env = [] {
                const char* e = std::getenv("FDSWEEP_GEMM_BAND");
                return e ? std::atoi(e) : -1;
            }();
            static const double band_mb = [] {
                const char* e = std::getenv("FDSWEEP_GEMM_BAND_MB");
                return e ? std::atof(e) : 24.0;
            }();
            const double l21_bytes = 3.0 * sizeof(double) * w * static_cast<double>(rest);
            const int band = band_env >= 0 ? band_env : (l21_bytes > band_mb * 1e6 ? 64 : 0);
            auto go = [&](auto kern) {
                ensure_dynamic_smem(reinterpret_cast<const void*>(kern), sm);
                dim3 g3(ceil_div(rest, GBM), ceil_div(c1 - c0, 32), pb.batch);
                FDS_LAUNCH(kern, g3, kGemmThreads, sm, st, tm.a, tm.b32, gm.l, gm.u32, pb.A, pb.mstride, pb.plane,
                           pb.n, pb.ld, k, c0, band);
            };
            // P-first prologue on the first chunk (measured 0.4 % faster at cfg4)
            if (w == 256) go(lu_gemm3m_tma_kernel<256, 32, 4, 2, kGemmThreads, 1>);
            else if (w == 128) go(lu_gemm3m_tma_kernel<128, 32, 4, 2, kGemmThreads, 1>);
            else go(lu_gemm3m_tma_kernel<64, 32, 4, 2, kGemmThreads, 1>);
        } else if (w == 128)
            FDS_LAUNCH(lu_gemm_tma_kernel<128>, gg, kGemmThreads, kGemmSmemDoubles * sizeof(double) + kTmaSmemPad, st,
                       tm.a, tm.b, pb.A, pb.mstride, pb.plane, pb.n, pb.ld, k, c0);
        else
            FDS_LAUNCH(lu_gemm_tma_kernel<64>, gg, kGemmThreads, kGemmSmemDoubles * sizeof(double) + kTmaSmemPad, st,
                       tm.a, tm.b, pb.A, pb.mstride, pb.plane, pb.n, pb.ld, k, c0);
    } else {
        FDS_LAUNCH(lu_gemm_kernel, gg, kGemmThreads, kGemmSmemDoubles * sizeof(double), st, pb.A, pb.mstride,
                   pb.plane, pb.n, pb.ld, k, w, c0, c1);
    }
    // algorithmic flops of A22 -= L21 U12 (complex): 8 * rest^2 * w per matrix
    profiler().end(st, ge, kProfLuGemm, 8.0 * rest * (c1 - c0) * w * pb.batch);
}

template <int NB>
void trailing_step(const LuProblem& pb, int k, int w, cudaStream_t st, double* linv) {
    trsm_step<NB>(pb, k, w, st, linv);
    gemm_step(pb, k, w, st);
}

}  // namespace

namespace {

// 16-wide sub-panels: for batches ~4x more matrices fit on chip at once
// (cfg2 panel 225 -> 77 ms); for a single matrix the narrower rank-1 updates
// still win (N=15360 panel 107 -> 97 ms). FDSWEEP_SUBPANEL=0/1 overrides.
bool subpanels_enabled() {
    static const int env = [] {
        const char* e = std::getenv("FDSWEEP_SUBPANEL");
        return e ? std::atoi(e) : -1;
    }();
    return env != 0;
}

bool use_subpanels(const LuProblem&) { return subpanels_enabled(); }

}  // namespace

int lu_panel_width(int n) {
    // NB = 64; the panel must fit one matrix's rows in the SMs' shared memory:
    // as 16-wide sub-panels (default) or as one 64-wide GEPP panel; otherwise 32.
    if (ceil_div(n, panel_rows_max<64>()) <= panel_ctas_max<64>()) return 64;
    if (subpanels_enabled() && ceil_div(n, panel_rows_max<kSub>()) <= panel_ctas_max<kSub>()) return 64;
    return 32;
}

namespace {

bool window_kernel() {  // FDSWEEP_WINDOW=gemm routes the sub-panel window updates through lu_gemm_kernel
    static const bool on = [] {
        const char* e = std::getenv("FDSWEEP_WINDOW");
        return !(e && std::string(e) == "gemm");
    }();
    return on;
}

void subpanel_block(const LuProblem& pb, LuWorkspace& ws, int k, int w, cudaStream_t st, bool coop) {
    cudaEvent_t pe;
    profiler().begin(st, kProfLuPanel, 0.0, pe);
    const bool keep = profiler().enabled;
    profiler().enabled = false;  // account the sub-steps as one panel
    for (int ks = k; ks < k + 64; ks += kSub) {
        panel_step<kSub>(pb, ws, ks, kSub, st, coop);
        FDS_LAUNCH(lu_sub_swap_trsm_kernel, pb.batch, 64, 0, st, pb.A, pb.mstride, pb.plane, pb.n, pb.ld, k, w, ks,
                   pb.ipiv);
        if (ks + kSub < k + 64) {
            // rank-16 update of the panel's remaining columns, window [ks+16, k+64)
            const int rows = pb.n - ks - kSub;
            if (rows > 0) {
                if (window_kernel())
                    FDS_LAUNCH(lu_window_update_kernel, dim3(ceil_div(rows, 64), pb.batch), kWinThreads, 0, st, pb.A,
                               pb.mstride, pb.plane, pb.n, pb.ld, ks, ks + kSub, k + 64);
                else
                    gemm_step(pb, ks, kSub, st, ks + kSub, k + 64);
            }
        }
    }
    profiler().enabled = keep;
    profiler().end(st, pe, kProfLuPanel, 8.0 * (pb.n - k) * w * w / 2.0 * pb.batch);
}

int lookahead_mode() {
    static const int env = [] {
        const char* e = std::getenv("FDSWEEP_LOOKAHEAD");
        return e ? std::atoi(e) : -1;
    }();
    return env;
}

// Single-matrix look-ahead on 128-column super-panels (default) or on
// 64-column panels (FDSWEEP_LOOKAHEAD_SP=0).
bool lookahead_sp() {
    static const bool v = [] {
        const char* e = std::getenv("FDSWEEP_LOOKAHEAD_SP");
        return !(e && std::atoi(e) == 0);
    }();
    return v;
}

bool use_lookahead(const LuProblem& pb) {
    const int env = lookahead_mode();
    if (env >= 0) return env != 0;
    // single matrices. Measured: 64-column look-ahead, N = 15360 399 -> 368 ms
    // (326 -> 306 ms with the 3M update) but N = 36864 3.88 -> 4.07 s, so it
    // stopped at N <= 24576; the super-panel look-ahead (lookahead_sp) takes
    // N = 15360 from 305 to 278 ms and N = 36864 from 3.88 to 3.80 s.
    if (pb.batch != 1) return false;
    return lookahead_sp() || pb.n <= 24576;
}

// Look-ahead: the trailing update of step k is split into the next panel's
// 64 columns and the rest; the next panel (16-wide sub-panels, plain launch on
// a high-priority stream) factors while the rest of the GEMM runs, so the
// latency-bound column steps hide behind the tensor-pipe work. The next
// step's swap+TRSM waits for both (same stream order as the serial schedule).
void lu_factor_lookahead(const LuProblem& pb, LuWorkspace& ws, cudaStream_t st) {
    ws.ensure_side();
    cudaStream_t s_hi = ws.side;
    cudaEvent_t ev_a = ws.ev[0], ev_p = ws.ev[1];
    // two L11^{-1} slots: the side stream forms the next panel's inverse while
    // the current one is still applied
    double* linv_buf = ws.linv(2 * pb.batch);
    double* slot[2] = {linv_buf, linv_buf + static_cast<size_t>(pb.batch) * kLinvStride};
    subpanel_block(pb, ws, 0, 64, st, true);
    bool ready = false;
    for (int k = 0; k < pb.n; k += 64) {
        const int w = std::min(64, pb.n - k);
        double* linv = slot[(k / 64) & 1];
        trsm_step<64>(pb, k, w, st, linv, ready);
        const int nx = k + w;
        if (nx >= pb.n) break;
        const int wn = std::min(64, pb.n - nx);
        ready = false;
        if (wn == 64) {
            gemm_step(pb, k, w, st, nx, nx + 64);
            FDS_CUDA(cudaEventRecord(ev_a, st));
            FDS_CUDA(cudaStreamWaitEvent(s_hi, ev_a, 0));
            subpanel_block(pb, ws, nx, 64, s_hi, false);
            if (pb.n - nx - 64 > 0) {  // trsm_step of nx has trailing columns to apply
                l11_inverse_step(pb, nx, s_hi, slot[(nx / 64) & 1]);
                ready = true;
            }
            FDS_CUDA(cudaEventRecord(ev_p, s_hi));
            gemm_step(pb, k, w, st, nx + 64, pb.n);
            FDS_CUDA(cudaStreamWaitEvent(st, ev_p, 0));
        } else {
            gemm_step(pb, k, w, st);
            panel_step<64>(pb, ws, nx, wn, st);
        }
    }
}

}  // namespace

namespace {

bool super_panels() {  // FDSWEEP_SUPER=0 (or FDSWEEP_SOLVE=blocked) keeps one trailing update per 64-column panel
    static const bool on = [] {
        const char* e = std::getenv("FDSWEEP_SUPER");
        const char* sv = std::getenv("FDSWEEP_SOLVE");
        return !(e && std::string(e) == "0") && !(sv && std::string(sv) == "blocked");
    }();
    return on;
}

template <class F>
void profiler_scope_trsm(cudaStream_t st, F f, double work) {
    cudaEvent_t e;
    profiler().begin(st, kProfLuTrsm, 0.0, e);
    f();
    profiler().end(st, e, kProfLuTrsm, work);
}

void swap_cols(const LuProblem& pb, int k, int cb, int ce, int mode, const double* linv, cudaStream_t st, int kp = 0,
               int rlen = 64) {
    if (ce <= cb) return;
    const size_t asmem = (2 * 64 * SAS + 2 * kApplyCols * SAS) * sizeof(double);
    ensure_dynamic_smem(reinterpret_cast<const void*>(lu_swap_apply_kernel), asmem);
    FDS_LAUNCH(lu_swap_apply_kernel, dim3(ceil_div(ce - cb, kApplyCols), pb.batch), kApplyThreads, asmem, st, pb.A,
               pb.mstride, pb.plane, pb.n, pb.ld, k, linv, cb, ce, mode, kp, rlen);
}

// Two 64-column panels P1 = [k, k+64), P2 = [k+64, k+128) with one rank-128
// trailing update: P1 is factored, swapped into and solved against the
// trailing columns (U12_1) and applied to P2's columns only; P2 is factored,
// its interchanges are applied to P1's L columns and to the trailing columns,
// P2's rows of the trailing columns take P1's update and U12_2 = L22^{-1} A12_2
// (one strip kernel, mode 3),
// and rows/columns >= k+128 take [L21_1 L21_2][U12_1; U12_2] in one pass —
// each trailing C tile is loaded and stored once per 128 columns of k instead
// of twice. Inside the 128-column super-panel the interchanges are in LAPACK
// order (P2's reach P1's L columns), across super-panels in LINPACK order.
void super_panel_step(const LuProblem& pb, LuWorkspace& ws, int k, cudaStream_t st) {
    double* linv = ws.linv(pb.batch);
    const int k2 = k + 64, rest = pb.n - k - 128;
    subpanel_block(pb, ws, k, 64, st, true);
    trsm_step<64>(pb, k, 64, st, linv);
    gemm_step(pb, k, 64, st, k2, k2 + 64);
    subpanel_block(pb, ws, k2, 64, st, true);
    profiler_scope_trsm(st, [&] {
        l11_inverse_step(pb, k2, st, linv);
        swap_cols(pb, k2, k, k2, 1, linv, st);  // P2's interchanges into P1's L columns
        // trailing strips: P2's interchanges, P1's rank-64 update of P2's rows, L22^{-1}
        swap_cols(pb, k2, k + 128, pb.n, 3, linv, st, k);
    }, (4.0 + 8.0) * 64 * 64 * std::max(rest, 0) * pb.batch);
    if (rest <= 0) return;
    gemm_step(pb, k, 128, st);
}

// Four 64-column panels P1..P4 = [k, k+256) with one rank-256 trailing update:
// the first half H1 = P1 P2 runs as super_panel_step except that its rank-128
// update reaches only the second half's columns; P3 is factored, its
// interchanges go into H1's L columns, P4's columns take L33^{-1} and P3's
// rank-64 update, and the trailing columns take P3's interchanges, H1's
// rank-128 update of P3's rows and L33^{-1} (strip mode 3, rlen 128); P4 is
// factored, its interchanges go into [k, k+192) and the trailing columns take
// them, the rank-192 update of P4's rows and L44^{-1}; then rows / columns
// >= k+256 take [L21_1 .. L21_4][U12_1; ..; U12_4] in one pass — the trailing C
// tiles are read and written once per 256 columns of k. Interchanges are in
// LAPACK order inside the 256 columns, LINPACK order across super-panels.
void super_panel256_step(const LuProblem& pb, LuWorkspace& ws, int k, cudaStream_t st) {
    double* linv = ws.linv(pb.batch);
    const int k2 = k + 64, k3 = k + 128, k4 = k + 192, kt = k + 256;
    // H1 (P1, P2) with its update restricted to H2's columns
    subpanel_block(pb, ws, k, 64, st, true);
    trsm_step<64>(pb, k, 64, st, linv);
    gemm_step(pb, k, 64, st, k2, k3);
    subpanel_block(pb, ws, k2, 64, st, true);
    profiler_scope_trsm(st, [&] {
        l11_inverse_step(pb, k2, st, linv);
        swap_cols(pb, k2, k, k2, 1, linv, st);
        swap_cols(pb, k2, k3, pb.n, 3, linv, st, k, 64);
    }, (4.0 + 8.0) * 64 * 64 * (pb.n - k3) * pb.batch);
    gemm_step(pb, k, 128, st, k3, kt);
    // P3
    subpanel_block(pb, ws, k3, 64, st, true);
    profiler_scope_trsm(st, [&] {
        l11_inverse_step(pb, k3, st, linv);
        swap_cols(pb, k3, k, k3, 1, linv, st);             // into H1's L columns
        swap_cols(pb, k3, k4, kt, 0, linv, st);            // P4's columns: swap + L33^{-1}
        swap_cols(pb, k3, kt, pb.n, 3, linv, st, k, 128);  // trailing: swap, H1's update, L33^{-1}
    }, (4.0 + 8.0 * 2) * 64 * 64 * (pb.n - k4) * pb.batch);
    gemm_step(pb, k3, 64, st, k4, kt);
    // P4
    subpanel_block(pb, ws, k4, 64, st, true);
    profiler_scope_trsm(st, [&] {
        l11_inverse_step(pb, k4, st, linv);
        swap_cols(pb, k4, k, k4, 1, linv, st);             // into [k, k+192)
        swap_cols(pb, k4, kt, pb.n, 3, linv, st, k, 192);  // trailing: swap, rank-192 update, L44^{-1}
    }, (4.0 + 8.0 * 3) * 64 * 64 * (pb.n - kt) * pb.batch);
    if (pb.n - kt <= 0) return;
    gemm_step(pb, k, 256, st);
}

// 256-column super-panels (needs the 3M trailing update). Measured on B200:
// the N = 3840 batch of 129 factors in 537 vs 552 ms with 256- vs 128-column
// super-panels, the N = 15360 batch of 8 in 1995 vs 1983 ms (the rank-256
// update does not raise the GEMM's steady-state rate there, and the second
// half's panels run on a longer critical path), so the default takes them for
// n <= 8192. FDSWEEP_SUPER256=0 / 1 forces them off / on.
bool super256(int n) {
    static const int env = [] {
        const char* e = std::getenv("FDSWEEP_SUPER256");
        return e ? std::atoi(e) : -1;
    }();
    if (!gemm_3m()) return false;
    return env >= 0 ? env != 0 : n <= 8192;
}

// Look-ahead on 128-column super-panels (single matrices): the super-panel at
// k is split into its internal part (P1 factored, its interchanges and L11^-1
// applied to P2's columns, P1's rank-64 update of P2, P2 factored, its
// interchanges into P1's L columns) and its trailing part (both panels'
// interchanges, the in-super-panel update and L^-1 on the columns >= k+128).
// After super-panel k's rank-128 update of the next super-panel's 128 columns,
// the next internal part runs on the side stream while the main stream applies
// the rank-128 update to the remaining columns — the latency-bound panels hide
// behind the rank-128 3M GEMM, whose C tiles are read and written once per 128
// columns (the 64-column look-ahead updates rank 64 at a time). The side
// stream's rank-64 update uses the four-product kernel (no operand planes to
// share with the main stream's 3M update).
void sp_internal(const LuProblem& pb, LuWorkspace& ws, int k, cudaStream_t st, double* l1, double* l2) {
    subpanel_block(pb, ws, k, 64, st, false);
    l11_inverse_step(pb, k, st, l1);
    swap_cols(pb, k, k + 64, k + 128, 0, l1, st);       // P2's columns: P1's interchanges + L11^-1
    gemm_step(pb, k, 64, st, k + 64, k + 128, -1, false);  // P1's rank-64 update of P2 (rows >= k+64)
    subpanel_block(pb, ws, k + 64, 64, st, false);
    l11_inverse_step(pb, k + 64, st, l2);
    swap_cols(pb, k + 64, k, k + 64, 1, l2, st);        // P2's interchanges into P1's L columns
}

void lu_factor_lookahead_sp(const LuProblem& pb, LuWorkspace& ws, cudaStream_t st) {
    ws.ensure_side();
    cudaStream_t s_hi = ws.side;
    cudaEvent_t ev_a = ws.ev[0], ev_p = ws.ev[1];
    double* lbuf = ws.linv(4 * pb.batch);
    auto rec = [&](int i, int half) {
        return lbuf + static_cast<size_t>((i & 1) * 2 + half) * pb.batch * kLinvStride;
    };
    const int n = pb.n;
    const int n128 = n / 128 * 128;
    sp_internal(pb, ws, 0, st, rec(0, 0), rec(0, 1));
    for (int k = 0, i = 0; k < n128; k += 128, ++i) {
        const int kn = k + 128;
        profiler_scope_trsm(st, [&] {
            swap_cols(pb, k, kn, n, 0, rec(i, 0), st);              // P1's interchanges + L11^-1, columns >= k+128
            swap_cols(pb, k + 64, kn, n, 3, rec(i, 1), st, k, 64);  // P2's interchanges, P1's update, L22^-1
        }, (4.0 + 8.0 + 4.0) * 64 * 64 * std::max(n - kn, 0) * pb.batch);
        if (kn + 128 <= n) {
            gemm_step(pb, k, 128, st, kn, kn + 128);  // the next super-panel's columns first
            FDS_CUDA(cudaEventRecord(ev_a, st));
            FDS_CUDA(cudaStreamWaitEvent(s_hi, ev_a, 0));
            sp_internal(pb, ws, kn, s_hi, rec(i + 1, 0), rec(i + 1, 1));
            FDS_CUDA(cudaEventRecord(ev_p, s_hi));
            gemm_step(pb, k, 128, st, kn + 128, n);
            FDS_CUDA(cudaStreamWaitEvent(st, ev_p, 0));
        } else {
            gemm_step(pb, k, 128, st);
        }
    }
    ws.super_end = n128;
    double* linv = ws.linv(pb.batch);  // the last < 128 columns: 64-column panels
    for (int k = n128; k < n; k += 64) {
        const int w = std::min(64, n - k);
        if (w == 64) {
            subpanel_block(pb, ws, k, w, st, true);
            trailing_step<64>(pb, k, w, st, linv);
        } else {
            panel_step<64>(pb, ws, k, w, st);
            trailing_step<64>(pb, k, w, st, linv);
        }
    }
}

}  // namespace

std::unique_lock<std::mutex> lu_device_gate() {
    static std::mutex mu;
    static std::map<int, std::unique_ptr<std::mutex>> gates;
    int dev = 0;
    FDS_CUDA(cudaGetDevice(&dev));
    std::mutex* g;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto& p = gates[dev];
        if (!p) p = std::make_unique<std::mutex>();
        g = p.get();
    }
    return std::unique_lock<std::mutex>(*g);
}

void lu_factor(const LuProblem& pb, LuWorkspace& ws, cudaStream_t st) {
    FDS_CUDA(cudaMemsetAsync(pb.info, 0, pb.batch * sizeof(int), st));
    ws.super_end = ws.super256_end = 0;
    struct G3Scope {  // the 3M update's operand planes live in this workspace
        explicit G3Scope(LuWorkspace* w) {
            w->g3_key_A = nullptr;
            w->g3_key_k = w->g3_key_w = -1;
            t_g3_ws = w;
        }
        ~G3Scope() { t_g3_ws = nullptr; }
    } g3scope(&ws);
    if (lu_panel_width(pb.n) == 64 && subpanels_enabled() && pb.n >= 128 && use_lookahead(pb)) {
        if (lookahead_sp() && super_panels() && pb.n >= 256)
            lu_factor_lookahead_sp(pb, ws, st);
        else
            lu_factor_lookahead(pb, ws, st);
        return;
    }
    const int nb = lu_panel_width(pb.n);
    for (int k = 0; k < pb.n; k += nb) {
        const int w = std::min(nb, pb.n - k);
        if (nb == 64 && w == 64 && use_subpanels(pb) && super_panels() && super256(pb.n) && k + 256 <= pb.n &&
            ws.super_end == ws.super256_end) {
            super_panel256_step(pb, ws, k, st);
            ws.super_end = ws.super256_end = k + 256;
            k += 192;  // four panels
        } else if (nb == 64 && w == 64 && use_subpanels(pb) && super_panels() && k + 128 <= pb.n) {
            super_panel_step(pb, ws, k, st);
            ws.super_end = k + 128;
            k += 64;  // two panels
        } else if (nb == 64 && w == 64 && use_subpanels(pb)) {
            subpanel_block(pb, ws, k, w, st, true);
            trailing_step<64>(pb, k, w, st, ws.linv(pb.batch));
        } else if (nb == 64) {
            panel_step<64>(pb, ws, k, w, st);
            trailing_step<64>(pb, k, w, st, ws.linv(pb.batch));
        } else {
            panel_step<32>(pb, ws, k, w, st);
            trailing_step<32>(pb, k, w, st, nullptr);
        }
    }
}

void LuWorkspace::ensure_solve(int batch, int n, int nblk) {
    const size_t yneed = static_cast<size_t>(batch) * n;
    if (yneed > ybuf_cap) {
        if (ybuf) cudaFree(ybuf);
        ybuf = nullptr;
        FDS_CUDA(cudaMalloc(&ybuf, yneed * sizeof(cplx)));
        ybuf_cap = yneed;
    }
    // pflag [batch][nblk], flags fwd / bwd [batch][nblk], tickets fwd / bwd
    const size_t fneed = 3 * static_cast<size_t>(batch) * nblk + 2;
    if (fneed > sflag_cap) {
        if (sflags) cudaFree(sflags);
        sflags = nullptr;
        FDS_CUDA(cudaMalloc(&sflags, fneed * sizeof(int)));
        sflag_cap = fneed;
    }
}

namespace {

bool dataflow_solve() {
    static const bool on = [] {
        const char* e = std::getenv("FDSWEEP_SOLVE");
        return !(e && std::string(e) == "blocked");
    }();
    return on;
}

void lu_solve_blocked(const LuProblem& pb, cplx* rhs, size_t rstride, cudaStream_t st);

}  // namespace

void lu_solve(const LuProblem& pb, cplx* rhs, size_t rstride, LuWorkspace& ws, cudaStream_t st) {
    if (!dataflow_solve() && ws.super_end == 0) {  // the per-panel solve follows nb-column interchange groups only
        lu_solve_blocked(pb, rhs, rstride, st);
        return;
    }
    const int nb = lu_panel_width(pb.n);
    const int nblk = ceil_div(pb.n, nb);
    const int ks = nb == 64 ? ws.super_end : 0;
    const int k1 = nb == 64 ? ws.super256_end : 0;
    ws.ensure_solve(pb.batch, pb.n, nblk);
    int* pflag = ws.sflags;  // [batch][groups] fits in the [batch][nblk] slot
    int* ffl = pflag + static_cast<size_t>(pb.batch) * nblk;
    int* bfl = ffl + static_cast<size_t>(pb.batch) * nblk;
    int* tk = bfl + static_cast<size_t>(pb.batch) * nblk;
    FDS_CUDA(cudaMemsetAsync(ffl, 0, (2 * static_cast<size_t>(pb.batch) * nblk + 2) * sizeof(int), st));
    const size_t smem = 2 * 64 * 64 * sizeof(double);
    const SwapGroups sg{pb.n, nb, k1, ks};
    const int groups = sg.count();
    FDS_LAUNCH(lu_pivflag_kernel, dim3(groups, pb.batch), 256, 0, st, sg, pb.ipiv, pflag);
    const int ctas = nblk * pb.batch;
    auto go = [&](auto fwd, auto bwd) {
        ensure_dynamic_smem(reinterpret_cast<const void*>(fwd), smem);
        ensure_dynamic_smem(reinterpret_cast<const void*>(bwd), smem);
        FDS_LAUNCH(fwd, ctas, kDfThreads, smem, st, pb.A, pb.mstride, pb.plane, pb.n, pb.ld, k1, ks, pb.ipiv, pflag,
                   rhs, rstride, ws.ybuf, ffl, tk);
        FDS_LAUNCH(bwd, ctas, kDfThreads, smem, st, pb.A, pb.mstride, pb.plane, pb.n, pb.ld, ws.ybuf, rhs, rstride, bfl,
                   tk + 1);
    };
    if (nb == 64) go(lu_fwd_df_kernel<64>, lu_bwd_df_kernel<64>);
    else go(lu_fwd_df_kernel<32>, lu_bwd_df_kernel<32>);
}

namespace {

void lu_solve_blocked(const LuProblem& pb, cplx* rhs, size_t rstride, cudaStream_t st) {
    const int nb = lu_panel_width(pb.n);
    for (int k = 0; k < pb.n; k += nb) {
        const int w = std::min(nb, pb.n - k);
        FDS_LAUNCH(lu_fwd_panel_kernel, pb.batch, kSolveW, 0, st, pb.A, pb.mstride, pb.plane, pb.n, pb.ld, k, w,
                   pb.ipiv, rhs, rstride);
        const int rest = pb.n - k - w;
        if (rest > 0) {
            dim3 g(ceil_div(rest, kGemvRows), pb.batch);
            FDS_LAUNCH(lu_gemv_kernel<true>, g, kGemvRows * kGemvGroups, 0, st, pb.A, pb.mstride, pb.plane, pb.n, pb.ld, k, w, rhs,
                       rstride);
        }
    }
    const int last = ((pb.n - 1) / nb) * nb;
    for (int k = last; k >= 0; k -= nb) {
        const int w = std::min(nb, pb.n - k);
        FDS_LAUNCH(lu_bwd_panel_kernel, pb.batch, kSolveW, 0, st, pb.A, pb.mstride, pb.plane, pb.n, pb.ld, k, w,
                   rhs, rstride);
        if (k > 0) {
            dim3 g(ceil_div(k, kGemvRows), pb.batch);
            FDS_LAUNCH(lu_gemv_kernel<false>, g, kGemvRows * kGemvGroups, 0, st, pb.A, pb.mstride, pb.plane, pb.n, pb.ld, k, w, rhs,
                       rstride);
        }
    }
}

}  // namespace

}  // namespace fdsb
