// Column-pivoted Householder least squares on the device (one CTA), for the
// two small dense systems of vector fitting:
//   * the stacked sigma system of relocate_poles (vecfit.cpp:281-285,
//     Eigen::ColPivHouseholderQR in the reference): K_orf*red x M, solved for
//     one right-hand side, plus the per-channel residual RMS (:287-295);
//   * the shared LS matrix [Re Phi; Im Phi] of identify_residues
//     (vecfit.cpp:385-395): 2J x M, turned into the explicit solve operator W
//     (M x 2J, W b = x) that vf_residue_mma_kernel applies to every channel.
// Semantics of the reference's decomposition: column pivoting on the largest
// remaining column norm (first maximum), norm downdating with a recompute when
// the downdated norm has lost half its digits (sqrt(eps) test), Householder
// sign convention beta = -sign(x0) ||x||, rank = #{|R_ii| > min(m,n) eps
// max|R_jj|} over the pivots taken before the remaining norms fall to
// eps-level, basic solution over those pivots. Reductions run as warp trees
// (fixed order, so results are reproducible run to run).
#include <cfloat>

#include "vf.cuh"

namespace fdsb {

namespace {

constexpr int kLsqThreads = 512;
constexpr int kLsqWarps = kLsqThreads / 32;
constexpr int kLsqCols = 128;  // right-hand sides solved together (one thread each)
constexpr double kSqrtEps = 1.4901161193847656e-08;  // sqrt(DBL_EPSILON) = 2^-26

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Storage of the working set: dynamic shared memory (SMEM) or a global
// workspace for systems that do not fit; one template instance each so the
// shared path compiles to LDS/STS.
struct LsqLayout {
    int m, n, lda;
    __host__ __device__ size_t a_doubles() const { return static_cast<size_t>(lda) * n; }
    __host__ __device__ size_t b_doubles() const { return static_cast<size_t>(m) * kLsqCols; }
    __host__ __device__ size_t total_doubles() const { return a_doubles() + 4 * static_cast<size_t>(n) + b_doubles() + (n + 1) / 2 + 2; }
};

}  // namespace

// in(i, j) = in[i*rs + j*cs]. Mode A (x_out != null): solve for rhs, x_out[n].
// Mode B (w_out != null): w_out[c*m + i] = wscale[c] * W(c, i) for the explicit
// solve operator. The factorization runs one Householder step per iteration
// (warp 0: pivot, interchange, reflector; all warps: reflector applied to the
// trailing columns, one warp per column, and the norm downdate); the solves run
// one thread per right-hand side (kLsqCols at a time) with no reductions:
// Q^T b by broadcast reads of each reflector, then column-oriented back
// substitution with the reciprocal diagonal.
template <bool SMEM>
__global__ void __launch_bounds__(kLsqThreads)
vf_lsq_kernel(int m, int n, const double* __restrict__ in, long long rs, long long cs, const double* __restrict__ rhs,
              double* gwork, double* __restrict__ x_out, double* __restrict__ w_out,
              const double* __restrict__ wscale, VfLsqStatus* __restrict__ status) {
    extern __shared__ double lsm[];
    __shared__ int s_nonzero, s_rank;
    __shared__ double s_maxpivot, s_thr;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int size = min(m, n);
    const LsqLayout L{m, n, m | 1};
    const int lda = L.lda;
    double* a = SMEM ? lsm : gwork;                  // lda x n, column-major (odd lda: conflict-free rows)
    double* upd = a + L.a_doubles();                 // downdated column norms
    double* dir = upd + n;                           // norms at the last recompute
    double* tau = dir + n;
    double* rdiag = tau + n;                         // 1 / R_ii
    double* bb = rdiag + n;                          // m x kLsqCols right-hand sides, row-major
    int* perm = reinterpret_cast<int*>(bb + L.b_doubles());

    for (size_t idx = tid; idx < static_cast<size_t>(m) * n; idx += kLsqThreads) {
        const int i = static_cast<int>(idx % m), j = static_cast<int>(idx / m);
        a[static_cast<size_t>(j) * lda + i] = in[static_cast<long long>(i) * rs + static_cast<long long>(j) * cs];
    }
    for (int j = tid; j < n; j += kLsqThreads) perm[j] = j;
    __syncthreads();
    for (int j = warp; j < n; j += kLsqWarps) {
        double s = 0.0;
        for (int i = lane; i < m; i += 32) s += a[static_cast<size_t>(j) * lda + i] * a[static_cast<size_t>(j) * lda + i];
        s = warp_sum(s);
        if (lane == 0) upd[j] = dir[j] = sqrt(s);
    }
    __syncthreads();
    if (tid == 0) {
        double mx = 0.0;
        for (int j = 0; j < n; ++j) mx = fmax(mx, upd[j]);
        s_thr = (mx * DBL_EPSILON) * (mx * DBL_EPSILON) / m;
        s_nonzero = size;
        s_maxpivot = 0.0;
    }
    for (int k = 0; k < size; ++k) {
        __syncthreads();
        if (warp == 0) {
            // pivot: largest remaining norm, first maximum (warp argmax)
            double bv = -1.0;
            int bj = n;
            for (int j = k + lane; j < n; j += 32) {
                const double u = upd[j];
                if (u > bv) { bv = u; bj = j; }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
                if (ov > bv || (ov == bv && oj < bj)) { bv = ov; bj = oj; }
            }
            const int big = bj;
            if (lane == 0 && s_nonzero == size && bv * bv < s_thr * (m - k)) s_nonzero = k;
            if (big != k) {
                for (int i = lane; i < m; i += 32) {
                    const double t = a[static_cast<size_t>(k) * lda + i];
                    a[static_cast<size_t>(k) * lda + i] = a[static_cast<size_t>(big) * lda + i];
                    a[static_cast<size_t>(big) * lda + i] = t;
                }
                if (lane == 0) {
                    double t = upd[k]; upd[k] = upd[big]; upd[big] = t;
                    t = dir[k]; dir[k] = dir[big]; dir[big] = t;
                    const int p = perm[k]; perm[k] = perm[big]; perm[big] = p;
                }
                __syncwarp();
            }
            // Householder vector of column k, rows k..m-1
            double* x = a + static_cast<size_t>(k) * lda + k;
            const int len = m - k;
            double tail = 0.0;
            for (int i = 1 + lane; i < len; i += 32) tail += x[i] * x[i];
            tail = warp_sum(tail);
            const double c0 = x[0];
            double t, beta;
            if (tail <= DBL_MIN) {
                t = 0.0;
                beta = c0;
                for (int i = 1 + lane; i < len; i += 32) x[i] = 0.0;
            } else {
                beta = sqrt(c0 * c0 + tail);
                if (c0 >= 0.0) beta = -beta;
                const double inv = 1.0 / (c0 - beta);
                for (int i = 1 + lane; i < len; i += 32) x[i] *= inv;
                t = (beta - c0) / beta;
            }
            __syncwarp();
            if (lane == 0) {
                x[0] = beta;
                tau[k] = t;
                rdiag[k] = 1.0 / beta;
                s_maxpivot = fmax(s_maxpivot, fabs(beta));
            }
        }
        __syncthreads();
        const double t = tau[k];
        const double* ess = a + static_cast<size_t>(k) * lda + k;
        for (int j = k + 1 + warp; j < n; j += kLsqWarps) {  // apply H_k, downdate the norm
            double* col = a + static_cast<size_t>(j) * lda + k;
            double c0 = col[0];
            if (t != 0.0) {
                double d = 0.0;
                for (int i = 1 + lane; i < m - k; i += 32) d += ess[i] * col[i];
                d = (warp_sum(d) + c0) * t;
                for (int i = 1 + lane; i < m - k; i += 32) col[i] -= d * ess[i];
                c0 -= d;
                if (lane == 0) col[0] = c0;
            }
            const double u = upd[j];
            if (u != 0.0) {  // every lane evaluates the test (no broadcast needed)
                double q = fabs(c0) / u;
                q = (1.0 + q) * (1.0 - q);
                if (q < 0.0) q = 0.0;
                const double r = u / dir[j];
                if (q * r * r <= kSqrtEps) {
                    __syncwarp();
                    double s = 0.0;
                    for (int i = 1 + lane; i < m - k; i += 32) s += col[i] * col[i];
                    s = warp_sum(s);
                    if (lane == 0) upd[j] = dir[j] = sqrt(s);
                } else if (lane == 0) {
                    upd[j] = u * sqrt(q);
                }
            }
        }
    }
    __syncthreads();
    if (tid == 0) {
        const double pre = fabs(s_maxpivot) * (size * DBL_EPSILON);
        int r = 0;
        for (int i = 0; i < s_nonzero; ++i) r += fabs(a[static_cast<size_t>(i) * lda + i]) > pre;
        s_rank = r;
        status->rank = r;
        status->nonzero = s_nonzero;
        status->maxpivot = s_maxpivot;
    }
    __syncthreads();
    if (s_rank < n) return;  // the caller raises NumericError; no solution is formed
    const int np = s_nonzero;
    const int nrhs = x_out ? 1 : m;
    for (int c0 = 0; c0 < nrhs; c0 += kLsqCols) {
        const int c = c0 + tid;
        const bool mine = tid < kLsqCols && c < nrhs;
        if (mine)
            for (int i = 0; i < m; ++i) bb[static_cast<size_t>(i) * kLsqCols + tid] = x_out ? rhs[i] : (i == c ? 1.0 : 0.0);
        if (mine) {
            double* b = bb + tid;  // this thread's column, stride kLsqCols
            for (int k = 0; k < np; ++k) {  // b <- Q^T b
                const double t = tau[k];
                if (t == 0.0) continue;
                const double* ess = a + static_cast<size_t>(k) * lda + k;
                double d0 = b[static_cast<size_t>(k) * kLsqCols], d1 = 0.0;
                int i = 1;
                for (; i + 1 < m - k; i += 2) {
                    d0 += ess[i] * b[static_cast<size_t>(k + i) * kLsqCols];
                    d1 += ess[i + 1] * b[static_cast<size_t>(k + i + 1) * kLsqCols];
                }
                if (i < m - k) d0 += ess[i] * b[static_cast<size_t>(k + i) * kLsqCols];
                const double d = (d0 + d1) * t;
                b[static_cast<size_t>(k) * kLsqCols] -= d;
                for (int r = 1; r < m - k; ++r) b[static_cast<size_t>(k + r) * kLsqCols] -= d * ess[r];
            }
            for (int i = np - 1; i >= 0; --i) {  // R11 z = (Q^T b)[0:np], column-oriented
                const double* col = a + static_cast<size_t>(i) * lda;
                const double zi = b[static_cast<size_t>(i) * kLsqCols] * rdiag[i];
                b[static_cast<size_t>(i) * kLsqCols] = zi;
                for (int j = 0; j < i; ++j) b[static_cast<size_t>(j) * kLsqCols] -= zi * col[j];
            }
            if (x_out) {
                for (int i = 0; i < n; ++i) x_out[i] = 0.0;
                for (int i = 0; i < np; ++i) x_out[perm[i]] = b[static_cast<size_t>(i) * kLsqCols];
            } else {
                for (int i = 0; i < n; ++i) w_out[static_cast<size_t>(i) * m + c] = 0.0;
                for (int i = 0; i < np; ++i)
                    w_out[static_cast<size_t>(perm[i]) * m + c] = wscale[perm[i]] * b[static_cast<size_t>(i) * kLsqCols];
            }
        }
    }
}

// Per-channel RMS of the relocation LS residual (vecfit.cpp:287-295):
// rms_k = sqrt((||R22_k y - beta_k||^2 + tail_k) / J); one warp per channel.
__global__ void vf_reloc_rms_kernel(int K, int red, int M, int J, const double* __restrict__ r22,
                                    const double* __restrict__ beta, const double* __restrict__ tail,
                                    const double* __restrict__ y, double* __restrict__ rms) {
    const int k = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (k >= K) return;
    double c2 = 0.0;
    for (int i = 0; i < red; ++i) {
        const double* row = r22 + (static_cast<size_t>(k) * red + i) * M;
        double v = 0.0;
        for (int c = lane; c < M; c += 32) v += row[c] * y[c];
        v = warp_sum(v) - beta[static_cast<size_t>(k) * red + i];
        c2 += v * v;
    }
    if (lane == 0) rms[k] = sqrt((c2 + tail[k]) / J);
}

void vf_lsq_launch(int m, int n, const double* in, long long rs, long long cs, const double* rhs, double* x_out,
                   double* w_out, const double* wscale, VfLsqStatus* status, cudaStream_t st) {
    const LsqLayout L{m, n, m | 1};
    const size_t bytes = L.total_doubles() * sizeof(double);
    if (bytes <= static_cast<size_t>(device_info().smem_optin) - 2048) {
        ensure_dynamic_smem(reinterpret_cast<const void*>(vf_lsq_kernel<true>), bytes);
        FDS_LAUNCH(vf_lsq_kernel<true>, 1, kLsqThreads, bytes, st, m, n, in, rs, cs, rhs, nullptr, x_out, w_out,
                   wscale, status);
    } else {
        double* gwork = static_cast<double*>(VfContext::get().lsq.get(bytes));
        FDS_LAUNCH(vf_lsq_kernel<false>, 1, kLsqThreads, 0, st, m, n, in, rs, cs, rhs, gwork, x_out, w_out, wscale,
                   status);
    }
}

void vf_reloc_rms_launch(int K, int red, int M, int J, const double* r22, const double* beta, const double* tail,
                         const double* y, double* rms, cudaStream_t st) {
    FDS_LAUNCH(vf_reloc_rms_kernel, ceil_div(K, 4), 128, 0, st, K, red, M, J, r22, beta, tail, y, rms);
}

}  // namespace fdsb
