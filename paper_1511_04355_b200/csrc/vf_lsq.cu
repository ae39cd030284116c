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

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Solves the factored system for the right-hand side in b (length m) with one
// warp; b is overwritten; x (length n) receives the basic solution.
__device__ void lsq_solve_warp(const double* a, int m, int n, int np, const double* tau, const int* perm, double* b,
                               double* x, int lane) {
    for (int k = 0; k < np; ++k) {  // b <- Q^T b
        const double t = tau[k];
        if (t == 0.0) continue;
        const double* ess = a + static_cast<size_t>(k) * m + k;
        double d = 0.0;
        for (int i = 1 + lane; i < m - k; i += 32) d += ess[i] * b[k + i];
        d = (warp_sum(d) + b[k]) * t;
        __syncwarp();
        if (lane == 0) b[k] -= d;
        for (int i = 1 + lane; i < m - k; i += 32) b[k + i] -= d * ess[i];
        __syncwarp();
    }
    for (int i = np - 1; i >= 0; --i) {  // R11 z = (Q^T b)[0:np], column-oriented (no reductions)
        const double* col = a + static_cast<size_t>(i) * m;
        const double zi = b[i] / col[i];
        __syncwarp();
        if (lane == 0) b[i] = zi;
        for (int j = lane; j < i; j += 32) b[j] -= zi * col[j];
        __syncwarp();
    }
    for (int i = lane; i < n; i += 32) x[i] = 0.0;
    __syncwarp();
    for (int i = lane; i < np; i += 32) x[perm[i]] = b[i];
    __syncwarp();
}

}  // namespace

// in(i, j) = in[i*rs + j*cs]. Mode A (x_out != null): solve for rhs, x_out[n].
// Mode B (w_out != null): w_out[c*m + i] = wscale[c] * W(c, i) for the explicit
// solve operator. Working storage: dynamic shared memory, or gwork when the
// system does not fit (then dynamic smem is 0).
__global__ void __launch_bounds__(kLsqThreads)
vf_lsq_kernel(int m, int n, const double* __restrict__ in, long long rs, long long cs, const double* __restrict__ rhs,
              double* gwork, double* __restrict__ x_out, double* __restrict__ w_out,
              const double* __restrict__ wscale, VfLsqStatus* __restrict__ status) {
    extern __shared__ double lsm[];
    __shared__ int s_nonzero, s_rank;
    __shared__ double s_maxpivot, s_thr;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int size = min(m, n);
    double* base = gwork ? gwork : lsm;
    double* a = base;                               // m x n, column-major
    double* upd = a + static_cast<size_t>(m) * n;   // downdated column norms
    double* dir = upd + n;                          // norms at the last recompute
    double* tau = dir + n;
    double* vec = tau + n;                          // kLsqWarps x m solve vectors
    double* xs = vec + static_cast<size_t>(kLsqWarps) * m;  // kLsqWarps x n
    int* perm = reinterpret_cast<int*>(xs + static_cast<size_t>(kLsqWarps) * n);
    const double eps = DBL_EPSILON;

    for (size_t idx = tid; idx < static_cast<size_t>(m) * n; idx += kLsqThreads) {
        const int i = static_cast<int>(idx % m), j = static_cast<int>(idx / m);
        a[idx] = in[static_cast<long long>(i) * rs + static_cast<long long>(j) * cs];
    }
    for (int j = tid; j < n; j += kLsqThreads) perm[j] = j;
    __syncthreads();
    for (int j = warp; j < n; j += kLsqWarps) {
        double s = 0.0;
        for (int i = lane; i < m; i += 32) s += a[static_cast<size_t>(j) * m + i] * a[static_cast<size_t>(j) * m + i];
        s = warp_sum(s);
        if (lane == 0) upd[j] = dir[j] = sqrt(s);
    }
    __syncthreads();
    if (tid == 0) {
        double mx = 0.0;
        for (int j = 0; j < n; ++j) mx = fmax(mx, upd[j]);
        s_thr = (mx * eps) * (mx * eps) / m;
        s_nonzero = size;
        s_maxpivot = 0.0;
    }
    for (int k = 0; k < size; ++k) {
        __syncthreads();
        if (warp == 0) {
            // pivot: largest remaining norm, first maximum (warp argmax)
            double bv = -1.0;
            int bj = n;
            for (int j = k + lane; j < n; j += 32)
                if (upd[j] > bv) { bv = upd[j]; bj = j; }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
                if (ov > bv || (ov == bv && oj < bj)) { bv = ov; bj = oj; }
            }
            const int big = bj;
            if (lane == 0 && s_nonzero == size && upd[big] * upd[big] < s_thr * (m - k)) s_nonzero = k;
            if (big != k) {
                for (int i = lane; i < m; i += 32) {
                    const double t = a[static_cast<size_t>(k) * m + i];
                    a[static_cast<size_t>(k) * m + i] = a[static_cast<size_t>(big) * m + i];
                    a[static_cast<size_t>(big) * m + i] = t;
                }
                if (lane == 0) {
                    double t = upd[k]; upd[k] = upd[big]; upd[big] = t;
                    t = dir[k]; dir[k] = dir[big]; dir[big] = t;
                    const int p = perm[k]; perm[k] = perm[big]; perm[big] = p;
                }
                __syncwarp();
            }
            // Householder vector of column k, rows k..m-1
            double* x = a + static_cast<size_t>(k) * m + k;
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
                s_maxpivot = fmax(s_maxpivot, fabs(beta));
            }
        }
        __syncthreads();
        const double t = tau[k];
        const double* ess = a + static_cast<size_t>(k) * m + k;
        for (int j = k + 1 + warp; j < n; j += kLsqWarps) {  // apply H_k, downdate the norm
            double* col = a + static_cast<size_t>(j) * m + k;
            if (t != 0.0) {
                double d = 0.0;
                for (int i = 1 + lane; i < m - k; i += 32) d += ess[i] * col[i];
                d = (warp_sum(d) + col[0]) * t;
                __syncwarp();
                if (lane == 0) col[0] -= d;
                for (int i = 1 + lane; i < m - k; i += 32) col[i] -= d * ess[i];
                __syncwarp();
            }
            int recompute = 0;
            if (lane == 0 && upd[j] != 0.0) {
                double q = fabs(col[0]) / upd[j];
                q = (1.0 + q) * (1.0 - q);
                if (q < 0.0) q = 0.0;
                const double r = upd[j] / dir[j];
                if (q * r * r <= sqrt(eps)) recompute = 1;
                else upd[j] *= sqrt(q);
            }
            recompute = __shfl_sync(0xffffffffu, recompute, 0);
            if (recompute) {
                double s = 0.0;
                for (int i = 1 + lane; i < m - k; i += 32) s += col[i] * col[i];
                s = warp_sum(s);
                if (lane == 0) upd[j] = dir[j] = sqrt(s);
            }
        }
    }
    __syncthreads();
    if (tid == 0) {
        const double pre = fabs(s_maxpivot) * (size * eps);
        int r = 0;
        for (int i = 0; i < s_nonzero; ++i) r += fabs(a[static_cast<size_t>(i) * m + i]) > pre;
        s_rank = r;
        status->rank = r;
        status->nonzero = s_nonzero;
        status->maxpivot = s_maxpivot;
    }
    __syncthreads();
    if (s_rank < n) return;  // the caller raises NumericError; no solution is formed
    const int np = s_nonzero;
    double* b = vec + static_cast<size_t>(warp) * m;
    double* x = xs + static_cast<size_t>(warp) * n;
    if (x_out) {
        if (warp == 0) {
            for (int i = lane; i < m; i += 32) b[i] = rhs[i];
            __syncwarp();
            lsq_solve_warp(a, m, n, np, tau, perm, b, x, lane);
            for (int i = lane; i < n; i += 32) x_out[i] = x[i];
        }
        return;
    }
    for (int c = warp; c < m; c += kLsqWarps) {  // W e_c for every unit vector
        for (int i = lane; i < m; i += 32) b[i] = i == c ? 1.0 : 0.0;
        __syncwarp();
        lsq_solve_warp(a, m, n, np, tau, perm, b, x, lane);
        for (int i = lane; i < n; i += 32) w_out[static_cast<size_t>(i) * m + c] = wscale[i] * x[i];
        __syncwarp();
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

size_t vf_lsq_bytes(int m, int n) {
    return sizeof(double) * (static_cast<size_t>(m) * n + 3 * static_cast<size_t>(n) +
                             static_cast<size_t>(kLsqWarps) * (m + n) + (n + 1) / 2 + 1);
}

void vf_lsq_launch(int m, int n, const double* in, long long rs, long long cs, const double* rhs, double* x_out,
                   double* w_out, const double* wscale, VfLsqStatus* status, cudaStream_t st) {
    const size_t bytes = vf_lsq_bytes(m, n);
    double* gwork = nullptr;
    size_t smem = bytes;
    if (bytes > static_cast<size_t>(device_info().smem_optin) - 2048) {
        gwork = static_cast<double*>(VfContext::get().lsq.get(bytes));
        smem = 0;
    } else {
        ensure_dynamic_smem(reinterpret_cast<const void*>(vf_lsq_kernel), smem);
    }
    FDS_LAUNCH(vf_lsq_kernel, 1, kLsqThreads, smem, st, m, n, in, rs, cs, rhs, gwork, x_out, w_out, wscale, status);
}

void vf_reloc_rms_launch(int K, int red, int M, int J, const double* r22, const double* beta, const double* tail,
                         const double* y, double* rms, cudaStream_t st) {
    FDS_LAUNCH(vf_reloc_rms_kernel, ceil_div(K, 4), 128, 0, st, K, red, M, J, r22, beta, tail, y, rms);
}

}  // namespace fdsb
