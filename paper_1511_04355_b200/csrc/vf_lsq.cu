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
    int m, n, lda, bcols;  // bcols: right-hand sides held at once (1 for a single solve)
    __host__ __device__ size_t a_doubles() const { return static_cast<size_t>(lda) * n; }
    __host__ __device__ size_t b_doubles() const { return static_cast<size_t>(m) * bcols; }
    __host__ __device__ size_t total_doubles() const { return a_doubles() + 4 * static_cast<size_t>(n) + b_doubles() + (n + 1) / 2 + 2; }
};

}  // namespace

// Solves with the factored system, one thread per right-hand side (kLsqCols at a
// time): b <- Q^T b by broadcast reads of each reflector, then column-oriented
// back substitution with the reciprocal diagonal; no reductions.
__device__ void lsq_solves(const double* a, int lda, const double* tau, const double* rdiag, const int* perm,
                           double* bb, int bcols, int m, int n, int np, const double* __restrict__ rhs,
                           double* __restrict__ x_out, double* __restrict__ w_out, const double* __restrict__ wscale,
                           int tid) {
    const int nrhs = x_out ? 1 : m;
    for (int c0 = 0; c0 < nrhs; c0 += bcols) {
        const int c = c0 + tid;
        const bool mine = tid < bcols && c < nrhs;
        if (mine)
            for (int i = 0; i < m; ++i) bb[static_cast<size_t>(i) * bcols + tid] = x_out ? rhs[i] : (i == c ? 1.0 : 0.0);
        if (mine) {
            double* b = bb + tid;  // this thread's column, stride bcols
            for (int k = 0; k < np; ++k) {  // b <- Q^T b
                const double t = tau[k];
                if (t == 0.0) continue;
                const double* ess = a + static_cast<size_t>(k) * lda + k;
                double d0 = b[static_cast<size_t>(k) * bcols], d1 = 0.0;
                int i = 1;
                for (; i + 1 < m - k; i += 2) {
                    d0 += ess[i] * b[static_cast<size_t>(k + i) * bcols];
                    d1 += ess[i + 1] * b[static_cast<size_t>(k + i + 1) * bcols];
                }
                if (i < m - k) d0 += ess[i] * b[static_cast<size_t>(k + i) * bcols];
                const double d = (d0 + d1) * t;
                b[static_cast<size_t>(k) * bcols] -= d;
                for (int r = 1; r < m - k; ++r) b[static_cast<size_t>(k + r) * bcols] -= d * ess[r];
            }
            for (int i = np - 1; i >= 0; --i) {  // R11 z = (Q^T b)[0:np], column-oriented
                const double* col = a + static_cast<size_t>(i) * lda;
                const double zi = b[static_cast<size_t>(i) * bcols] * rdiag[i];
                b[static_cast<size_t>(i) * bcols] = zi;
                for (int j = 0; j < i; ++j) b[static_cast<size_t>(j) * bcols] -= zi * col[j];
            }
            if (x_out) {
                for (int i = 0; i < n; ++i) x_out[i] = 0.0;
                for (int i = 0; i < np; ++i) x_out[perm[i]] = b[static_cast<size_t>(i) * bcols];
            } else {
                for (int i = 0; i < n; ++i) w_out[static_cast<size_t>(i) * m + c] = 0.0;
                for (int i = 0; i < np; ++i)
                    w_out[static_cast<size_t>(perm[i]) * m + c] = wscale[perm[i]] * b[static_cast<size_t>(i) * bcols];
            }
        }
    }
}

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
    const LsqLayout L{m, n, m | 1, x_out ? 1 : kLsqCols};
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
    lsq_solves(a, lda, tau, rdiag, perm, bb, L.bcols, m, n, s_nonzero, rhs, x_out, w_out, wscale, tid);
}

// Systems with n <= 64 columns (every VF system of the bench and the AFS
// loop): the factorization runs on warp 0 alone, lane j owning columns j and
// j + 32 — each Householder step is then a handful of __syncwarp()s (pivot by
// warp argmax, reflector by one lane, trailing update and norm downdate by the
// owning lanes with no reductions) instead of two CTA barriers; the solves run
// on all 128 threads as in vf_lsq_kernel. Same decisions as vf_lsq_kernel.
constexpr int kLsqSmallThreads = 128;
__global__ void __launch_bounds__(kLsqSmallThreads)
vf_lsq_small_kernel(int m, int n, int m_thr, const double* __restrict__ in, long long rs, long long cs,
                    const double* __restrict__ rhs, double* __restrict__ x_out, double* __restrict__ w_out,
                    const double* __restrict__ wscale, VfLsqStatus* __restrict__ status,
                    double* __restrict__ fact_out, int* __restrict__ perm_out) {
    extern __shared__ double lsm[];
    __shared__ int s_nonzero, s_rank;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int size = min(m, n);
    const LsqLayout L{m, n, m | 1, (x_out || fact_out) ? 1 : kLsqCols};
    const int lda = L.lda;
    double* a = lsm;
    double* upd = a + L.a_doubles();
    double* dir = upd + n;
    double* tau = dir + n;
    double* rdiag = tau + n;
    double* bb = rdiag + n;
    int* perm = reinterpret_cast<int*>(bb + L.b_doubles());
    for (size_t idx = tid; idx < static_cast<size_t>(m) * n; idx += kLsqSmallThreads) {
        const int i = static_cast<int>(idx % m), j = static_cast<int>(idx / m);
        a[static_cast<size_t>(j) * lda + i] = in[static_cast<long long>(i) * rs + static_cast<long long>(j) * cs];
    }
    for (int j = tid; j < n; j += kLsqSmallThreads) perm[j] = j;
    __syncthreads();
    if (warp == 0) {
        // column norms: lane-owned columns, sequential over rows
        double mx = 0.0;
        for (int j = lane; j < n; j += 32) {
            const double* col = a + static_cast<size_t>(j) * lda;
            double s0 = 0.0, s1 = 0.0;
            int i = 0;
            for (; i + 1 < m; i += 2) { s0 += col[i] * col[i]; s1 += col[i + 1] * col[i + 1]; }
            if (i < m) s0 += col[i] * col[i];
            upd[j] = dir[j] = sqrt(s0 + s1);
        }
        __syncwarp();
        for (int j = 0; j < n; ++j) mx = fmax(mx, upd[j]);  // every lane: same order, same value
        // m_thr: the row count of the system before any row reduction (Eigen's
        // thresholds use the rows of the matrix it factors, vecfit.cpp:281)
        const double thr = (mx * DBL_EPSILON) * (mx * DBL_EPSILON) / m_thr;
        int nonzero = size;
        double maxpivot = 0.0;
        for (int k = 0; k < size; ++k) {
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
            if (nonzero == size && bv * bv < thr * (m_thr - k)) nonzero = k;
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
            }
            maxpivot = fmax(maxpivot, fabs(beta));
            __syncwarp();
            // trailing columns: lane j owns column j (and j + 32)
            for (int j = k + 1 + lane; j < n; j += 32) {
                double* col = a + static_cast<size_t>(j) * lda + k;
                double cv = col[0];
                if (t != 0.0) {
                    double d0 = cv, d1 = 0.0;
                    int i = 1;
                    for (; i + 1 < len; i += 2) { d0 += x[i] * col[i]; d1 += x[i + 1] * col[i + 1]; }
                    if (i < len) d0 += x[i] * col[i];
                    const double d = (d0 + d1) * t;
                    for (int r = 1; r < len; ++r) col[r] -= d * x[r];
                    cv -= d;
                    col[0] = cv;
                }
                const double u = upd[j];
                if (u != 0.0) {
                    double q = fabs(cv) / u;
                    q = (1.0 + q) * (1.0 - q);
                    if (q < 0.0) q = 0.0;
                    const double r = u / dir[j];
                    if (q * r * r <= kSqrtEps) {
                        double s0 = 0.0, s1 = 0.0;
                        int i = 1;
                        for (; i + 1 < len; i += 2) { s0 += col[i] * col[i]; s1 += col[i + 1] * col[i + 1]; }
                        if (i < len) s0 += col[i] * col[i];
                        upd[j] = dir[j] = sqrt(s0 + s1);
                    } else {
                        upd[j] = u * sqrt(q);
                    }
                }
            }
            __syncwarp();
        }
        if (lane == 0) {
            const double pre = fabs(maxpivot) * (min(m_thr, n) * DBL_EPSILON);
            int r = 0;
            for (int i = 0; i < nonzero; ++i) r += fabs(a[static_cast<size_t>(i) * lda + i]) > pre;
            s_rank = r;
            s_nonzero = nonzero;
            status->rank = r;
            status->nonzero = nonzero;
            status->maxpivot = maxpivot;
        }
    }
    __syncthreads();
    if (fact_out) {  // factorization only: R (upper triangle, lda = m | 1 columns of n) and the permutation
        for (size_t idx = tid; idx < static_cast<size_t>(n) * n; idx += kLsqSmallThreads) {
            const int r = static_cast<int>(idx % n), c = static_cast<int>(idx / n);
            fact_out[idx] = r <= c ? a[static_cast<size_t>(c) * lda + r] : 0.0;
        }
        for (int j2 = tid; j2 < n; j2 += kLsqSmallThreads) perm_out[j2] = perm[j2];
        return;
    }
    if (s_rank < n) return;  // the caller raises NumericError; no solution is formed
    lsq_solves(a, lda, tau, rdiag, perm, bb, L.bcols, m, n, s_nonzero, rhs, x_out, w_out, wscale, tid);
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

// Row reduction of the stacked sigma system: the K channel blocks [R22_k | beta_k]
// (red x M upper-triangular, vecfit.cpp:265-279) are folded pairwise into one
// M x (M+1) triangular system by unpivoted Householder steps in shared memory
// (only row blocks of 2 * red rows are ever resident). Column pivoting on the
// folded R makes the same choices as on the stacked matrix up to rounding (the
// column norms and Gram matrix are invariant under the orthogonal folding), so
// the pivoted factorization then runs on an M x M system that fits on chip.
constexpr int kFoldThreads = 512;
// Generic form: the m x n system in(i, j) = in[i*rs + j*cs] (with an optional
// right-hand side as column n) is folded in chunks of `chunk` rows; chunks
// already upper-triangular (the R22 blocks) skip their first reduction.
__global__ void __launch_bounds__(kFoldThreads)
vf_fold_kernel(int m, int n, const double* __restrict__ in, long long rs, long long cs,
               const double* __restrict__ rhs, int chunk, int first_triangular, double* __restrict__ out) {
    extern __shared__ double fsm_[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = kFoldThreads / 32;
    const int cols = n + (rhs ? 1 : 0);
    const int lda = (n + chunk) | 1;
    double* z = fsm_;  // lda x cols, column-major
    __shared__ double s_tau;
    int cur = 0;
    for (int r0 = 0; r0 < m; r0 += chunk) {
        const int rows = min(chunk, m - r0);
        __syncthreads();
        for (int idx = tid; idx < rows * cols; idx += kFoldThreads) {
            const int i = idx % rows, c = idx / rows;
            const long long row = r0 + i;
            z[static_cast<size_t>(c) * lda + cur + i] =
                c < n ? in[row * rs + static_cast<long long>(c) * cs] : rhs[row];
        }
        const int total = cur + rows;
        const int steps = (r0 == 0 && first_triangular) ? 0 : min(total, n);
        for (int c = 0; c < steps; ++c) {
            __syncthreads();
            if (warp == 0) {
                double* x = z + static_cast<size_t>(c) * lda + c;
                const int len = total - c;
                double tail = 0.0;
                for (int i = 1 + lane; i < len; i += 32) tail += x[i] * x[i];
                tail = warp_sum(tail);
                const double c0 = x[0];
                double t = 0.0, beta_h = c0;
                if (tail > DBL_MIN) {
                    beta_h = sqrt(c0 * c0 + tail);
                    if (c0 >= 0.0) beta_h = -beta_h;
                    const double inv = 1.0 / (c0 - beta_h);
                    for (int i = 1 + lane; i < len; i += 32) x[i] *= inv;
                    t = (beta_h - c0) / beta_h;
                } else {
                    for (int i = 1 + lane; i < len; i += 32) x[i] = 0.0;
                }
                __syncwarp();
                if (lane == 0) {
                    x[0] = beta_h;
                    s_tau = t;
                }
            }
            __syncthreads();
            const double t = s_tau;
            if (t == 0.0) continue;
            const double* v = z + static_cast<size_t>(c) * lda + c;
            for (int j = c + 1 + warp; j < cols; j += NW) {
                double* col = z + static_cast<size_t>(j) * lda + c;
                double d = 0.0;
                for (int i = 1 + lane; i < total - c; i += 32) d += v[i] * col[i];
                d = (warp_sum(d) + col[0]) * t;
                __syncwarp();
                if (lane == 0) col[0] -= d;
                for (int i = 1 + lane; i < total - c; i += 32) col[i] -= d * v[i];
            }
        }
        __syncthreads();
        // keep the triangle: rows below min(total, n) only carry the residual
        const int keep = min(total, n);
        for (int idx = tid; idx < keep * n; idx += kFoldThreads) {
            const int i = idx % keep, c = idx / keep;
            if (i > c) z[static_cast<size_t>(c) * lda + i] = 0.0;  // reflector storage -> R's zeros
        }
        cur = keep;
    }
    __syncthreads();
    for (int idx = tid; idx < n * cols; idx += kFoldThreads) {  // n x cols, zero rows past cur
        const int i = idx % n, c = idx / n;
        out[static_cast<size_t>(c) * n + i] = i < cur ? z[static_cast<size_t>(c) * lda + i] : 0.0;
    }
}

// W = P R^{-1} R^{-T} P^T A^T for systems too large for one CTA's shared
// memory (2J x M beyond ~220 KB): R is the pivoted-QR factor of the folded A
// (so R^T R = P^T A^T A P). One thread per row a_i of A: forward substitution
// y = R^{-T} (P^T a_i), back substitution z = R^{-1} y, W[perm[j]][i] =
// wscale[perm[j]] z_j; the thread's y/z live in shared memory ([n][128]), R is
// read by all threads at once (broadcast) from L2.
constexpr int kWThreads = 128;
__global__ void __launch_bounds__(kWThreads)
vf_w_sne_kernel(int m, int n, const double* __restrict__ a /*col-major m x n*/, const double* __restrict__ R,
                const int* __restrict__ perm, const double* __restrict__ wscale, double* __restrict__ w_out) {
    extern __shared__ double wsm_[];
    const int t = threadIdx.x, i = blockIdx.x * kWThreads + t;
    if (i >= m) return;
    double* y = wsm_ + t;  // y[j * kWThreads]
    for (int j = 0; j < n; ++j) {  // R^T y = P^T a_i (R upper: column j of R holds R[0..j][j])
        double v = a[static_cast<size_t>(perm[j]) * m + i];
        for (int l = 0; l < j; ++l) v -= R[static_cast<size_t>(j) * n + l] * y[l * kWThreads];
        y[j * kWThreads] = v / R[static_cast<size_t>(j) * n + j];
    }
    for (int j = n - 1; j >= 0; --j) {  // R z = y
        double v = y[j * kWThreads];
        for (int l = j + 1; l < n; ++l) v -= R[static_cast<size_t>(l) * n + j] * y[l * kWThreads];
        y[j * kWThreads] = v / R[static_cast<size_t>(j) * n + j];
    }
    for (int j = 0; j < n; ++j) w_out[static_cast<size_t>(perm[j]) * m + i] = wscale[perm[j]] * y[j * kWThreads];
}

void vf_lsq_launch(int m, int n, const double* in, long long rs, long long cs, const double* rhs, double* x_out,
                   double* w_out, const double* wscale, VfLsqStatus* status, cudaStream_t st, int m_thr) {
    if (m_thr <= 0) m_thr = m;
    const LsqLayout L{m, n, m | 1, x_out ? 1 : kLsqCols};
    const size_t bytes = L.total_doubles() * sizeof(double);
    if (n <= 128 && bytes <= static_cast<size_t>(device_info().smem_optin) - 2048) {
        ensure_dynamic_smem(reinterpret_cast<const void*>(vf_lsq_small_kernel), bytes);
        FDS_LAUNCH(vf_lsq_small_kernel, 1, kLsqSmallThreads, bytes, st, m, n, m_thr, in, rs, cs, rhs, x_out, w_out,
                   wscale, status, nullptr, nullptr);
    } else if (m_thr != m) {
        throw CudaError("vf_lsq: reduced system does not fit on chip");
    } else if (bytes <= static_cast<size_t>(device_info().smem_optin) - 2048) {
        ensure_dynamic_smem(reinterpret_cast<const void*>(vf_lsq_kernel<true>), bytes);
        FDS_LAUNCH(vf_lsq_kernel<true>, 1, kLsqThreads, bytes, st, m, n, in, rs, cs, rhs, nullptr, x_out, w_out,
                   wscale, status);
    } else {
        double* gwork = static_cast<double*>(VfContext::get().lsq.get(bytes));
        FDS_LAUNCH(vf_lsq_kernel<false>, 1, kLsqThreads, 0, st, m, n, in, rs, cs, rhs, gwork, x_out, w_out, wscale,
                   status);
    }
}

void vf_lsq_stacked_launch(int K, int red, int M, const double* r22, const double* beta, double* y,
                           VfLsqStatus* status, cudaStream_t st) {
    const int m = K * red;
    const LsqLayout L{m, M, m | 1, 1};
    const size_t direct = L.total_doubles() * sizeof(double);
    const size_t optin = static_cast<size_t>(device_info().smem_optin) - 2048;
    const size_t fold = static_cast<size_t>((M + red) | 1) * (M + 1) * sizeof(double);
    if ((M <= 128 && direct <= optin) || K == 1 || fold > optin || M > 128) {
        vf_lsq_launch(m, M, r22, M, 1, beta, y, nullptr, nullptr, status, st);
        return;
    }
    auto& cx = VfContext::get();
    double* z = static_cast<double*>(cx.lsq.get(sizeof(double) * static_cast<size_t>(M) * (M + 1)));
    ensure_dynamic_smem(reinterpret_cast<const void*>(vf_fold_kernel), fold);
    FDS_LAUNCH(vf_fold_kernel, 1, kFoldThreads, fold, st, m, M, r22, M, 1, beta, red, 1, z);
    // the folded M x M system keeps Eigen's thresholds of the K red-row original
    vf_lsq_launch(M, M, z, 1, M, z + static_cast<size_t>(M) * M, y, nullptr, nullptr, status, st, m);
}

bool vf_lsq_fits(int m, int n, bool single_rhs) {
    const LsqLayout L{m, n, m | 1, single_rhs ? 1 : kLsqCols};
    return L.total_doubles() * sizeof(double) <= static_cast<size_t>(device_info().smem_optin) - 2048;
}

void vf_lsq_operator_large(int m, int n, const double* a, const double* wscale, double* w_out, VfLsqStatus* status,
                           cudaStream_t st) {
    const size_t optin = static_cast<size_t>(device_info().smem_optin) - 2048;
    const int chunk = n;
    const size_t fold = static_cast<size_t>((n + chunk) | 1) * n * sizeof(double);
    if (n > 128 || fold > optin) {  // beyond the folded path: one CTA over global memory
        vf_lsq_launch(m, n, a, 1, m, nullptr, nullptr, w_out, wscale, status, st);
        return;
    }
    auto& cx = VfContext::get();
    double* z = static_cast<double*>(cx.lsq.get(sizeof(double) * (2 * static_cast<size_t>(n) * n + n)));
    double* R = z + static_cast<size_t>(n) * n;
    int* perm = reinterpret_cast<int*>(R + static_cast<size_t>(n) * n);
    ensure_dynamic_smem(reinterpret_cast<const void*>(vf_fold_kernel), fold);
    FDS_LAUNCH(vf_fold_kernel, 1, kFoldThreads, fold, st, m, n, a, 1, m, nullptr, chunk, 0, z);
    const LsqLayout L{n, n, n | 1, 1};
    const size_t bytes = L.total_doubles() * sizeof(double);
    ensure_dynamic_smem(reinterpret_cast<const void*>(vf_lsq_small_kernel), bytes);
    FDS_LAUNCH(vf_lsq_small_kernel, 1, kLsqSmallThreads, bytes, st, n, n, m, z, 1, n, nullptr, nullptr, nullptr,
               nullptr, status, R, perm);
    const size_t wsmem = static_cast<size_t>(n) * kWThreads * sizeof(double);
    ensure_dynamic_smem(reinterpret_cast<const void*>(vf_w_sne_kernel), wsmem);
    FDS_LAUNCH(vf_w_sne_kernel, ceil_div(m, kWThreads), kWThreads, wsmem, st, m, n, a, R, perm, wscale, w_out);
}

void vf_reloc_rms_launch(int K, int red, int M, int J, const double* r22, const double* beta, const double* tail,
                         const double* y, double* rms, cudaStream_t st) {
    FDS_LAUNCH(vf_reloc_rms_kernel, ceil_div(K, 4), 128, 0, st, K, red, M, J, r22, beta, tail, y, rms);
}

}  // namespace fdsb
