// Restarted, right-preconditioned GMRES on a dense device-resident system.
//
//   gm_pinv_kernel       3x3 complex diagonal-block inverses (one per element):
//                        the block-Jacobi preconditioner M^{-1}.
//   gm_matvec_kernel     y = A x, planar column-major A: each CTA owns 512 rows
//                        (two per thread, 16-byte loads) x a 1024-column chunk
//                        (x chunk staged in smem, 8-column unroll so every thread
//                        keeps 16 coalesced 16-byte loads in flight); partial
//                        sums reduced over chunks in a fixed order
//                        (gm_chunk_reduce_kernel). HBM-bound: 16 n² bytes.
//   gm_dots_kernel       h_i = <V_i, w> for all Krylov vectors at once (fixed
//                        block partition + tree, so reductions are reproducible).
//   gm_axpy_kernel       w -= V h / x += V y style updates, thread per row.
//
// Classical Gram–Schmidt applied twice (CGS2) keeps the basis orthogonal to
// rounding; the small Hessenberg least-squares problem (Givens rotations) runs
// on the host.
#include <cmath>
#include <complex>
#include <vector>

#include "gmres.cuh"

namespace fdsb {

namespace {

constexpr int kMvThreads = 256, kMvRows = 2 * kMvThreads, kMvCols = 1024, kDotThreads = 256, kDotRows = 2048;

__global__ void gm_pinv_kernel(const double* __restrict__ Are, const double* __restrict__ Aim, int ne, int ld,
                               cplx* __restrict__ pinv) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= ne) return;
    cplx a[3][3], x[3][3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            const size_t gi = static_cast<size_t>(3 * e + j) * ld + 3 * e + i;
            a[i][j] = mk(Are[gi], Aim[gi]);
            x[i][j] = mk(i == j ? 1.0 : 0.0, 0.0);
        }
    // Gauss–Jordan with partial pivoting
    for (int c = 0; c < 3; ++c) {
        int p = c;
        for (int r = c + 1; r < 3; ++r)
            if (abs2(a[r][c]) > abs2(a[p][c])) p = r;
        if (p != c)
            for (int j = 0; j < 3; ++j) {
                const cplx t = a[c][j]; a[c][j] = a[p][j]; a[p][j] = t;
                const cplx u = x[c][j]; x[c][j] = x[p][j]; x[p][j] = u;
            }
        const cplx inv = crecip(a[c][c]);
        for (int j = 0; j < 3; ++j) {
            a[c][j] = a[c][j] * inv;
            x[c][j] = x[c][j] * inv;
        }
        for (int r = 0; r < 3; ++r) {
            if (r == c) continue;
            const cplx f = a[r][c];
            for (int j = 0; j < 3; ++j) {
                a[r][j] = a[r][j] - f * a[c][j];
                x[r][j] = x[r][j] - f * x[c][j];
            }
        }
    }
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) pinv[9 * static_cast<size_t>(e) + 3 * i + j] = x[i][j];
}

__global__ void gm_precond_kernel(const cplx* __restrict__ pinv, const cplx* __restrict__ x, int ne,
                                  cplx* __restrict__ z) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= ne) return;
    const cplx* P = pinv + 9 * static_cast<size_t>(e);
    const cplx x0 = x[3 * e], x1 = x[3 * e + 1], x2 = x[3 * e + 2];
    for (int i = 0; i < 3; ++i) z[3 * e + i] = P[3 * i] * x0 + P[3 * i + 1] * x1 + P[3 * i + 2] * x2;
}

// Each thread owns two adjacent rows (16-byte loads), so a warp streams 512
// contiguous bytes of a column per plane and a CTA 4 KB.
__global__ void __launch_bounds__(kMvThreads)
gm_matvec_kernel(const double* __restrict__ Are, const double* __restrict__ Aim, int n, int ld,
                 const cplx* __restrict__ x, cplx* __restrict__ partial) {
    __shared__ cplx xs[kMvCols];
    const int c0 = blockIdx.y * kMvCols, cn = min(kMvCols, n - c0);
    for (int q = threadIdx.x; q < cn; q += kMvThreads) xs[q] = x[c0 + q];
    __syncthreads();
    const int r = blockIdx.x * kMvRows + 2 * threadIdx.x;  // rows r, r+1 (ld is even, A is 16 B aligned)
    if (r >= n) return;
    const double* pr = Are + static_cast<size_t>(c0) * ld + r;
    const double* pi = Aim + static_cast<size_t>(c0) * ld + r;
    double s0r = 0.0, s0i = 0.0, s1r = 0.0, s1i = 0.0;
    int c = 0;
    for (; c + 8 <= cn; c += 8) {
        double2 ar[8], ai[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            ar[u] = __ldcs(reinterpret_cast<const double2*>(pr + static_cast<size_t>(c + u) * ld));
            ai[u] = __ldcs(reinterpret_cast<const double2*>(pi + static_cast<size_t>(c + u) * ld));
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const cplx v = xs[c + u];
            s0r += ar[u].x * v.re - ai[u].x * v.im;
            s0i += ar[u].x * v.im + ai[u].x * v.re;
            s1r += ar[u].y * v.re - ai[u].y * v.im;
            s1i += ar[u].y * v.im + ai[u].y * v.re;
        }
    }
    for (; c < cn; ++c) {
        const double2 ar = *reinterpret_cast<const double2*>(pr + static_cast<size_t>(c) * ld);
        const double2 ai = *reinterpret_cast<const double2*>(pi + static_cast<size_t>(c) * ld);
        const cplx v = xs[c];
        s0r += ar.x * v.re - ai.x * v.im;
        s0i += ar.x * v.im + ai.x * v.re;
        s1r += ar.y * v.re - ai.y * v.im;
        s1i += ar.y * v.im + ai.y * v.re;
    }
    cplx* out = partial + static_cast<size_t>(blockIdx.y) * n;
    out[r] = mk(s0r, s0i);
    if (r + 1 < n) out[r + 1] = mk(s1r, s1i);
}

// y = sum over chunks of partial (fixed order); optionally y = b - y.
__global__ void gm_chunk_reduce_kernel(const cplx* __restrict__ partial, int nchunk, int n,
                                       const cplx* __restrict__ b, cplx* __restrict__ y) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    cplx s = mk(0.0, 0.0);
    for (int q = 0; q < nchunk; ++q) s = s + partial[static_cast<size_t>(q) * n + r];
    y[r] = b ? b[r] - s : s;
}

// partial[blk][i] = sum over the block's rows of conj(V_i[r]) w[r], i < cnt.
__global__ void __launch_bounds__(kDotThreads)
gm_dots_kernel(const cplx* __restrict__ V, int n, int cnt, const cplx* __restrict__ w, cplx* __restrict__ partial) {
    __shared__ cplx red[kDotThreads];
    const int r0 = blockIdx.x * kDotRows;
    const int r1 = min(n, r0 + kDotRows);
    for (int i = 0; i < cnt; ++i) {
        const cplx* vi = V + static_cast<size_t>(i) * n;
        cplx s = mk(0.0, 0.0);
        for (int r = r0 + threadIdx.x; r < r1; r += kDotThreads) s = s + conjg(vi[r]) * w[r];
        red[threadIdx.x] = s;
        __syncthreads();
        for (int h = kDotThreads / 2; h > 0; h >>= 1) {
            if (threadIdx.x < h) red[threadIdx.x] = red[threadIdx.x] + red[threadIdx.x + h];
            __syncthreads();
        }
        if (threadIdx.x == 0) partial[static_cast<size_t>(blockIdx.x) * cnt + i] = red[0];
        __syncthreads();
    }
}

__global__ void gm_dots_reduce_kernel(const cplx* __restrict__ partial, int nblk, int cnt, cplx* __restrict__ h) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cnt) return;
    cplx s = mk(0.0, 0.0);
    for (int q = 0; q < nblk; ++q) s = s + partial[static_cast<size_t>(q) * cnt + i];
    h[i] = s;
}

// y[r] = alpha * y[r] + sign * sum_{i<cnt} V_i[r] c_i   (c in device memory)
__global__ void gm_axpy_kernel(const cplx* __restrict__ V, int n, int cnt, const cplx* __restrict__ c, double sign,
                               double alpha, cplx* __restrict__ y) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    cplx s = mk(0.0, 0.0);
    for (int i = 0; i < cnt; ++i) s = s + V[static_cast<size_t>(i) * n + r] * c[i];
    y[r] = y[r] * alpha + s * sign;
}

__global__ void gm_scale_kernel(const cplx* __restrict__ x, int n, double s, cplx* __restrict__ y) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) y[r] = x[r] * s;
}

using Cx = std::complex<double>;

struct Ops {
    const double *Are, *Aim;
    int n, ld;
    GmresWorkspace& ws;
    cudaStream_t st;
    cplx* partial() const { return reinterpret_cast<cplx*>(ws.partial); }
    int nchunk() const { return ceil_div(n, kMvCols); }
    // y = A x  (or y = b - A x)
    void matvec(const cplx* x, cplx* y, const cplx* b = nullptr) const {
        dim3 g(ceil_div(n, kMvRows), nchunk());
        FDS_LAUNCH(gm_matvec_kernel, g, kMvThreads, 0, st, Are, Aim, n, ld, x, partial());
        FDS_LAUNCH(gm_chunk_reduce_kernel, ceil_div(n, 256), 256, 0, st, partial(), nchunk(), n, b, y);
    }
    void precond(const cplx* x, cplx* z) const {
        FDS_LAUNCH(gm_precond_kernel, ceil_div(n / 3, 128), 128, 0, st, reinterpret_cast<const cplx*>(ws.pinv), x,
                   n / 3, z);
    }
    // h[0..cnt) = V^H w, copied to the host
    void dots(const cplx* V, int cnt, const cplx* w, std::vector<Cx>& h) const {
        const int nblk = ceil_div(n, kDotRows);
        cplx* hd = reinterpret_cast<cplx*>(ws.h_dev);
        FDS_LAUNCH(gm_dots_kernel, nblk, kDotThreads, 0, st, V, n, cnt, w, partial());
        FDS_LAUNCH(gm_dots_reduce_kernel, ceil_div(cnt, 64), 64, 0, st, partial(), nblk, cnt, hd);
        h.resize(cnt);
        FDS_CUDA(cudaMemcpyAsync(h.data(), hd, cnt * sizeof(cplx), cudaMemcpyDeviceToHost, st));
        FDS_CUDA(cudaStreamSynchronize(st));
    }
    void axpy(const cplx* V, int cnt, const std::vector<Cx>& c, double sign, double alpha, cplx* y) const {
        cplx* hd = reinterpret_cast<cplx*>(ws.h_dev);
        FDS_CUDA(cudaMemcpyAsync(hd, c.data(), cnt * sizeof(cplx), cudaMemcpyHostToDevice, st));
        FDS_LAUNCH(gm_axpy_kernel, ceil_div(n, 256), 256, 0, st, V, n, cnt, hd, sign, alpha, y);
    }
    double norm(const cplx* w) const {
        std::vector<Cx> h;
        dots(w, 1, w, h);
        return std::sqrt(std::max(h[0].real(), 0.0));
    }
};

}  // namespace

void GmresWorkspace::ensure(int n, int m) {
    if (static_cast<size_t>(n) <= n_cap && m <= m_cap) return;
    release();
    const size_t nc = static_cast<size_t>(n);
    const size_t nchunk = (nc + kMvCols - 1) / kMvCols;
    FDS_CUDA(cudaMalloc(&V, 2 * nc * (m + 1) * sizeof(double)));
    FDS_CUDA(cudaMalloc(&w, 2 * nc * sizeof(double)));
    FDS_CUDA(cudaMalloc(&z, 2 * nc * sizeof(double)));
    FDS_CUDA(cudaMalloc(&pinv, 2 * 3 * nc * sizeof(double)));
    const size_t nblk = (nc + kDotRows - 1) / kDotRows;
    FDS_CUDA(cudaMalloc(&partial, 2 * std::max(nchunk * nc, nblk * (m + 2)) * sizeof(double)));
    FDS_CUDA(cudaMalloc(&h_dev, 2 * (m + 2) * sizeof(double)));
    FDS_CUDA(cudaMalloc(&bsave, 2 * nc * sizeof(double)));
    n_cap = nc;
    m_cap = m;
}

void GmresWorkspace::release() {
    for (double* p : {V, w, z, pinv, partial, h_dev, bsave})
        if (p) cudaFree(p);
    V = w = z = pinv = partial = h_dev = bsave = nullptr;
    n_cap = 0;
    m_cap = 0;
}

GmresStats gmres_solve(const double* Are, const double* Aim, int n, int ld, cplx* b, const GmresParams& p,
                       GmresWorkspace& ws, cudaStream_t st) {
    if (n % 3 != 0) throw ValidationError("gmres: n must be a multiple of 3 (element-major DOFs)");
    const int m = std::max(1, p.restart);
    ws.ensure(n, m);
    Ops op{Are, Aim, n, ld, ws, st};
    cplx* V = reinterpret_cast<cplx*>(ws.V);
    cplx* w = reinterpret_cast<cplx*>(ws.w);
    cplx* z = reinterpret_cast<cplx*>(ws.z);
    cplx* bsave = reinterpret_cast<cplx*>(ws.bsave);
    auto col = [&](int i) { return V + static_cast<size_t>(i) * n; };
    FDS_LAUNCH(gm_pinv_kernel, ceil_div(n / 3, 128), 128, 0, st, Are, Aim, n / 3, ld, reinterpret_cast<cplx*>(ws.pinv));
    // keep the right-hand side; x accumulates in b's buffer from x = 0, and r = b - A x = b
    FDS_CUDA(cudaMemcpyAsync(bsave, b, n * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
    FDS_CUDA(cudaMemcpyAsync(w, b, n * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
    FDS_CUDA(cudaMemsetAsync(b, 0, n * sizeof(cplx), st));
    const double bnorm = op.norm(w);
    GmresStats stats;
    if (bnorm == 0.0) return stats;  // x = 0
    double beta = bnorm;
    std::vector<Cx> H(static_cast<size_t>(m + 1) * m), cs(m), sn(m), g(m + 1), h, h2;
    while (true) {
        if (beta / bnorm <= p.tol || stats.iterations >= p.max_iter) break;
        FDS_LAUNCH(gm_scale_kernel, ceil_div(n, 256), 256, 0, st, w, n, 1.0 / beta, col(0));
        std::fill(g.begin(), g.end(), Cx(0.0, 0.0));
        g[0] = beta;
        int j = 0;
        for (; j < m && stats.iterations < p.max_iter; ++j) {
            op.precond(col(j), z);
            op.matvec(z, w);
            op.dots(V, j + 1, w, h);  // CGS, twice
            op.axpy(V, j + 1, h, -1.0, 1.0, w);
            op.dots(V, j + 1, w, h2);
            op.axpy(V, j + 1, h2, -1.0, 1.0, w);
            for (int i = 0; i <= j; ++i) H[static_cast<size_t>(i) * m + j] = h[i] + h2[i];
            const double hn = op.norm(w);
            H[static_cast<size_t>(j + 1) * m + j] = hn;
            // previous rotations, then a new one zeroing H[j+1][j]
            for (int i = 0; i < j; ++i) {
                const Cx a = H[static_cast<size_t>(i) * m + j], bb = H[static_cast<size_t>(i + 1) * m + j];
                H[static_cast<size_t>(i) * m + j] = std::conj(cs[i]) * a + std::conj(sn[i]) * bb;
                H[static_cast<size_t>(i + 1) * m + j] = -sn[i] * a + cs[i] * bb;
            }
            const Cx a = H[static_cast<size_t>(j) * m + j], bb = H[static_cast<size_t>(j + 1) * m + j];
            const double den = std::sqrt(std::norm(a) + std::norm(bb));
            if (den == 0.0) throw NumericError("gmres: breakdown (zero Krylov column)");
            cs[j] = a / den;
            sn[j] = bb / den;
            H[static_cast<size_t>(j) * m + j] = den;
            H[static_cast<size_t>(j + 1) * m + j] = 0.0;
            g[j + 1] = -sn[j] * g[j];
            g[j] = std::conj(cs[j]) * g[j];
            ++stats.iterations;
            if (hn > 0.0) FDS_LAUNCH(gm_scale_kernel, ceil_div(n, 256), 256, 0, st, w, n, 1.0 / hn, col(j + 1));
            if (std::abs(g[j + 1]) / bnorm <= p.tol || hn == 0.0) {
                ++j;
                break;
            }
        }
        // y = H^{-1} g (upper triangular j x j); x += M^{-1} V y
        std::vector<Cx> y(j);
        for (int i = j - 1; i >= 0; --i) {
            Cx s = g[i];
            for (int q = i + 1; q < j; ++q) s -= H[static_cast<size_t>(i) * m + q] * y[q];
            y[i] = s / H[static_cast<size_t>(i) * m + i];
        }
        op.axpy(V, j, y, 1.0, 0.0, w);  // w = V y
        op.precond(w, z);
        op.axpy(z, 1, std::vector<Cx>{Cx(1.0, 0.0)}, 1.0, 1.0, b);  // x += M^{-1} V y
        op.matvec(b, w, bsave);                                     // true residual r = b - A x
        beta = op.norm(w);
    }
    stats.rel_residual = beta / bnorm;
    if (!(stats.rel_residual <= p.tol))
        throw ConvergenceError("gmres: relative residual " + std::to_string(stats.rel_residual) + " after " +
                               std::to_string(stats.iterations) + " iterations");
    return stats;
}

}  // namespace fdsb
