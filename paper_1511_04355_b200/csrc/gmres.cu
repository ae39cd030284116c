// Restarted, right-preconditioned GMRES on dense device-resident systems, run
// for a batch of independent systems in lockstep (one launch per operation for
// every still-active system, one host round trip per Arnoldi step).
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
// Classical Gram–Schmidt applied twice (CGS2) keeps each basis orthogonal to
// rounding; the small Hessenberg least-squares problems (Givens rotations) run
// on the host. A system leaves the Arnoldi loop when its own residual estimate
// reaches tol, so converged systems stop costing matrix-vector products.
#include <algorithm>
#include <cmath>
#include <complex>
#include <vector>

#include "gmres.cuh"

namespace fdsb {

namespace {

constexpr int kMvThreads = 256, kMvRows = 2 * kMvThreads, kMvCols = 1024, kDotThreads = 256, kDotRows = 2048;

// per-system vector: system b at base + b * stride (+ off)
struct SysVec {
    cplx* base;
    size_t stride;
    __host__ __device__ cplx* at(int b, size_t off = 0) const { return base + b * stride + off; }
};

__global__ void gm_pinv_kernel(const double* __restrict__ A, size_t mstride, size_t plane, int ne, int ld,
                               cplx* __restrict__ pinv) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    if (e >= ne) return;
    const double* Are = A + b * mstride;
    const double* Aim = Are + plane;
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
    cplx* P = pinv + (static_cast<size_t>(b) * ne + e) * 9;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) P[3 * i + j] = x[i][j];
}

__global__ void gm_precond_kernel(const cplx* __restrict__ pinv, int ne, const int* __restrict__ act, SysVec x,
                                  size_t xoff, SysVec z) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= ne) return;
    const int b = act[blockIdx.y];
    const cplx* P = pinv + (static_cast<size_t>(b) * ne + e) * 9;
    const cplx* xb = x.at(b, xoff);
    cplx* zb = z.at(b);
    const cplx x0 = xb[3 * e], x1 = xb[3 * e + 1], x2 = xb[3 * e + 2];
    for (int i = 0; i < 3; ++i) zb[3 * e + i] = P[3 * i] * x0 + P[3 * i + 1] * x1 + P[3 * i + 2] * x2;
}

// Each thread owns two adjacent rows (16-byte loads), so a warp streams 512
// contiguous bytes of a column per plane and a CTA 4 KB.
__global__ void __launch_bounds__(kMvThreads, 4)
gm_matvec_kernel(const double* __restrict__ A, size_t mstride, size_t plane, int n, int ld,
                 const int* __restrict__ act, SysVec xv, cplx* __restrict__ partial, int nchunk) {
    __shared__ cplx xs[kMvCols];
    const int a = blockIdx.z, b = act[a];
    const double* Are = A + b * mstride;
    const double* Aim = Are + plane;
    const cplx* x = xv.at(b);
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
    cplx* out = partial + (static_cast<size_t>(a) * nchunk + blockIdx.y) * n;
    out[r] = mk(s0r, s0i);
    if (r + 1 < n) out[r + 1] = mk(s1r, s1i);
}

// y_b = sum over chunks (fixed order); with rhs: y_b = rhs_b - sum.
__global__ void gm_chunk_reduce_kernel(const cplx* __restrict__ partial, int nchunk, int n,
                                       const int* __restrict__ act, SysVec rhs, bool with_rhs, SysVec y) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int a = blockIdx.y, b = act[a];
    const cplx* p = partial + static_cast<size_t>(a) * nchunk * n;
    cplx s = mk(0.0, 0.0);
    for (int q = 0; q < nchunk; ++q) s = s + p[static_cast<size_t>(q) * n + r];
    y.at(b)[r] = with_rhs ? rhs.at(b)[r] - s : s;
}

// partial[a][blk][i] = sum over the block's rows of conj(V_i[r]) w[r], i < cnt.
__global__ void __launch_bounds__(kDotThreads)
gm_dots_kernel(SysVec V, int n, int cnt, const int* __restrict__ act, SysVec w, cplx* __restrict__ partial) {
    __shared__ cplx red[kDotThreads];
    const int a = blockIdx.y, b = act[a];
    const cplx* wb = w.at(b);
    const int r0 = blockIdx.x * kDotRows;
    const int r1 = min(n, r0 + kDotRows);
    cplx* out = partial + (static_cast<size_t>(a) * gridDim.x + blockIdx.x) * cnt;
    for (int i = 0; i < cnt; ++i) {
        const cplx* vi = V.at(b, static_cast<size_t>(i) * n);
        cplx s = mk(0.0, 0.0);
        for (int r = r0 + threadIdx.x; r < r1; r += kDotThreads) s = s + conjg(vi[r]) * wb[r];
        red[threadIdx.x] = s;
        __syncthreads();
        for (int h = kDotThreads / 2; h > 0; h >>= 1) {
            if (threadIdx.x < h) red[threadIdx.x] = red[threadIdx.x] + red[threadIdx.x + h];
            __syncthreads();
        }
        if (threadIdx.x == 0) out[i] = red[0];
        __syncthreads();
    }
}

__global__ void gm_dots_reduce_kernel(const cplx* __restrict__ partial, int nblk, int cnt, cplx* __restrict__ h) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int a = blockIdx.y;
    if (i >= cnt) return;
    const cplx* p = partial + static_cast<size_t>(a) * nblk * cnt;
    cplx s = mk(0.0, 0.0);
    for (int q = 0; q < nblk; ++q) s = s + p[static_cast<size_t>(q) * cnt + i];
    h[static_cast<size_t>(a) * cnt + i] = s;
}

// y_b = alpha * y_b + sign * sum_{i<cnt} V_b,i c[a][i]
__global__ void gm_axpy_kernel(SysVec V, int n, int cnt, const int* __restrict__ act, const cplx* __restrict__ c,
                               double sign, double alpha, SysVec y) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int a = blockIdx.y, b = act[a];
    const cplx* ca = c + static_cast<size_t>(a) * cnt;
    cplx s = mk(0.0, 0.0);
    for (int i = 0; i < cnt; ++i) s = s + V.at(b, static_cast<size_t>(i) * n)[r] * ca[i];
    cplx* yb = y.at(b);
    yb[r] = yb[r] * alpha + s * sign;
}

// y_b (+off) = x_b * s[a]
__global__ void gm_scale_kernel(SysVec x, int n, const int* __restrict__ act, const double* __restrict__ s, SysVec y,
                                size_t yoff) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int a = blockIdx.y, b = act[a];
    y.at(b, yoff)[r] = x.at(b)[r] * s[a];
}

using Cx = std::complex<double>;

struct Ops {
    const double* A;
    size_t mstride, plane;
    int n, ld, B, m;
    GmresWorkspace& ws;
    cudaStream_t st;
    int nact = 0;
    int* act_dev() const { return ws.act; }
    cplx* partial() const { return reinterpret_cast<cplx*>(ws.partial); }
    cplx* hbuf() const { return reinterpret_cast<cplx*>(ws.h_dev); }
    int nchunk() const { return ceil_div(n, kMvCols); }
    // Staging rule: a pinned slot is rewritten only after a stream synchronisation
    // that follows its previous copy (every Arnoldi step synchronises in dots()).
    void set_active(const std::vector<int>& act) {
        nact = static_cast<int>(act.size());
        if (!nact) return;
        std::copy(act.begin(), act.end(), ws.pin_act);
        FDS_CUDA(cudaMemcpyAsync(ws.act, ws.pin_act, nact * sizeof(int), cudaMemcpyHostToDevice, st));
    }
    SysVec V() const { return {reinterpret_cast<cplx*>(ws.V), static_cast<size_t>(m + 1) * n}; }
    SysVec vec(double* p) const { return {reinterpret_cast<cplx*>(p), static_cast<size_t>(n)}; }
    // y = A x, or y = rhs - A x
    void matvec(SysVec x, SysVec y, const SysVec* rhs = nullptr) const {
        dim3 g(ceil_div(n, kMvRows), nchunk(), nact);
        FDS_LAUNCH(gm_matvec_kernel, g, kMvThreads, 0, st, A, mstride, plane, n, ld, act_dev(), x, partial(),
                   nchunk());
        dim3 gr(ceil_div(n, 256), nact);
        FDS_LAUNCH(gm_chunk_reduce_kernel, gr, 256, 0, st, partial(), nchunk(), n, act_dev(), rhs ? *rhs : y,
                   rhs != nullptr, y);
    }
    void precond(SysVec x, size_t xoff, SysVec z) const {
        dim3 g(ceil_div(n / 3, 128), nact);
        FDS_LAUNCH(gm_precond_kernel, g, 128, 0, st, reinterpret_cast<const cplx*>(ws.pinv), n / 3, act_dev(), x,
                   xoff, z);
    }
    // h[a][0..cnt) = V_b^H w_b, to the host
    void dots(SysVec Vv, int cnt, SysVec w, std::vector<Cx>& h) const {
        const int nblk = ceil_div(n, kDotRows);
        FDS_LAUNCH(gm_dots_kernel, dim3(nblk, nact), kDotThreads, 0, st, Vv, n, cnt, act_dev(), w, partial());
        FDS_LAUNCH(gm_dots_reduce_kernel, dim3(ceil_div(cnt, 64), nact), 64, 0, st, partial(), nblk, cnt, hbuf());
        h.resize(static_cast<size_t>(nact) * cnt);
        FDS_CUDA(cudaMemcpyAsync(h.data(), hbuf(), h.size() * sizeof(cplx), cudaMemcpyDeviceToHost, st));
        FDS_CUDA(cudaStreamSynchronize(st));
    }
    // y_b = alpha y_b + sign * V_b c[a]   (c: host, [nact][cnt]; staged in pinned slot `slot`)
    void axpy(SysVec Vv, int cnt, const std::vector<Cx>& c, double sign, double alpha, SysVec y, int slot = 0) const {
        std::copy(c.begin(), c.end(), reinterpret_cast<Cx*>(ws.pin_coef[slot]));
        cplx* dst = hbuf() + static_cast<size_t>(slot) * B * (m + 2);
        FDS_CUDA(cudaMemcpyAsync(dst, ws.pin_coef[slot], c.size() * sizeof(cplx), cudaMemcpyHostToDevice, st));
        FDS_LAUNCH(gm_axpy_kernel, dim3(ceil_div(n, 256), nact), 256, 0, st, Vv, n, cnt, act_dev(), dst, sign, alpha,
                   y);
    }
    void norms(SysVec w, std::vector<double>& out) const {
        std::vector<Cx> h;
        dots(w, 1, w, h);
        out.resize(nact);
        for (int a = 0; a < nact; ++a) out[a] = std::sqrt(std::max(h[a].real(), 0.0));
    }
    void scale(SysVec x, const std::vector<double>& s, SysVec y, size_t yoff) const {
        std::copy(s.begin(), s.begin() + nact, ws.pin_scal);
        FDS_CUDA(cudaMemcpyAsync(ws.scal, ws.pin_scal, nact * sizeof(double), cudaMemcpyHostToDevice, st));
        FDS_LAUNCH(gm_scale_kernel, dim3(ceil_div(n, 256), nact), 256, 0, st, x, n, act_dev(), ws.scal, y, yoff);
    }
};

// per-system Arnoldi / Givens state of one cycle
struct Cycle {
    std::vector<Cx> H, cs, sn, g;
    int j = 0;  // columns built
    void reset(int m, double beta) {
        H.assign(static_cast<size_t>(m + 1) * m, Cx(0.0, 0.0));
        cs.assign(m, Cx(0.0, 0.0));
        sn.assign(m, Cx(0.0, 0.0));
        g.assign(m + 1, Cx(0.0, 0.0));
        g[0] = beta;
        j = 0;
    }
};

}  // namespace

void GmresWorkspace::ensure(int n, int m, int B) {
    if (static_cast<size_t>(n) <= n_cap && m <= m_cap && B <= b_cap) return;
    release();
    const size_t nc = static_cast<size_t>(n), bb = static_cast<size_t>(B);
    const size_t nchunk = (nc + kMvCols - 1) / kMvCols;
    const size_t nblk = (nc + kDotRows - 1) / kDotRows;
    FDS_CUDA(cudaMalloc(&V, 2 * nc * (m + 1) * bb * sizeof(double)));
    FDS_CUDA(cudaMalloc(&w, 2 * nc * bb * sizeof(double)));
    FDS_CUDA(cudaMalloc(&z, 2 * nc * bb * sizeof(double)));
    FDS_CUDA(cudaMalloc(&bsave, 2 * nc * bb * sizeof(double)));
    FDS_CUDA(cudaMalloc(&pinv, 2 * 3 * nc * bb * sizeof(double)));
    FDS_CUDA(cudaMalloc(&partial, 2 * bb * std::max(nchunk * nc, nblk * (m + 2)) * sizeof(double)));
    FDS_CUDA(cudaMalloc(&h_dev, 2 * 2 * bb * (m + 2) * sizeof(double)));  // dots results / two coefficient slots
    FDS_CUDA(cudaMallocHost(&pin_act, bb * sizeof(int)));
    FDS_CUDA(cudaMallocHost(&pin_coef[0], 2 * bb * (m + 2) * sizeof(double)));
    FDS_CUDA(cudaMallocHost(&pin_coef[1], 2 * bb * (m + 2) * sizeof(double)));
    FDS_CUDA(cudaMallocHost(&pin_scal, bb * sizeof(double)));
    FDS_CUDA(cudaMalloc(&scal, bb * sizeof(double)));
    FDS_CUDA(cudaMalloc(&act, bb * sizeof(int)));
    n_cap = nc;
    m_cap = m;
    b_cap = B;
}

void GmresWorkspace::release() {
    for (double* p : {V, w, z, pinv, partial, h_dev, bsave, scal})
        if (p) cudaFree(p);
    if (act) cudaFree(act);
    for (void* q : {static_cast<void*>(pin_act), static_cast<void*>(pin_coef[0]), static_cast<void*>(pin_coef[1]),
                    static_cast<void*>(pin_scal)})
        if (q) cudaFreeHost(q);
    V = w = z = pinv = partial = h_dev = bsave = scal = nullptr;
    act = nullptr;
    pin_act = nullptr;
    pin_coef[0] = pin_coef[1] = pin_scal = nullptr;
    n_cap = 0;
    m_cap = 0;
    b_cap = 0;
}

std::vector<GmresStats> gmres_solve_batch(const double* A, size_t mstride, size_t plane, int n, int ld, int B,
                                          cplx* rhs, size_t rstride, const GmresParams& p, GmresWorkspace& ws,
                                          cudaStream_t st) {
    if (n % 3 != 0) throw ValidationError("gmres: n must be a multiple of 3 (element-major DOFs)");
    std::vector<GmresStats> stats(B);
    if (B == 0) return stats;
    const int m = std::max(1, p.restart);
    ws.ensure(n, m, B);
    Ops op{A, mstride, plane, n, ld, B, m, ws, st};
    const SysVec V = op.V(), w = op.vec(ws.w), z = op.vec(ws.z), bs = op.vec(ws.bsave);
    const SysVec x{rhs, rstride};
    FDS_LAUNCH(gm_pinv_kernel, dim3(ceil_div(n / 3, 128), B), 128, 0, st, A, mstride, plane, n / 3, ld,
               reinterpret_cast<cplx*>(ws.pinv));
    // save b, r = b (x = 0), x := 0
    for (int b = 0; b < B; ++b) {
        FDS_CUDA(cudaMemcpyAsync(bs.at(b), x.at(b), n * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
        FDS_CUDA(cudaMemcpyAsync(w.at(b), x.at(b), n * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
        FDS_CUDA(cudaMemsetAsync(x.at(b), 0, n * sizeof(cplx), st));
    }
    std::vector<int> all(B);
    for (int b = 0; b < B; ++b) all[b] = b;
    op.set_active(all);
    std::vector<double> bnorm, beta;
    op.norms(w, bnorm);
    beta = bnorm;
    std::vector<Cycle> cyc(B);
    std::vector<int> live;  // systems still being solved (b = 0 gives x = 0 at once)
    for (int b = 0; b < B; ++b)
        if (bnorm[b] > 0.0) live.push_back(b);
    std::vector<Cx> h, h2, coef;
    std::vector<double> hn, sc;
    std::vector<double> prev(B, 1.0);  // relative residual at the start of the previous cycle
    bool first = true;
    while (true) {
        std::vector<int> act;  // systems that still need a cycle
        for (int b : live) {
            stats[b].rel_residual = beta[b] / bnorm[b];
            // a full restart cycle that did not halve the residual is stagnation
            // (e.g. near an interior resonance): give up early, the caller falls back
            const bool stalled = !first && stats[b].rel_residual > 0.5 * prev[b];
            prev[b] = stats[b].rel_residual;
            if (stats[b].rel_residual > p.tol && stats[b].iterations < p.max_iter && !stalled) act.push_back(b);
        }
        first = false;
        live = act;
        if (live.empty()) break;
        // new cycle: V_b0 = r_b / beta_b
        op.set_active(live);
        sc.resize(live.size());
        for (size_t a = 0; a < live.size(); ++a) {
            sc[a] = 1.0 / beta[live[a]];
            cyc[live[a]].reset(m, beta[live[a]]);
        }
        op.scale(w, sc, V, 0);
        std::vector<int> arn = live;  // systems still extending their basis in this cycle
        for (int j = 0; j < m && !arn.empty(); ++j) {
            if (j > 0) op.set_active(arn);  // j = 0: the device list already holds `live`
            const int na = static_cast<int>(arn.size());
            op.precond(V, static_cast<size_t>(j) * n, z);
            op.matvec(z, w);
            op.dots(V, j + 1, w, h);  // CGS, twice
            op.axpy(V, j + 1, h, -1.0, 1.0, w);
            op.dots(V, j + 1, w, h2);
            op.axpy(V, j + 1, h2, -1.0, 1.0, w);
            op.norms(w, hn);
            sc.assign(na, 0.0);
            std::vector<int> next;
            for (int a = 0; a < na; ++a) {
                const int b = arn[a];
                Cycle& c = cyc[b];
                auto Hc = [&](int i, int col) -> Cx& { return c.H[static_cast<size_t>(i) * m + col]; };
                for (int i = 0; i <= j; ++i)
                    Hc(i, j) = h[static_cast<size_t>(a) * (j + 1) + i] + h2[static_cast<size_t>(a) * (j + 1) + i];
                Hc(j + 1, j) = hn[a];
                for (int i = 0; i < j; ++i) {  // previous rotations
                    const Cx u = Hc(i, j), v = Hc(i + 1, j);
                    Hc(i, j) = std::conj(c.cs[i]) * u + std::conj(c.sn[i]) * v;
                    Hc(i + 1, j) = -c.sn[i] * u + c.cs[i] * v;
                }
                const Cx u = Hc(j, j), v = Hc(j + 1, j);
                const double den = std::sqrt(std::norm(u) + std::norm(v));
                if (den == 0.0) throw NumericError("gmres: breakdown (zero Krylov column)");
                c.cs[j] = u / den;
                c.sn[j] = v / den;
                Hc(j, j) = den;
                Hc(j + 1, j) = 0.0;
                c.g[j + 1] = -c.sn[j] * c.g[j];
                c.g[j] = std::conj(c.cs[j]) * c.g[j];
                c.j = j + 1;
                ++stats[b].iterations;
                sc[a] = hn[a] > 0.0 ? 1.0 / hn[a] : 0.0;
                const bool done = std::abs(c.g[j + 1]) / bnorm[b] <= p.tol || hn[a] == 0.0 ||
                                  stats[b].iterations >= p.max_iter;
                if (!done) next.push_back(b);
            }
            op.scale(w, sc, V, static_cast<size_t>(j + 1) * n);
            arn = next;
        }
        // y_b = H_b^{-1} g_b; x_b += M^{-1} V_b y_b; true residual
        op.set_active(live);
        int jmax = 0;
        for (int b : live) jmax = std::max(jmax, cyc[b].j);
        coef.assign(live.size() * static_cast<size_t>(jmax), Cx(0.0, 0.0));
        for (size_t a = 0; a < live.size(); ++a) {
            Cycle& c = cyc[live[a]];
            for (int i = c.j - 1; i >= 0; --i) {
                Cx s = c.g[i];
                for (int q = i + 1; q < c.j; ++q) s -= c.H[static_cast<size_t>(i) * m + q] * coef[a * jmax + q];
                coef[a * jmax + i] = s / c.H[static_cast<size_t>(i) * m + i];
            }
        }
        op.axpy(V, jmax, coef, 1.0, 0.0, w, 0);  // w = V y
        op.precond(w, 0, z);
        coef.assign(live.size(), Cx(1.0, 0.0));
        op.axpy(z, 1, coef, 1.0, 1.0, x, 1);  // x += M^{-1} V y (second staging slot: no sync in between)
        op.matvec(x, w, &bs);             // r = b - A x
        op.norms(w, hn);
        for (size_t a = 0; a < live.size(); ++a) beta[live[a]] = hn[a];
    }
    for (int b = 0; b < B; ++b) stats[b].converged = stats[b].rel_residual <= p.tol;
    return stats;
}

GmresStats gmres_solve(const double* Are, const double* Aim, int n, int ld, cplx* b, const GmresParams& p,
                       GmresWorkspace& ws, cudaStream_t st) {
    const size_t plane = static_cast<size_t>(Aim - Are);
    const GmresStats r = gmres_solve_batch(Are, 2 * plane, plane, n, ld, 1, b, static_cast<size_t>(n), p, ws, st)[0];
    if (!r.converged)
        throw ConvergenceError("gmres: relative residual " + std::to_string(r.rel_residual) + " after " +
                               std::to_string(r.iterations) + " iterations");
    return r;
}

}  // namespace fdsb
