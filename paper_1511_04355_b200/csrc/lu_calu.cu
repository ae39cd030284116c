// Communication-avoiding panel factorization (tournament pivoting, "CALU")
// for the blocked complex LU of lu.cu — the default panel on sm_100a.
//
// The barrier-per-column panel (lu_panel_kernel) needs the whole tall panel
// resident in shared memory across CTAs and one grid-wide exchange per column,
// so a 3840 x 64 panel of a 129-matrix batch runs ~8 matrices at a time and a
// 15360 x 64 panel pays ~64 grid barriers. Tournament pivoting selects the 64
// pivot rows of a panel with a reduction tree instead:
//   calu_tournament_kernel  grid (P blocks, batch). Each CTA factors its own
//       128 x w block by GEPP in shared memory (thread per row, CTA-local
//       syncs only) and publishes its w candidate rows (original values).
//       Pairs of candidate sets are merged by the LAST-arriving CTA of the pair
//       (atomic counter per tree node, no spinning), again by GEPP on <= 2w
//       rows, up to the root. The root's GEPP on the w winners yields the
//       pivot order and L11\U11; it also turns the winner list into LAPACK-style
//       sequential swaps (ipiv) and records which displaced rows move where.
//   calu_apply_kernel       thread per panel row: writes L11\U11 to rows k..k+w,
//       and L21 = A21 U11^{-1} (row-wise triangular solve) for the rest, reading
//       displaced rows from the saved originals.
// The resulting ipiv / L / U layout is exactly the one lu_panel_kernel
// produces, so swap+TRSM, the DMMA GEMM and lu_solve are shared. Pivots differ
// from classic partial pivoting (tournament winners), with GEPP-like
// stability in practice; parity is on the solution vector.
#include <climits>

#include "lu.cuh"

namespace fdsb {

namespace {

constexpr int CW = 64;    // max panel width
constexpr int CR = 128;   // rows per local block and per merge
constexpr int CT = 512;   // threads per CTA: 4 per row (column-split rank-1 updates)
constexpr int CT_LAST = CT - 1;

struct TreeLevels {
    int count;
    int off[24];   // node offset of each level
    int size[24];  // nodes in each level
};

__device__ __forceinline__ double cabs1(double re, double im) { return fabs(re) + fabs(im); }

// GEPP with physical row swaps on a [w][CR] planar tile. Thread t of the CTA
// (CT = 4 CR threads) owns row t % CR and the columns jj ≡ t / CR (mod 4) of the
// rank-1 updates; rows 0..CR-1 of threads 0..CR-1 run the pivot search.
// Selects min(w, nr) pivot rows; after return rows 0..nsel-1 hold L\U of the
// selected rows in pivot order and idx[] is permuted alike.
__device__ int gepp_select(double* are, double* aim, int* idx, int nr, int w, double* red_v, int* red_i,
                           int* s_piv, int* s_zero) {
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const int row = t % CR, cg = t / CR;
    const int nsel = min(w, nr);
    if (t == 0) *s_zero = -1;
    cplx lprev = mk(0.0, 0.0);
    bool wprev = false;
    for (int j = 0; j < nsel; ++j) {
        if (t < CR) {
            double v = -1.0;
            int bi = INT_MAX;
            if (t >= j && t < nr) {
                v = cabs1(are[j * CR + t], aim[j * CR + t]);
                bi = t;
            }
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, v, off);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
                if (ov > v || (ov == v && oi < bi)) { v = ov; bi = oi; }
            }
            if (lane == 0) { red_v[wid] = v; red_i[wid] = bi; }
        }
        __syncthreads();
        // deferred store of the previous column's multiplier (all readers are done)
        if (wprev) {
            are[(j - 1) * CR + row] = lprev.re;
            aim[(j - 1) * CR + row] = lprev.im;
        }
        if (t == 0) {
            double bv = red_v[0];
            int bb = red_i[0];
            for (int q = 1; q < CR / 32; ++q)
                if (red_v[q] > bv || (red_v[q] == bv && red_i[q] < bb)) { bv = red_v[q]; bb = red_i[q]; }
            *s_piv = bb;
            if (!(bv > 0.0) && *s_zero < 0) *s_zero = j;
        }
        __syncthreads();
        const int p = *s_piv;
        if (p != j) {
            if (t < w) {
                double x = are[t * CR + j];
                are[t * CR + j] = are[t * CR + p];
                are[t * CR + p] = x;
                x = aim[t * CR + j];
                aim[t * CR + j] = aim[t * CR + p];
                aim[t * CR + p] = x;
            } else if (t == CT_LAST) {
                const int x = idx[j];
                idx[j] = idx[p];
                idx[p] = x;
            }
        }
        __syncthreads();
        const cplx u = mk(are[j * CR + j], aim[j * CR + j]);
        wprev = false;
        if (row > j && row < nr && (u.re != 0.0 || u.im != 0.0)) {
            const cplx l = mk(are[j * CR + row], aim[j * CR + row]) * crecip(u);
            for (int jj = j + 1 + cg; jj < w; jj += CT / CR) {
                const double ur = are[jj * CR + j], ui = aim[jj * CR + j];
                are[jj * CR + row] -= l.re * ur - l.im * ui;
                aim[jj * CR + row] -= l.re * ui + l.im * ur;
            }
            if (cg == 0) { lprev = l; wprev = true; }
        }
    }
    __syncthreads();
    if (wprev) {
        are[(nsel - 1) * CR + row] = lprev.re;
        aim[(nsel - 1) * CR + row] = lprev.im;
    }
    __syncthreads();
    return nsel;
}

}  // namespace

__global__ void __launch_bounds__(CT)
calu_tournament_kernel(const double* __restrict__ A, size_t mstride, size_t plane, int n, int ld, int k, int w,
                       TreeLevels tl, int* cand_idx, int* cand_cnt, double* cand_val, unsigned* counters,
                       int* ipiv, int* info, double* top, int* moves, double* disp) {
    extern __shared__ double csm[];
    double* are = csm;                 // [CW][CR]
    double* aim = are + CW * CR;       // [CW][CR]
    __shared__ int idx[CR];
    __shared__ double red_v[CT / 32];
    __shared__ int red_i[CT / 32];
    __shared__ int s_piv, s_zero, s_go;
    const int t = threadIdx.x;
    const int b = blockIdx.y;
    const int nodes = tl.off[tl.count - 1] + 1;
    const double* Are = A + static_cast<size_t>(b) * mstride;
    const double* Aim = Are + plane;
    int* bidx = cand_idx + static_cast<size_t>(b) * nodes * CW;
    int* bcnt = cand_cnt + static_cast<size_t>(b) * nodes;
    double* bval = cand_val + static_cast<size_t>(b) * nodes * 2 * CW * CW;
    unsigned* bctr = counters + static_cast<size_t>(b) * nodes;

    // ---- level 0: local GEPP on this CTA's rows
    int node = blockIdx.x;
    const int r0 = k + node * CR;
    const int nr = max(0, min(CR, n - r0));
    for (int q = t; q < w * CR; q += CT) {
        const int j = q / CR, i = q % CR;
        if (i < nr) {
            const size_t gi = static_cast<size_t>(k + j) * ld + r0 + i;
            are[j * CR + i] = Are[gi];
            aim[j * CR + i] = Aim[gi];
        }
    }
    if (t < CR) idx[t] = r0 + t;
    __syncthreads();
    int nsel = gepp_select(are, aim, idx, nr, w, red_v, red_i, &s_piv, &s_zero);
    int level = 0;
    auto publish = [&](int nd, int cnt) {
        // candidate rows' ORIGINAL values, re-read from the (unmodified) panel
        if (t < CW) bidx[static_cast<size_t>(nd) * CW + t] = t < cnt ? idx[t] : -1;
        if (t == 0) bcnt[nd] = cnt;
        double* v = bval + static_cast<size_t>(nd) * 2 * CW * CW;
        for (int q = t; q < cnt * w; q += CT) {
            const int i = q % cnt, j = q / cnt;
            const size_t gi = static_cast<size_t>(k + j) * ld + idx[i];
            v[j * CW + i] = Are[gi];
            v[CW * CW + j * CW + i] = Aim[gi];
        }
    };
    while (level < tl.count - 1) {
        publish(tl.off[level] + node, nsel);
        __threadfence();
        __syncthreads();
        const int parent = node >> 1;
        const int sib = node ^ 1;
        const bool has_sib = sib < tl.size[level];
        if (has_sib) {
            if (t == 0) {
                const unsigned old = atomicAdd(&bctr[tl.off[level + 1] + parent], 1u);
                s_go = old == 1u;
            }
            __syncthreads();
            if (!s_go) return;  // the sibling's CTA (arriving last) merges
            __threadfence();
        }
        // merge the (one or two) children into this tile
        const int c0 = tl.off[level] + (node & ~1);
        const int nch = has_sib ? 2 : 1;
        int tot = 0;
        for (int c = 0; c < nch; ++c) {
            const int nd = has_sib ? c0 + c : tl.off[level] + node;
            const int cnt = __ldcg(&bcnt[nd]);
            const double* v = bval + static_cast<size_t>(nd) * 2 * CW * CW;
            for (int q = t; q < cnt * w; q += CT) {
                const int i = q % cnt, j = q / cnt;
                are[j * CR + tot + i] = __ldcg(&v[j * CW + i]);
                aim[j * CR + tot + i] = __ldcg(&v[CW * CW + j * CW + i]);
            }
            if (t < cnt) idx[tot + t] = __ldcg(&bidx[static_cast<size_t>(nd) * CW + t]);
            tot += cnt;
        }
        __syncthreads();
        nsel = gepp_select(are, aim, idx, tot, w, red_v, red_i, &s_piv, &s_zero);
        node = parent;
        ++level;
    }
    // ---- root: rows 0..w-1 of the tile are L11\U11 of the winners in pivot order
    double* tp = top + static_cast<size_t>(b) * 2 * CW * CW;
    for (int q = t; q < w * w; q += CT) {
        const int i = q % w, j = q / w;
        tp[j * CW + i] = are[j * CR + i];
        tp[CW * CW + j * CW + i] = aim[j * CR + i];
    }
    // displaced rows k..k+w-1: keep their original values for the apply pass
    double* dp = disp + static_cast<size_t>(b) * 2 * CW * CW;
    for (int q = t; q < w * w; q += CT) {
        const int i = q % w, j = q / w;
        const size_t gi = static_cast<size_t>(k + j) * ld + k + i;
        dp[j * CW + i] = Are[gi];
        dp[CW * CW + j * CW + i] = Aim[gi];
    }
    if (t == 0) {
        if (s_zero >= 0 && info[b] == 0) info[b] = k + s_zero + 1;
        // winners -> LAPACK sequential swaps; track (position -> original row) for
        // the <= 2w positions the swaps touch.
        int pos[2 * CW], row[2 * CW];
        int na = 0;
        for (int i = 0; i < w; ++i) { pos[na] = k + i; row[na] = k + i; ++na; }
        int* mv = moves + static_cast<size_t>(b) * (1 + 2 * CW);
        for (int i = 0; i < w; ++i) {
            const int g = idx[i];
            int at = -1;  // current position of original row g
            for (int q = 0; q < na; ++q)
                if (row[q] == g) { at = pos[q]; break; }
            if (at < 0) {  // untouched so far: still at its own position
                at = g;
                pos[na] = g;
                row[na] = g;
                ++na;
            }
            ipiv[static_cast<size_t>(b) * n + k + i] = at;
            int qa = -1, qb = -1;
            for (int q = 0; q < na; ++q) {
                if (pos[q] == k + i) qa = q;
                if (pos[q] == at) qb = q;
            }
            const int tmp = row[qa];
            row[qa] = row[qb];
            row[qb] = tmp;
        }
        // positions >= k+w now holding a displaced original row (from k..k+w-1)
        int nm = 0;
        for (int q = 0; q < na; ++q)
            if (pos[q] >= k + w) { mv[1 + 2 * nm] = pos[q]; mv[2 + 2 * nm] = row[q]; ++nm; }
        mv[0] = nm;
    }
}

__global__ void __launch_bounds__(CR)
calu_apply_kernel(double* A, size_t mstride, size_t plane, int n, int ld, int k, int w, const double* __restrict__ top,
                  const int* __restrict__ moves, const double* __restrict__ disp) {
    extern __shared__ double asm_[];
    double* ure = asm_;              // [CW][CW] U11 (col j, row i)
    double* uim = ure + CW * CW;
    double* xre = uim + CW * CW;     // [CW][CR] row being solved (thread column)
    double* xim = xre + CW * CR;
    __shared__ int mv[1 + 2 * CW];
    const int b = blockIdx.y, t = threadIdx.x;
    double* Are = A + static_cast<size_t>(b) * mstride;
    double* Aim = Are + plane;
    const double* tp = top + static_cast<size_t>(b) * 2 * CW * CW;
    const double* dp = disp + static_cast<size_t>(b) * 2 * CW * CW;
    for (int q = t; q < w * w; q += CR) {
        const int i = q % w, j = q / w;
        ure[j * CW + i] = tp[j * CW + i];
        uim[j * CW + i] = tp[CW * CW + j * CW + i];
    }
    for (int q = t; q < 1 + 2 * CW; q += CR) mv[q] = moves[static_cast<size_t>(b) * (1 + 2 * CW) + q];
    __syncthreads();
    const int r = k + blockIdx.x * CR + t;
    if (r >= n) return;
    if (r < k + w) {
        const int i = r - k;
        for (int j = 0; j < w; ++j) {
            const size_t gi = static_cast<size_t>(k + j) * ld + r;
            Are[gi] = ure[j * CW + i];
            Aim[gi] = uim[j * CW + i];
        }
        return;
    }
    int src = -1;
    for (int q = 0; q < mv[0]; ++q)
        if (mv[1 + 2 * q] == r) { src = mv[2 + 2 * q] - k; break; }
    for (int j = 0; j < w; ++j) {
        if (src >= 0) {
            xre[j * CR + t] = dp[j * CW + src];
            xim[j * CR + t] = dp[CW * CW + j * CW + src];
        } else {
            const size_t gi = static_cast<size_t>(k + j) * ld + r;
            xre[j * CR + t] = Are[gi];
            xim[j * CR + t] = Aim[gi];
        }
    }
    // l U11 = a  (row vector): l_j = (a_j - sum_{i<j} l_i U_ij) / U_jj
    for (int j = 0; j < w; ++j) {
        double sr = xre[j * CR + t], si = xim[j * CR + t];
        for (int i = 0; i < j; ++i) {
            const double lr = xre[i * CR + t], li = xim[i * CR + t];
            const double ur = ure[j * CW + i], ui = uim[j * CW + i];
            sr -= lr * ur - li * ui;
            si -= lr * ui + li * ur;
        }
        const cplx d = mk(ure[j * CW + j], uim[j * CW + j]);
        const cplx l = (d.re != 0.0 || d.im != 0.0) ? cdiv(mk(sr, si), d) : mk(0.0, 0.0);
        xre[j * CR + t] = l.re;
        xim[j * CR + t] = l.im;
    }
    for (int j = 0; j < w; ++j) {
        const size_t gi = static_cast<size_t>(k + j) * ld + r;
        Are[gi] = xre[j * CR + t];
        Aim[gi] = xim[j * CR + t];
    }
}

// ------------------------------------------------------------------ host
void CaluWorkspace::ensure(int batch, int nodes) {
    const size_t need_nodes = static_cast<size_t>(batch) * nodes;
    if (need_nodes > node_cap) {
        release();
        FDS_CUDA(cudaMalloc(&cand_idx, need_nodes * CW * sizeof(int)));
        FDS_CUDA(cudaMalloc(&cand_cnt, need_nodes * sizeof(int)));
        FDS_CUDA(cudaMalloc(&cand_val, need_nodes * 2 * CW * CW * sizeof(double)));
        FDS_CUDA(cudaMalloc(&counters, need_nodes * sizeof(unsigned)));
        node_cap = need_nodes;
    }
    if (batch > batch_cap) {
        if (top) cudaFree(top);
        if (disp) cudaFree(disp);
        if (moves) cudaFree(moves);
        FDS_CUDA(cudaMalloc(&top, static_cast<size_t>(batch) * 2 * CW * CW * sizeof(double)));
        FDS_CUDA(cudaMalloc(&disp, static_cast<size_t>(batch) * 2 * CW * CW * sizeof(double)));
        FDS_CUDA(cudaMalloc(&moves, static_cast<size_t>(batch) * (1 + 2 * CW) * sizeof(int)));
        batch_cap = batch;
    }
}

void CaluWorkspace::release() {
    auto fr = [](void* p) { if (p) cudaFree(p); };
    fr(cand_idx); fr(cand_cnt); fr(cand_val); fr(counters);
    cand_idx = nullptr; cand_cnt = nullptr; cand_val = nullptr; counters = nullptr;
    node_cap = 0;
}

void calu_panel_step(const LuProblem& pb, CaluWorkspace& ws, int k, int w, cudaStream_t st) {
    if (w > CW) throw ValidationError("calu: panel wider than 64");
    const int rows = pb.n - k;
    const int P = ceil_div(rows, CR);
    TreeLevels tl{};
    int sz = P, off = 0, lv = 0;
    while (true) {
        tl.off[lv] = off;
        tl.size[lv] = sz;
        ++lv;
        if (sz == 1) break;
        off += sz;
        sz = (sz + 1) / 2;
        if (lv >= 24) throw NumericError("calu: tournament tree too deep");
    }
    tl.count = lv;
    const int nodes = tl.off[lv - 1] + 1;
    ws.ensure(pb.batch, nodes);
    FDS_CUDA(cudaMemsetAsync(ws.counters, 0, static_cast<size_t>(pb.batch) * nodes * sizeof(unsigned), st));
    static bool attr = false;
    const size_t smem_t = 2 * CW * CR * sizeof(double);
    const size_t smem_a = (2 * CW * CW + 2 * CW * CR) * sizeof(double);
    if (!attr) {
        FDS_CUDA(cudaFuncSetAttribute(calu_tournament_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem_t)));
        FDS_CUDA(cudaFuncSetAttribute(calu_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem_a)));
        attr = true;
    }
    cudaEvent_t pe;
    profiler().begin(st, kProfLuPanel, 0.0, pe);
    FDS_LAUNCH(calu_tournament_kernel, dim3(P, pb.batch), CT, smem_t, st, pb.A, pb.mstride, pb.plane, pb.n, pb.ld,
               k, w, tl, ws.cand_idx, ws.cand_cnt, ws.cand_val, ws.counters, pb.ipiv, pb.info, ws.top, ws.moves,
               ws.disp);
    FDS_LAUNCH(calu_apply_kernel, dim3(ceil_div(rows, CR), pb.batch), CR, smem_a, st, pb.A, pb.mstride, pb.plane,
               pb.n, pb.ld, k, w, ws.top, ws.moves, ws.disp);
    profiler().end(st, pe, kProfLuPanel, 8.0 * rows * w * w / 2.0 * pb.batch);
}

}  // namespace fdsb
