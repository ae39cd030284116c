// Common-pole vector fitting on sm_100a — replaces proj/src/vecfit.cpp
// (vecfit.hpp:48-86) and the dense-grid kernels of proj/src/afs.cpp
// (channel_errors :118-145, select_new_frequency :147-187).
//
// Device work (batched over channels / DOFs):
//   vf_reloc_qr_kernel   one CTA per ORF channel: Householder QR of the real
//                        2J x (2M+1) block [Φ·D1 | −diag(f_k)Φ·D2 | b_k]
//                        (vecfit.cpp:242-279) in shared memory; emits the R22
//                        rows, the matching Qᵀb and the tail norm.
//   vf_residue_kernel    identify_residues for every channel at once
//                        (vecfit.cpp:356-408): the LS matrix [Re Φ; Im Φ] is
//                        identical for all channels, so its pivoted QR is
//                        factored once on the host into the solve operator W
//                        (M x 2J) and the kernel applies x = W b per channel
//                        (thread per channel, W chunk in smem, pair-aware
//                        residue packing), output residues [m][k].
//   vf_rms_kernel        per-channel residual RMS of the fitted model.
//   vf_inv_table_kernel  1/(s_g − a_m) over the dense grid, [m][g].
//   vf_chanerr_kernel    CTA per channel: max_g|f_H − f_L|, max_g|f_H|.
//   vf_select_kernel     exclusion-radius filtered argmax of |f_H − f_L| for the
//                        worst ORF channel (first maximum = smallest ω).
//   vf_eval_kernel       eval_model / fit_error_evf (vecfit.cpp:490-526): thread
//                        per (s, channel) partial-fraction sum, exact pole
//                        collisions flagged for NumericError.
// The shared pivoted QR and the stacked σ least squares run on one CTA
// (vf_lsq.cu); only the M x M relocation eigenproblem stays on the host
// (eig_host.cpp).
#include <algorithm>
#include <cmath>
#include <limits>

#include "eig_host.h"

#include <cstdlib>
#include <cstring>
#include <type_traits>
#include "vf.cuh"

namespace fdsb {

// ------------------------------------------------------------------ workspace
void* VfContext::Buf::get(size_t need) {
    if (need > bytes) {
        if (p) cudaFree(p);
        p = nullptr;
        FDS_CUDA(cudaMalloc(&p, need));
        bytes = need;
    }
    return p;
}

void VfContext::release() {
    if (st) cudaStreamSynchronize(st);
    for (Buf* b : {&values, &resid, &W, &phi, &rms, &tab, &tab2, &out, &misc, &misc2, &qr, &lsq, &lsq_io, &chanerr}) {
        if (b->p) cudaFree(b->p);
        b->p = nullptr;
        b->bytes = 0;
    }
    w_valid = false;
    w_key.clear();
}

VfContext& VfContext::get() {
    static thread_local VfContext ctx;
    if (!ctx.st) {
        device_info();
        FDS_CUDA(cudaStreamCreateWithFlags(&ctx.st, cudaStreamNonBlocking));
    }
    return ctx;
}

// ------------------------------------------------------------------ host helpers
namespace {

bool near_conj(Cx a, Cx b, double tol) {
    const double sc = std::max({std::abs(a), std::abs(b), 1e-300});
    return std::abs(a - std::conj(b)) <= tol * sc;
}

// Real-parameterised partial-fraction basis (vecfit.cpp:38-69), phi[m*J + j].
std::vector<Cx> basis(const std::vector<Cx>& s, const std::vector<Cx>& poles) {
    const int J = static_cast<int>(s.size()), M = static_cast<int>(poles.size());
    std::vector<Cx> phi(static_cast<size_t>(J) * M);
    const Cx I(0.0, 1.0);
    for (int j = 0; j < J; ++j) {
        int m = 0;
        while (m < M) {
            const Cx p = poles[m];
            if (p.imag() != 0.0) {
                const Cx d1 = s[j] - p, d2 = s[j] - std::conj(p);
                if (d1 == 0.0 || d2 == 0.0) throw NumericError("sample frequency coincides with a pole");
                phi[static_cast<size_t>(m) * J + j] = 1.0 / d1 + 1.0 / d2;
                phi[static_cast<size_t>(m + 1) * J + j] = I / d1 - I / d2;
                m += 2;
            } else {
                const Cx d = s[j] - p;
                if (d == 0.0) throw NumericError("sample frequency coincides with a pole");
                phi[static_cast<size_t>(m) * J + j] = 1.0 / d;
                m += 1;
            }
        }
    }
    return phi;
}

int pair_count(const std::vector<Cx>& canon) {
    int p = 0;
    while (2 * p + 1 < static_cast<int>(canon.size()) && canon[2 * p].imag() != 0.0) ++p;
    return p;
}

double movement_of(const std::vector<Cx>& oldp, const std::vector<Cx>& newp) {  // vecfit.cpp:90-106
    double worst = 0.0;
    for (Cx p : newp) {
        double best = std::numeric_limits<double>::infinity();
        Cx match = oldp.empty() ? Cx(0, 0) : oldp[0];
        for (Cx q : oldp) {
            const double d = std::abs(p - q);
            if (d < best) { best = d; match = q; }
        }
        worst = std::max(worst, best / std::max(std::abs(match), 1e-30));
    }
    return worst;
}

}  // namespace

std::vector<Cx> canonical_order(const std::vector<Cx>& poles) {
    std::vector<Cx> heads, reals;
    std::vector<char> used(poles.size(), 0);
    for (size_t i = 0; i < poles.size(); ++i) {
        if (used[i]) continue;
        if (poles[i].imag() == 0.0) { reals.push_back(poles[i]); used[i] = 1; continue; }
        size_t k = i + 1;
        for (; k < poles.size(); ++k)
            if (!used[k] && poles[k].imag() != 0.0 && near_conj(poles[i], poles[k], 1e-9)) break;
        if (k == poles.size()) throw ValidationError("pole set is not closed under conjugation");
        heads.push_back(poles[i].imag() > 0.0 ? poles[i] : poles[k]);
        used[i] = used[k] = 1;
    }
    std::vector<Cx> out;
    out.reserve(poles.size());
    for (Cx h : heads) { out.push_back(h); out.push_back(std::conj(h)); }
    out.insert(out.end(), reals.begin(), reals.end());
    return out;
}

bool conj_closed(const std::vector<Cx>& poles, double tol) {
    std::vector<char> used(poles.size(), 0);
    for (size_t i = 0; i < poles.size(); ++i) {
        if (used[i] || poles[i].imag() == 0.0) continue;
        bool hit = false;
        for (size_t k = 0; k < poles.size() && !hit; ++k)
            if (k != i && !used[k] && near_conj(poles[i], poles[k], tol)) { used[i] = used[k] = 1; hit = true; }
        if (!hit) return false;
    }
    return true;
}

void require_distinct(const std::vector<Cx>& s) {
    std::vector<Cx> v = s;
    std::sort(v.begin(), v.end(), [](Cx a, Cx b) { return a.real() != b.real() ? a.real() < b.real() : a.imag() < b.imag(); });
    for (size_t j = 1; j < v.size(); ++j)
        if (v[j] == v[j - 1]) throw ValidationError("duplicate sample frequencies");
}

std::vector<Cx> start_poles(double omega_max, int order) {
    if (order < 1) throw ValidationError("initial_poles: order must be >= 1");
    if (!(omega_max > 0.0)) throw ValidationError("initial_poles: omega_max must be positive");
    std::vector<Cx> p;
    const int pairs = order / 2;
    for (int i = 1; i <= pairs; ++i) {
        const double beta = omega_max * static_cast<double>(i) / pairs;
        p.emplace_back(-beta / 100.0, beta);
        p.emplace_back(-beta / 100.0, -beta);
    }
    if (order % 2 == 1) p.emplace_back(-omega_max / 100.0, 0.0);
    return p;
}

// ------------------------------------------------------------------ kernels
namespace {

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += red[w];
    return t;
}

}  // namespace

// 32 warps: each Householder step's column updates are latency-bound (the
// matrix lives in global memory once 2J x (2M+1) exceeds shared memory), so the
// CTA keeps up to 32 columns in flight (J = 210, M = 104: 8 warps took 6.7 ms)
constexpr int kRelocQrThreads = 1024;

__global__ void __launch_bounds__(kRelocQrThreads)
vf_reloc_qr_kernel(int J, int M, int K, const cplx* __restrict__ vals, const cplx* __restrict__ phi,
                   const double* __restrict__ cscale, const double* __restrict__ sscale, double* gwork,
                   double* __restrict__ r22, double* __restrict__ beta_out, double* __restrict__ tail) {
    extern __shared__ double qsm[];
    __shared__ double red[32];
    __shared__ double s_tau, s_beta, s_inv;
    const int k = blockIdx.x;
    const int rows = 2 * J, cols = 2 * M + 1;
    const int top = min(2 * M, rows), red_rows = max(0, top - M);
    double* a = gwork ? gwork + static_cast<size_t>(k) * rows * cols : qsm;
    for (int idx = threadIdx.x; idx < rows * cols; idx += blockDim.x) {
        const int i = idx % rows, c = idx / rows;
        const int j = i >> 1, part = i & 1;
        const cplx f = vals[static_cast<size_t>(j) * K + k];
        double v;
        if (c < M) {
            const cplx p = phi[static_cast<size_t>(c) * J + j];
            v = (part ? p.im : p.re) * cscale[c];
        } else if (c < 2 * M) {
            const int m = c - M;
            const cplx r = -(f * phi[static_cast<size_t>(m) * J + j]) * sscale[m];
            v = part ? r.im : r.re;
        } else {
            v = part ? f.im : f.re;
        }
        a[static_cast<size_t>(c) * rows + i] = v;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    for (int q = 0; q < top; ++q) {
        double* col = a + static_cast<size_t>(q) * rows;
        double part = 0.0;
        for (int i = q + 1 + threadIdx.x; i < rows; i += blockDim.x) part += col[i] * col[i];
        const double sig = block_sum(part, red);
        if (threadIdx.x == 0) {
            const double x0 = col[q];
            if (sig <= 2.2250738585072014e-308) {
                s_tau = 0.0;
                s_beta = x0;
                s_inv = 0.0;
            } else {
                const double nrm = sqrt(x0 * x0 + sig);
                const double bt = x0 >= 0.0 ? -nrm : nrm;
                s_beta = bt;
                s_inv = 1.0 / (x0 - bt);
                s_tau = (bt - x0) / bt;
            }
        }
        __syncthreads();
        const double tau = s_tau;
        for (int i = q + 1 + threadIdx.x; i < rows; i += blockDim.x) col[i] = tau == 0.0 ? 0.0 : col[i] * s_inv;
        __syncthreads();
        if (threadIdx.x == 0) col[q] = s_beta;
        __syncthreads();
        if (tau != 0.0) {
            for (int c = q + 1 + warp; c < cols; c += nwarp) {
                double* cc = a + static_cast<size_t>(c) * rows;
                double d = 0.0;
                for (int i = q + 1 + lane; i < rows; i += 32) d += col[i] * cc[i];
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) d += __shfl_xor_sync(0xffffffffu, d, off);
                d = (d + cc[q]) * tau;
                if (lane == 0) cc[q] -= d;
                for (int i = q + 1 + lane; i < rows; i += 32) cc[i] -= d * col[i];
            }
        }
        __syncthreads();
    }
    // R22 = R[M:top, M:2M] (upper-triangular view), beta = (Q^T b)[M:top], tail = ||(Q^T b)[top:]||^2
    for (int idx = threadIdx.x; idx < red_rows * M; idx += blockDim.x) {
        const int i = idx / M, c = idx % M;
        r22[(static_cast<size_t>(k) * red_rows + i) * M + c] = c >= i ? a[static_cast<size_t>(M + c) * rows + M + i] : 0.0;
    }
    const double* bcol = a + static_cast<size_t>(2 * M) * rows;
    for (int i = threadIdx.x; i < red_rows; i += blockDim.x) beta_out[static_cast<size_t>(k) * red_rows + i] = bcol[M + i];
    double tp = 0.0;
    for (int i = top + threadIdx.x; i < rows; i += blockDim.x) tp += bcol[i] * bcol[i];
    const double tt = block_sum(tp, red);
    if (threadIdx.x == 0) tail[k] = tt;
}

constexpr int kResChunk = 8;
constexpr int kResThreads = 128;

__global__ void __launch_bounds__(kResThreads)
vf_residue_kernel(int J, int K, int M, int P, const cplx* __restrict__ vals, const double* __restrict__ W,
                  cplx* __restrict__ res, int heads) {
    extern __shared__ double wsm[];  // [kResChunk][2J]
    const int m0 = blockIdx.y * kResChunk;
    const int cm = min(kResChunk, M - m0);
    for (int idx = threadIdx.x; idx < cm * 2 * J; idx += blockDim.x)
        wsm[idx] = W[static_cast<size_t>(m0) * 2 * J + idx];
    __syncthreads();
    const int k = blockIdx.x * kResThreads + threadIdx.x;
    if (k >= K) return;
    double x[kResChunk];
#pragma unroll
    for (int c = 0; c < kResChunk; ++c) x[c] = 0.0;
    for (int j = 0; j < J; ++j) {
        const cplx f = vals[static_cast<size_t>(j) * K + k];
#pragma unroll
        for (int c = 0; c < kResChunk; ++c) {
            if (c < cm) x[c] += wsm[c * 2 * J + 2 * j] * f.re + wsm[c * 2 * J + 2 * j + 1] * f.im;
        }
    }
    // canonical packing (vecfit.cpp:72-88): pairs first (heads at even slots), reals last
#pragma unroll
    for (int c = 0; c < kResChunk; ++c) {
        const int m = m0 + c;
        if (c >= cm) break;
        cplx r;
        if (m < 2 * P) {
            r = (m % 2 == 0) ? mk(x[c], x[c + 1 < kResChunk ? c + 1 : c]) : mk(x[c - 1 >= 0 ? c - 1 : 0], -x[c]);
        } else {
            r = mk(x[c], 0.0);
        }
        if (heads && m < 2 * P && (m & 1)) continue;  // conjugate row not requested
        res[static_cast<size_t>(m) * K + k] = r;
    }
}

// identify_residues apply on the FP64 tensor pipe: X (M x K) = W (M x 2J) B (2J x K),
// B[2j + part][k] = (Re, Im) of values[j][k]. CTA: 64 output rows (poles) x 64
// channels, 4 warps of 32x32, the whole 2J reduction staged in smem.
constexpr int kRmS = 68;
__device__ __forceinline__ void dmma_v(double& c0, double& c1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c0), "+d"(c1)
        : "d"(a), "d"(b));
}

constexpr int kResNI = 2;  // 8-channel sub-tiles per warp (16 channels): low registers, many warps

// Steps (4 q values each) per channel tile, padded to a multiple of the prefetch depth.
__host__ __device__ inline int res_steps(int J, int PF) { return ((J + 1) / 2 + PF - 1) / PF * PF; }

template <int MT, int PF>
__global__ void __launch_bounds__(128, 4)
vf_residue_mma_kernel(int J, int K, int M, int P, const cplx* __restrict__ vals, const double* __restrict__ W,
                      cplx* __restrict__ res, int heads) {
    // Persistent CTAs; W (the shared solve operator, M x 2J) staged once in smem
    // as the A operand, zero past row M and past column 2J (the padded steps).
    // Each warp owns 16 channels x 8 MT poles per tile; its B fragments (Re/Im
    // of values[j][k]) come straight from HBM through a register ring of PF
    // steps that runs ACROSS tiles: the last chunk of a tile prefetches the
    // first chunk of the warp's next tile, so HBM latency is never exposed at
    // tile boundaries. Each load instruction covers whole 128 B lines.
    extern __shared__ double rsm2[];
    const int Q = 2 * J, Sp = res_steps(J, PF), Qs = 4 * Sp, chunks = Sp / PF;
    double* As = rsm2;  // [Qs][kRmS], As[q][m] = W[m][q]  (M <= 64 per launch slice)
    const int m0 = blockIdx.y * 64;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int idx = tid; idx < Qs * 64; idx += blockDim.x) {
        const int m = idx / Qs, q = idx % Qs;
        As[q * kRmS + m] = (m0 + m < M && q < Q) ? W[static_cast<size_t>(m0 + m) * Q + q] : 0.0;
    }
    __syncthreads();
    const double* vd = reinterpret_cast<const double*>(vals);
    const int q_l = lane & 3, n_l = lane >> 2;
    const int j0 = q_l >> 1, part = q_l & 1;
    const double* Al = As + q_l * kRmS + n_l;
    const int warps_total = gridDim.x * (blockDim.x >> 5);
    const size_t row2 = 2 * static_cast<size_t>(K);  // doubles per value row j
    // lane's channel columns of a tile (clamped: ragged columns are computed, not stored)
    auto cols = [&](int tile, const double* (&bc)[kResNI]) {
#pragma unroll
        for (int ni = 0; ni < kResNI; ++ni)
            bc[ni] = vd + static_cast<size_t>(min(tile * (8 * kResNI) + ni * 8 + n_l, K - 1)) * 2 + part;
    };
    // step st reads value row j = 2 st + j0 (clamped: rows past J meet zero columns of W)
    auto bload = [&](const double* (&bc)[kResNI], int st, double (&fb)[kResNI]) {
        const size_t off = static_cast<size_t>(min(2 * st + j0, J - 1)) * row2;
#pragma unroll
        for (int ni = 0; ni < kResNI; ++ni) fb[ni] = __ldcs(bc[ni] + off);
    };
    int tile = blockIdx.x * (blockDim.x >> 5) + warp;
    if (tile * (8 * kResNI) >= K) return;
    const double* bc[kResNI];
    cols(tile, bc);
    double ring[PF][kResNI];
#pragma unroll
    for (int p = 0; p < PF; ++p) bload(bc, p, ring[p]);
    for (; tile * (8 * kResNI) < K; tile += warps_total) {
        const int kb = tile * (8 * kResNI);
        double acc[MT][kResNI][2];
#pragma unroll
        for (int mi = 0; mi < MT; ++mi)
#pragma unroll
            for (int ni = 0; ni < kResNI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
        for (int c = 0; c < chunks; ++c) {
            // prefetch target: the next chunk of this tile, or chunk 0 of the next tile
            const bool last = c + 1 == chunks;
            const int nc = last ? 0 : c + 1;
            const bool more = !last || (tile + warps_total) * (8 * kResNI) < K;
            if (last) cols(tile + warps_total, bc);
#pragma unroll
            for (int p = 0; p < PF; ++p) {
                double fb[kResNI];
#pragma unroll
                for (int ni = 0; ni < kResNI; ++ni) fb[ni] = ring[p][ni];
                if (more) bload(bc, nc * PF + p, ring[p]);
                const double* a = Al + 4 * (c * PF + p) * kRmS;
#pragma unroll
                for (int mi = 0; mi < MT; ++mi) {
                    const double fa = a[mi * 8];
#pragma unroll
                    for (int ni = 0; ni < kResNI; ++ni) dmma_v(acc[mi][ni][0], acc[mi][ni][1], fa, fb[ni]);
                }
            }
        }
        const int mtiles = min(MT, (M - m0 + 7) / 8);
        // canonical packing: rows m (even, < 2P) and m+1 form one conjugate pair;
        // the partner row sits 4 lanes away in the accumulator fragment.
#pragma unroll
        for (int mi = 0; mi < MT; ++mi) {
            if (mi >= mtiles) break;
            const int m = m0 + mi * 8 + n_l;
#pragma unroll
            for (int ni = 0; ni < kResNI; ++ni)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const double x = acc[mi][ni][e];
                    const double y = __shfl_xor_sync(0xffffffffu, x, 4);
                    const int k = kb + ni * 8 + 2 * q_l + e;
                    if (m >= M || k >= K || (heads && m < 2 * P && (m & 1))) continue;
                    cplx r;
                    if (m < 2 * P) r = (m % 2 == 0) ? mk(x, y) : mk(y, -x);
                    else r = mk(x, 0.0);
                    __stcs(reinterpret_cast<double2*>(res) + static_cast<size_t>(m) * K + k, make_double2(r.re, r.im));
                }
        }
    }
}

__global__ void vf_rms_kernel(int J, int K, int M, const cplx* __restrict__ vals, const cplx* __restrict__ res,
                              const cplx* __restrict__ invd /*[m][j]*/, double* __restrict__ rms) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    double sq = 0.0;
    for (int j = 0; j < J; ++j) {
        cplx fit = mk(0.0, 0.0);
        for (int m = 0; m < M; ++m) fit = fit + res[static_cast<size_t>(m) * K + k] * invd[static_cast<size_t>(m) * J + j];
        const cplx d = fit - vals[static_cast<size_t>(j) * K + k];
        sq += abs2(d);
    }
    rms[k] = sqrt(sq / J);
}

// Few channels (the AFS fits: K = 5 ... 48): one CTA per channel, threads over
// the samples, fixed-order block reduction (the thread-per-channel kernel above
// runs a J x M loop on one thread per channel and only K threads in total).
__global__ void __launch_bounds__(128) vf_rms_cta_kernel(int J, int K, int M, const cplx* __restrict__ vals,
                                                         const cplx* __restrict__ res,
                                                         const cplx* __restrict__ invd /*[m][j]*/,
                                                         double* __restrict__ rms) {
    __shared__ double red[8];
    const int k = blockIdx.x;
    double sq = 0.0;
    for (int j = threadIdx.x; j < J; j += blockDim.x) {
        cplx fit = mk(0.0, 0.0);
        for (int m = 0; m < M; ++m) fit = fit + res[static_cast<size_t>(m) * K + k] * invd[static_cast<size_t>(m) * J + j];
        sq += abs2(fit - vals[static_cast<size_t>(j) * K + k]);
    }
    const double t = block_sum(sq, red);
    if (threadIdx.x == 0) rms[k] = sqrt(t / J);
}

__global__ void vf_inv_table_kernel(int G, int M, const cplx* __restrict__ grid, const cplx* __restrict__ poles,
                                    cplx* __restrict__ inv /*[m][g]*/) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= G * M) return;
    const int m = idx / G, g = idx % G;
    inv[idx] = crecip(grid[g] - poles[m]);
}

__device__ __forceinline__ void model_at(int g, int G, int M, const cplx* r, const cplx* inv, cplx& acc) {
    acc = mk(0.0, 0.0);
    for (int m = 0; m < M; ++m) acc = acc + r[m] * inv[static_cast<size_t>(m) * G + g];
}

__global__ void __launch_bounds__(256)
vf_chanerr_kernel(int G, int MH, int ML, int K, const cplx* __restrict__ rh, const cplx* __restrict__ rl,
                  size_t sk_h, size_t sm_h, size_t sk_l, size_t sm_l,  // residue (k, m) at r[k*sk + m*sm]
                  const cplx* __restrict__ invh, const cplx* __restrict__ invl,
                  double* __restrict__ out /*[k][2]: max|fH-fL|, max|fH|*/) {
    extern __shared__ cplx rsm[];
    __shared__ double red[2][8];
    const int k = blockIdx.x;
    for (int m = threadIdx.x; m < MH; m += blockDim.x) rsm[m] = rh[k * sk_h + m * sm_h];
    for (int m = threadIdx.x; m < ML; m += blockDim.x) rsm[MH + m] = rl[k * sk_l + m * sm_l];
    __syncthreads();
    double md = 0.0, mh = 0.0;
    // grid chunk blockIdx.y of gridDim.y (partial maxima, combined by
    // vf_chanerr_combine_kernel: max is exact, so the result is split-independent)
    const int gc = (G + gridDim.y - 1) / gridDim.y;
    const int g1 = min(G, static_cast<int>(blockIdx.y + 1) * gc);
    for (int g = blockIdx.y * gc + threadIdx.x; g < g1; g += blockDim.x) {
        cplx fh, fl;
        model_at(g, G, MH, rsm, invh, fh);
        model_at(g, G, ML, rsm + MH, invl, fl);
        const cplx d = fh - fl;
        md = fmax(md, hypot(d.re, d.im));
        mh = fmax(mh, hypot(fh.re, fh.im));
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        md = fmax(md, __shfl_xor_sync(0xffffffffu, md, off));
        mh = fmax(mh, __shfl_xor_sync(0xffffffffu, mh, off));
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) { red[0][wid] = md; red[1][wid] = mh; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { md = fmax(md, red[0][w]); mh = fmax(mh, red[1][w]); }
        md = fmax(md, red[0][0]);
        mh = fmax(mh, red[1][0]);
        out[2 * (static_cast<size_t>(blockIdx.y) * K + k)] = md;
        out[2 * (static_cast<size_t>(blockIdx.y) * K + k) + 1] = mh;
    }
}

__global__ void vf_chanerr_combine_kernel(int K, int S, const double* __restrict__ part, double* __restrict__ out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= K) return;
    double md = part[2 * k], mh = part[2 * k + 1];
    for (int s = 1; s < S; ++s) {
        md = fmax(md, part[2 * (static_cast<size_t>(s) * K + k)]);
        mh = fmax(mh, part[2 * (static_cast<size_t>(s) * K + k) + 1]);
    }
    out[2 * k] = md;
    out[2 * k + 1] = mh;
}

__global__ void __launch_bounds__(1024)
vf_select_kernel(int G, int MH, int ML, const cplx* __restrict__ rh, const cplx* __restrict__ rl, size_t sm_h,
                 size_t sm_l, const cplx* __restrict__ invh, const cplx* __restrict__ invl, const cplx* __restrict__ grid,
                 int nex, const double* __restrict__ ex_im, double radius, int* __restrict__ out) {
    extern __shared__ double exs[];
    __shared__ cplx r[512];
    __shared__ double bv[32];
    __shared__ int bi[32];
    for (int i = threadIdx.x; i < nex; i += blockDim.x) exs[i] = ex_im[i];
    for (int m = threadIdx.x; m < MH; m += blockDim.x) r[m] = rh[m * sm_h];
    for (int m = threadIdx.x; m < ML; m += blockDim.x) r[MH + m] = rl[m * sm_l];
    __syncthreads();
    double best = -1.0;
    int bidx = 0x7fffffff;
    for (int g = threadIdx.x; g < G; g += blockDim.x) {
        const double im = grid[g].im;
        bool excl = false;
        for (int e = 0; e < nex && !excl; ++e) excl = fabs(im - exs[e]) < radius;
        if (excl) continue;
        cplx fh, fl;
        model_at(g, G, MH, r, invh, fh);
        model_at(g, G, ML, r + MH, invl, fl);
        const cplx d = fh - fl;
        const double v = hypot(d.re, d.im);
        if (v > best) { best = v; bidx = g; }  // g increases per thread: first max kept
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bidx, off);
        if (ov > best || (ov == best && oi < bidx)) { best = ov; bidx = oi; }
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) { bv[wid] = best; bi[wid] = bidx; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
            if (bv[w] > bv[0] || (bv[w] == bv[0] && bi[w] < bi[0])) { bv[0] = bv[w]; bi[0] = bi[w]; }
        out[0] = bv[0] >= 0.0 ? bi[0] : -1;
    }
}

// channel errors -> E2 over the test positions, the worst ORF channel
// (afs.cpp:151-160: first strict max in ORF order) and the first channel with
// an identically zero high-order fit (afs.cpp:138-141). One CTA.
__global__ void __launch_bounds__(1024)
afs_reduce_errors_kernel(int K, const double* __restrict__ ce /*[k][2]*/, int KT, const int* __restrict__ test_pos,
                         int KO, const int* __restrict__ orf_pos, AfsErrReduce* __restrict__ out) {
    __shared__ double bv[32];
    __shared__ int bi[32];
    __shared__ int zero_k;
    if (threadIdx.x == 0) zero_k = 0x7fffffff;
    __syncthreads();
    for (int k = threadIdx.x; k < K; k += blockDim.x)
        if (ce[2 * k + 1] == 0.0) atomicMin(&zero_k, k);
    double e2 = -INFINITY;  // std::max(e2, e) keeps e2 on NaN, as fmax does
    for (int q = threadIdx.x; q < KT; q += blockDim.x) {
        const int k = test_pos[q];
        e2 = fmax(e2, ce[2 * k] / ce[2 * k + 1]);
    }
    double best = -1.0;  // (error, list index): larger error, then smaller index
    int bidx = 0x7fffffff;
    for (int q = threadIdx.x; q < KO; q += blockDim.x) {
        const int k = orf_pos[q];
        const double e = ce[2 * k] / ce[2 * k + 1];
        if (e > best) { best = e; bidx = q; }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        e2 = fmax(e2, __shfl_xor_sync(0xffffffffu, e2, off));
        const double ov = __shfl_xor_sync(0xffffffffu, best, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bidx, off);
        if (ov > best || (ov == best && oi < bidx)) { best = ov; bidx = oi; }
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __shared__ double be2[32];
    if (lane == 0) { bv[wid] = best; bi[wid] = bidx; be2[wid] = e2; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            if (bv[w] > bv[0] || (bv[w] == bv[0] && bi[w] < bi[0])) { bv[0] = bv[w]; bi[0] = bi[w]; }
            be2[0] = fmax(be2[0], be2[w]);
        }
        out->e2 = be2[0];
        out->kmax = orf_pos[bi[0] == 0x7fffffff ? 0 : bi[0]];
        out->zero_k = zero_k == 0x7fffffff ? -1 : zero_k;
    }
}

__global__ void vf_gather_channels_kernel(int K, int M, int KT, const cplx* __restrict__ src /*[m][K]*/,
                                          const int* __restrict__ pos, cplx* __restrict__ dst /*[m][KT]*/) {
    const size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<size_t>(M) * KT) return;
    const int m = static_cast<int>(idx / KT), q = static_cast<int>(idx % KT);
    dst[idx] = src[static_cast<size_t>(m) * K + pos[q]];
}

// identify_residues apply, bulk-copy fed (default for J <= 64, M <= 64 per
// slice): X (M x K) = W (M x 2J) B (2J x K), computed transposed as
// X^T = B^T W^T. One persistent CTA per SM walks 64-channel tiles; a producer
// warp streams each tile's J value rows (1 KB contiguous runs of
// values[j][k0..k0+63]) into a ST-deep shared-memory ring with cp.async.bulk
// (mbarrier transaction counts, no registers spent on the copy); 2*MT consumer
// warps each own one 8-pole m-tile of W — its fragments for all steps live in
// registers for the whole kernel — and one 32-channel half of the tile, reading
// value fragments from the ring (row stride 136 doubles: the two value rows a
// fragment spans land 16 banks apart). With channels as the DMMA's M side, a
// lane's two accumulators are poles 2 q, 2 q + 1 of one channel: both halves of
// a conjugate pair, packed without shuffles. Step counts divisible by four run
// as branch-free groups of four k-steps (16 DMMAs per group).
constexpr int kRtTile = 64;        // channels per tile
constexpr int kRtRow = 2 * kRtTile + 8;  // doubles per staged value row
template <int MT, int SP, int ST>
__global__ void __launch_bounds__(32 + 64 * MT, 1)
vf_residue_tma_kernel(int J, int K, int M, int P, const cplx* __restrict__ vals, const double* __restrict__ W,
                      cplx* __restrict__ res, int heads) {
    static_assert(SP % 4 == 0, "step capacity in groups of four");
    extern __shared__ double rtm_raw[];
    double* ring = rtm_raw;
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + static_cast<size_t>(ST) * J * kRtRow);
    uint64_t* empty = full + ST;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int m0 = blockIdx.y * 64;
    const int ntiles = (K + kRtTile - 1) / kRtTile;
    const int Q = 2 * J;
    constexpr int kConsumers = 2 * MT;
    if (tid == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumers);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (warp == 0) {  // producer
        int i = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
            const int s = i % ST;
            if (i >= ST) mbar_wait(&empty[s], ((i / ST) - 1) & 1);
            fds_jitter(i);
            const int k0 = t * kRtTile;
            const unsigned bytes = static_cast<unsigned>(min(kRtTile, K - k0)) * 16u;
            if (lane == 0) mbar_expect_tx(&full[s], bytes * J);
            __syncwarp();
            double* st = ring + static_cast<size_t>(s) * J * kRtRow;
            for (int j = lane; j < J; j += 32)
                bulk_load(st + j * kRtRow, vals + static_cast<size_t>(j) * K + k0, bytes, &full[s]);
        }
        return;
    }
    const int cw = warp - 1, mt = cw >> 1, half = cw & 1;
    const int q_l = lane & 3, n_l = lane >> 2;
    const int j0 = q_l >> 1, part = q_l & 1;
    // W fragments of this warp's m-tile for every step: W[m][4 st + q_l] (zero padded)
    double fw[SP];
    {
        const int mrow = m0 + mt * 8 + n_l;
#pragma unroll
        for (int st = 0; st < SP; ++st) {
            const int q = 4 * st + q_l;
            fw[st] = (mrow < M && q < Q) ? W[static_cast<size_t>(mrow) * Q + q] : 0.0;
        }
    }
    const int steps = (J + 1) / 2;
    const bool grouped = steps % 4 == 0;
    const int mb = m0 + mt * 8 + 2 * q_l;  // this lane's pole rows mb, mb + 1
    int i = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
        const int s = i % ST;
        mbar_wait(&full[s], (i / ST) & 1);
        const double* st_base = ring + static_cast<size_t>(s) * J * kRtRow + (half * 32 + n_l) * 2 + part;
        double acc[4][2];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
        // value fragment of step st, channel group nt: row 2 st + j0 (the odd-J tail
        // row meets zero W columns; clamp the read)
        if (grouped) {
#pragma unroll
            for (int g = 0; g < SP / 4; ++g) {
                if (4 * g < steps) {
                    double fv[4][4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const double* b = st_base + (2 * (4 * g + u) + j0) * kRtRow;
#pragma unroll
                        for (int nt = 0; nt < 4; ++nt) fv[u][nt] = b[nt * 16];
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u)
#pragma unroll
                        for (int nt = 0; nt < 4; ++nt) dmma_v(acc[nt][0], acc[nt][1], fv[u][nt], fw[4 * g + u]);
                }
            }
        } else {
#pragma unroll
            for (int st = 0; st < SP; ++st) {
                if (st < steps) {
                    const double* b = st_base + min(2 * st + j0, J - 1) * kRtRow;
                    double fv[4];
#pragma unroll
                    for (int nt = 0; nt < 4; ++nt) fv[nt] = b[nt * 16];
#pragma unroll
                    for (int nt = 0; nt < 4; ++nt) dmma_v(acc[nt][0], acc[nt][1], fv[nt], fw[st]);
                }
            }
        }
        fds_jitter(i);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        // canonical packing: rows m (even, < 2P) and m + 1 form one conjugate pair
        // (m + 1 holds the conjugate); rows >= 2P are real poles
        const int k0 = t * kRtTile + half * 32;
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
            const int k = k0 + nt * 8 + n_l;
            if (k >= K) continue;
            const double x = acc[nt][0], y = acc[nt][1];
            double2* dst = reinterpret_cast<double2*>(res) + static_cast<size_t>(mb) * K + k;
            if (mb < 2 * P) {
                __stcs(dst, make_double2(x, y));
                if (!heads) __stcs(dst + K, make_double2(x, -y));
            } else {
                if (mb < M) __stcs(dst, make_double2(x, 0.0));
                if (mb + 1 < M) __stcs(dst + K, make_double2(y, 0.0));
            }
        }
    }
}

// out[g*K + k] = sum_m res[k*M + m] / (s_g - a_m) (vecfit.cpp:490-509); *hit is
// set when some s_g equals a pole exactly (the reference's NumericError).
__global__ void vf_eval_kernel(int M, const cplx* __restrict__ poles, int K, const cplx* __restrict__ res, int G,
                               const cplx* __restrict__ s, cplx* __restrict__ out, int* __restrict__ hit) {
    const size_t idx = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<size_t>(G) * K) return;
    const int g = static_cast<int>(idx / K), k = static_cast<int>(idx % K);
    const cplx sg = s[g];
    cplx acc = mk(0.0, 0.0);
    for (int m = 0; m < M; ++m) {
        const cplx d = sg - poles[m];
        if (d.re == 0.0 && d.im == 0.0) {
            *hit = 1;
            return;
        }
        acc = acc + cdiv(res[static_cast<size_t>(k) * M + m], d);
    }
    out[idx] = acc;
}

// fit_error_evf (vecfit.cpp:511-526) for one channel: one CTA, fixed-order
// tree reduction of sum |fit - data|^2 and sum |data|^2 over the J samples.
__global__ void vf_evf_kernel(int M, const cplx* __restrict__ poles, const cplx* __restrict__ res_k, int J,
                              const cplx* __restrict__ s, const cplx* __restrict__ data, int dstride,
                              double* __restrict__ out2, int* __restrict__ hit) {
    __shared__ double rn[256], rd[256];
    double num = 0.0, den = 0.0;
    for (int j = threadIdx.x; j < J; j += blockDim.x) {
        cplx acc = mk(0.0, 0.0);
        for (int m = 0; m < M; ++m) {
            const cplx d = s[j] - poles[m];
            if (d.re == 0.0 && d.im == 0.0) { *hit = 1; break; }
            acc = acc + cdiv(res_k[m], d);
        }
        const cplx v = data[static_cast<size_t>(j) * dstride];
        num += abs2(acc - v);
        den += abs2(v);
    }
    rn[threadIdx.x] = num;
    rd[threadIdx.x] = den;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            rn[threadIdx.x] += rn[threadIdx.x + w];
            rd[threadIdx.x] += rd[threadIdx.x + w];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out2[0] = rn[0];
        out2[1] = rd[0];
    }
}

void vf_eval_model(const std::vector<Cx>& poles, const Cx* res_km, int K, const std::vector<Cx>& s, Cx* out) {
    const int M = static_cast<int>(poles.size()), G = static_cast<int>(s.size());
    if (G == 0 || K == 0) return;
    auto& cx = VfContext::get();
    const size_t nres = static_cast<size_t>(K) * M, nout = static_cast<size_t>(G) * K;
    cplx* d = static_cast<cplx*>(cx.values.get(sizeof(cplx) * (M + nres + G + nout) + sizeof(int)));
    cplx *dp = d, *dr = dp + M, *ds = dr + nres, *dout = ds + G;
    int* dhit = reinterpret_cast<int*>(dout + nout);
    FDS_CUDA(cudaMemcpyAsync(dp, poles.data(), M * sizeof(cplx), cudaMemcpyHostToDevice, cx.st));
    FDS_CUDA(cudaMemcpyAsync(dr, res_km, nres * sizeof(cplx), cudaMemcpyHostToDevice, cx.st));
    FDS_CUDA(cudaMemcpyAsync(ds, s.data(), G * sizeof(cplx), cudaMemcpyHostToDevice, cx.st));
    FDS_CUDA(cudaMemsetAsync(dhit, 0, sizeof(int), cx.st));
    FDS_LAUNCH(vf_eval_kernel, static_cast<unsigned>((nout + 255) / 256), 256, 0, cx.st, M, dp, K, dr, G, ds, dout, dhit);
    int hit = 0;
    FDS_CUDA(cudaMemcpyAsync(&hit, dhit, sizeof(int), cudaMemcpyDeviceToHost, cx.st));
    FDS_CUDA(cudaMemcpyAsync(out, dout, nout * sizeof(cplx), cudaMemcpyDeviceToHost, cx.st));
    FDS_CUDA(cudaStreamSynchronize(cx.st));
    if (hit) throw NumericError("eval_model: s coincides with a pole");
}

double vf_fit_error_evf(const std::vector<Cx>& poles, const Cx* res_k, const std::vector<Cx>& s, const Cx* data,
                        int dstride) {
    const int M = static_cast<int>(poles.size()), J = static_cast<int>(s.size());
    if (J == 0) throw ValidationError("fit_error_evf: no samples");
    auto& cx = VfContext::get();
    cplx* d = static_cast<cplx*>(cx.values.get(sizeof(cplx) * (2 * M + 2 * static_cast<size_t>(J) + 2)));
    cplx *dp = d, *dr = dp + M, *ds = dr + M, *dd = ds + J;
    double* d2 = reinterpret_cast<double*>(dd + J);
    int* dhit = reinterpret_cast<int*>(d2 + 2);
    std::vector<Cx> col(J);
    for (int j = 0; j < J; ++j) col[j] = data[static_cast<size_t>(j) * dstride];
    FDS_CUDA(cudaMemcpyAsync(dp, poles.data(), M * sizeof(cplx), cudaMemcpyHostToDevice, cx.st));
    FDS_CUDA(cudaMemcpyAsync(dr, res_k, M * sizeof(cplx), cudaMemcpyHostToDevice, cx.st));
    FDS_CUDA(cudaMemcpyAsync(ds, s.data(), J * sizeof(cplx), cudaMemcpyHostToDevice, cx.st));
    FDS_CUDA(cudaMemcpyAsync(dd, col.data(), J * sizeof(cplx), cudaMemcpyHostToDevice, cx.st));
    FDS_CUDA(cudaMemsetAsync(dhit, 0, sizeof(int), cx.st));
    FDS_LAUNCH(vf_evf_kernel, 1, 256, 0, cx.st, M, dp, dr, J, ds, dd, 1, d2, dhit);
    double h2[2];
    int hit = 0;
    FDS_CUDA(cudaMemcpyAsync(h2, d2, sizeof(h2), cudaMemcpyDeviceToHost, cx.st));
    FDS_CUDA(cudaMemcpyAsync(&hit, dhit, sizeof(int), cudaMemcpyDeviceToHost, cx.st));
    FDS_CUDA(cudaStreamSynchronize(cx.st));
    if (hit) throw NumericError("eval_model: s coincides with a pole");
    if (h2[1] == 0.0) throw NumericError("fit_error_evf: zero-norm sample data");
    return std::sqrt(h2[0] / h2[1]);
}

// ------------------------------------------------------------------ host drivers
namespace {

template <class T>
T* dev(VfContext::Buf& b, size_t count) {
    return static_cast<T*>(b.get(count * sizeof(T)));
}

// vf_chanerr_kernel over K channels, the grid split into S chunks when K alone
// cannot fill the GPU (the AFS fits have K = 5 ... 48 channels).
void chanerr_run(VfContext& cx, cudaStream_t st, int G, int MH, int ML, int K, const cplx* rh, const cplx* rl,
                 size_t sk_h, size_t sm_h, size_t sk_l, size_t sm_l, const cplx* invh, const cplx* invl,
                 double* out) {
    const int S = std::max(1, std::min(std::min(16, G), ceil_div(4 * device_info().sms, K)));
    const size_t smem = (MH + ML) * sizeof(cplx);
    if (S == 1) {
        FDS_LAUNCH(vf_chanerr_kernel, K, 256, smem, st, G, MH, ML, K, rh, rl, sk_h, sm_h, sk_l, sm_l, invh, invl, out);
        return;
    }
    double* part = dev<double>(cx.chanerr, 2 * static_cast<size_t>(K) * S);
    FDS_LAUNCH(vf_chanerr_kernel, dim3(K, S), 256, smem, st, G, MH, ML, K, rh, rl, sk_h, sm_h, sk_l, sm_l, invh,
               invl, part);
    FDS_LAUNCH(vf_chanerr_combine_kernel, ceil_div(K, 128), 128, 0, st, K, S, part, out);
}

// Does any grid point coincide with a pole (eval_model's collision check,
// vecfit.cpp:494-496, over every (grid point, pole) pair)? Sorted-grid lookup
// instead of the G x M scan (4096 x 240 pairs per AFS iteration).
bool grid_hits_pole(const std::vector<Cx>& grid, const std::vector<Cx>& a, const std::vector<Cx>& b) {
    auto less = [](const Cx& x, const Cx& y) { return x.real() < y.real() || (x.real() == y.real() && x.imag() < y.imag()); };
    std::vector<Cx> g(grid);
    std::sort(g.begin(), g.end(), less);
    for (const auto* ps : {&a, &b})
        for (const Cx& p : *ps)
            if (std::binary_search(g.begin(), g.end(), p, less)) return true;
    return false;
}

}  // namespace

RelocResult vf_relocate(const std::vector<Cx>& s, const Cx* values, int K, const std::vector<Cx>& poles_in) {
    // vecfit.cpp:188-354
    const int J = static_cast<int>(s.size());
    const int M = static_cast<int>(poles_in.size());
    if (J == 0) throw ValidationError("relocate_poles: no samples");
    if (K < 1) throw ValidationError("relocate_poles: no channels");
    if (2 * J < M + 1) throw ValidationError("relocate_poles: too few samples for the order");
    require_distinct(s);
    const std::vector<Cx> poles = canonical_order(poles_in);
    const std::vector<Cx> phi = basis(s, poles);
    std::vector<double> cscale(M), sscale(M);
    for (int m = 0; m < M; ++m) {
        double n2 = 0.0, sq = 0.0;
        for (int j = 0; j < J; ++j) n2 += std::norm(phi[static_cast<size_t>(m) * J + j]);
        for (int k = 0; k < K; ++k)
            for (int j = 0; j < J; ++j) sq += std::norm(values[static_cast<size_t>(j) * K + k] * phi[static_cast<size_t>(m) * J + j]);
        const double n = std::sqrt(n2);
        cscale[m] = n > 0.0 ? 1.0 / n : 1.0;
        sscale[m] = sq > 0.0 ? 1.0 / std::sqrt(sq) : 1.0;
    }
    auto& cx = VfContext::get();
    const int rows = 2 * J, cols = 2 * M + 1;
    const int top = std::min(2 * M, rows), red = std::max(0, top - M);
    cplx* dvals = dev<cplx>(cx.values, static_cast<size_t>(J) * K);
    cplx* dphi = dev<cplx>(cx.phi, static_cast<size_t>(J) * M);
    double* dsc = dev<double>(cx.misc, 2 * static_cast<size_t>(M));
    double* dr22 = dev<double>(cx.resid, static_cast<size_t>(K) * red * M + static_cast<size_t>(K) * red + K);
    double* dbeta = dr22 + static_cast<size_t>(K) * red * M;
    double* dtail = dbeta + static_cast<size_t>(K) * red;
    FDS_CUDA(cudaMemcpyAsync(dvals, values, sizeof(cplx) * J * K, cudaMemcpyHostToDevice, cx.st));
    FDS_CUDA(cudaMemcpyAsync(dphi, phi.data(), sizeof(cplx) * J * M, cudaMemcpyHostToDevice, cx.st));
    FDS_CUDA(cudaMemcpyAsync(dsc, cscale.data(), sizeof(double) * M, cudaMemcpyHostToDevice, cx.st));
    FDS_CUDA(cudaMemcpyAsync(dsc + M, sscale.data(), sizeof(double) * M, cudaMemcpyHostToDevice, cx.st));
    const size_t mat_bytes = static_cast<size_t>(rows) * cols * sizeof(double);
    double* gwork = nullptr;
    size_t smem = mat_bytes;
    if (mat_bytes > device_info().smem_optin - 4096) {
        gwork = dev<double>(cx.qr, static_cast<size_t>(rows) * cols * K);
        smem = 0;
    } else {
        ensure_dynamic_smem(reinterpret_cast<const void*>(vf_reloc_qr_kernel), smem);
    }
    FDS_LAUNCH(vf_reloc_qr_kernel, K, kRelocQrThreads, smem, cx.st, J, M, K, dvals, dphi, dsc, dsc + M, gwork, dr22, dbeta,
               dtail);
    // stacked sigma least squares (vecfit.cpp:281-285) and the per-channel RMS
    // (:287-295) on the device; only y, the RMS and the rank come back
    double* dy = dev<double>(cx.lsq_io, static_cast<size_t>(M) + K + 2 * sizeof(VfLsqStatus) / sizeof(double) + 2);
    double* drms = dy + M;
    auto* dstat = reinterpret_cast<VfLsqStatus*>(drms + K);
    vf_lsq_stacked_launch(K, red, M, dr22, dbeta, dy, dstat, cx.st);
    vf_reloc_rms_launch(K, red, M, J, dr22, dbeta, dtail, dy, drms, cx.st);
    std::vector<double> hy(static_cast<size_t>(M) + K);
    VfLsqStatus hst;
    FDS_CUDA(cudaMemcpyAsync(&hst, dstat, sizeof(hst), cudaMemcpyDeviceToHost, cx.st));
    FDS_CUDA(cudaMemcpyAsync(hy.data(), dy, hy.size() * sizeof(double), cudaMemcpyDeviceToHost, cx.st));
    FDS_CUDA(cudaStreamSynchronize(cx.st));
    if (hst.rank < M) throw NumericError("relocate_poles: rank-deficient least-squares system");
    const std::vector<double> y(hy.begin(), hy.begin() + M);
    RelocResult out;
    out.rms.assign(hy.begin() + M, hy.end());
    // zeros of sigma: eig(blockdiag(poles) - b c^T) (vecfit.cpp:297-324)
    struct {
        int m;
        std::vector<double> v;
        double& at(int i, int j) { return v[static_cast<size_t>(j) * m + i]; }
    } h{M, std::vector<double>(static_cast<size_t>(M) * M, 0.0)};
    std::vector<double> bv(M), cr(M);
    for (int m = 0; m < M;) {
        if (poles[m].imag() != 0.0) {
            h.at(m, m) = poles[m].real();
            h.at(m, m + 1) = poles[m].imag();
            h.at(m + 1, m) = -poles[m].imag();
            h.at(m + 1, m + 1) = poles[m].real();
            bv[m] = 2.0;
            bv[m + 1] = 0.0;
            cr[m] = sscale[m] * y[m];
            cr[m + 1] = sscale[m + 1] * y[m + 1];
            m += 2;
        } else {
            h.at(m, m) = poles[m].real();
            bv[m] = 1.0;
            cr[m] = sscale[m] * y[m];
            m += 1;
        }
    }
    for (int i = 0; i < M; ++i)
        for (int c = 0; c < M; ++c) h.at(i, c) -= bv[i] * cr[c];
    std::vector<Cx> ev;
    if (!eig::eigenvalues(M, h.v.data(), ev)) throw NumericError("relocate_poles: eigenvalue iteration failed");
    std::vector<Cx> heads, reals;
    int neg = 0;
    for (Cx e : ev) {
        if (e.imag() > 0.0) heads.push_back(e);
        else if (e.imag() < 0.0) ++neg;
        else reals.push_back(e);
    }
    if (neg != static_cast<int>(heads.size())) throw NumericError("relocate_poles: eigenvalues not conjugate-paired");
    for (Cx hd : heads) { out.poles.push_back(hd); out.poles.push_back(std::conj(hd)); }
    out.poles.insert(out.poles.end(), reals.begin(), reals.end());
    out.movement = movement_of(poles, out.poles);
    return out;
}

void vf_residues_device(const std::vector<Cx>& s, const cplx* values_dev, int K, const std::vector<Cx>& poles,
                        cplx* res_dev, double* rms_dev, cudaStream_t st, bool heads_only) {
    // vecfit.cpp:356-408 for all channels: factor [Re Φ; Im Φ] (column-scaled)
    // once on the host, apply its solve operator on the device.
    const int J = static_cast<int>(s.size()), M = static_cast<int>(poles.size());
    if (J < 1) throw ValidationError("identify_residues: no samples");
    if (2 * J < M) throw ValidationError("identify_residues: too few samples for the order");
    require_distinct(s);
    const int rows = 2 * J;
    auto& cx = VfContext::get();
    // The solve operator depends only on (s, poles): the last one stays in HBM
    // and is reused when a call repeats them bit for bit (e.g. the final
    // all-channel fit of run_afs after the last iteration's high-order fit,
    // afs.cpp:379-393).
    std::vector<double> key;
    key.reserve(2 + 2 * (J + M));
    key.push_back(J);
    key.push_back(M);
    for (Cx x : s) { key.push_back(x.real()); key.push_back(x.imag()); }
    for (Cx x : poles) { key.push_back(x.real()); key.push_back(x.imag()); }
    double* dW = dev<double>(cx.W, static_cast<size_t>(M) * rows);
    const bool cached = cx.w_valid && cx.w_key.size() == key.size() &&
                        std::memcmp(cx.w_key.data(), key.data(), key.size() * sizeof(double)) == 0;
    if (!cached) {
        cx.w_valid = false;
        const std::vector<Cx> phi = basis(s, poles);
        std::vector<double> a(static_cast<size_t>(rows) * M), scale(M);  // column-major [Re Phi; Im Phi]
        for (int m = 0; m < M; ++m) {
            double n2 = 0.0;
            for (int j = 0; j < J; ++j) {
                const Cx v = phi[static_cast<size_t>(m) * J + j];
                a[static_cast<size_t>(m) * rows + 2 * j] = v.real();
                a[static_cast<size_t>(m) * rows + 2 * j + 1] = v.imag();
                n2 += v.real() * v.real() + v.imag() * v.imag();
            }
            const double n = std::sqrt(n2);
            scale[m] = n > 0.0 ? 1.0 / n : 1.0;
            for (int i = 0; i < rows; ++i) a[static_cast<size_t>(m) * rows + i] *= scale[m];
        }
        // one shared pivoted QR (vecfit.cpp:389) turned into the solve operator
        // W (M x 2J, rows pre-scaled) on the device
        double* da = dev<double>(cx.lsq_io, a.size() + M + 2 * sizeof(VfLsqStatus) / sizeof(double) + 2);
        double* dscale = da + a.size();
        auto* dstat = reinterpret_cast<VfLsqStatus*>(dscale + M);
        FDS_CUDA(cudaMemcpyAsync(da, a.data(), a.size() * sizeof(double), cudaMemcpyHostToDevice, st));
        FDS_CUDA(cudaMemcpyAsync(dscale, scale.data(), M * sizeof(double), cudaMemcpyHostToDevice, st));
        if (vf_lsq_fits(rows, M, false))
            vf_lsq_launch(rows, M, da, 1, rows, nullptr, nullptr, dW, dscale, dstat, st);
        else
            vf_lsq_operator_large(rows, M, da, dscale, dW, dstat, st);
        VfLsqStatus hst;
        FDS_CUDA(cudaMemcpyAsync(&hst, dstat, sizeof(hst), cudaMemcpyDeviceToHost, st));
        FDS_CUDA(cudaStreamSynchronize(st));
        if (hst.rank < M) throw NumericError("identify_residues: rank-deficient least-squares system");
        cx.w_key = std::move(key);
        cx.w_valid = true;
    }
    const int P = pair_count(poles);
    const size_t smem = static_cast<size_t>(kResChunk) * 2 * J * sizeof(double);
    ensure_dynamic_smem(reinterpret_cast<const void*>(vf_residue_kernel), smem);
    const int PF = (((J + 1) / 2) % 5 == 0) ? 5 : 4;  // prefetch depth dividing the step count when possible
    const size_t msmem = static_cast<size_t>(4 * res_steps(J, PF)) * kRmS * sizeof(double);
    cudaEvent_t pe;
    profiler().begin(st, kProfVfResidue, 0.0, pe);
    const int hf = heads_only ? 1 : 0;
    const int mt_all = std::min(8, ceil_div(M, 8));
    const size_t row_bytes = static_cast<size_t>(J) * kRtRow * sizeof(double);
    const int rt_st = std::min<int>(4, static_cast<int>((device_info().smem_optin - 1024) / std::max<size_t>(row_bytes, 1)));
    if (J <= 64 && rt_st >= 2 && !std::getenv("FDSWEEP_RESIDUE_LEGACY")) {
        const size_t tsmem = rt_st * row_bytes + 2 * 4 * sizeof(uint64_t);
        const int ctas = std::min(ceil_div(K, kRtTile), device_info().sms);
        auto go = [&](auto kern) {
            ensure_dynamic_smem(reinterpret_cast<const void*>(kern), tsmem);
            FDS_LAUNCH(kern, dim3(ctas, ceil_div(M, 64)), 32 + 64 * mt_all, tsmem, st, J, K, M, P, values_dev, dW,
                       res_dev, hf);
        };
        auto by_sp = [&](auto mtc) {
            constexpr int MTc = decltype(mtc)::value;
            const int sp = (J + 1) / 2;
            auto by_st = [&](auto spc) {
                constexpr int SPc = decltype(spc)::value;
                if (rt_st >= 4) go(vf_residue_tma_kernel<MTc, SPc, 4>);
                else if (rt_st == 3) go(vf_residue_tma_kernel<MTc, SPc, 3>);
                else go(vf_residue_tma_kernel<MTc, SPc, 2>);
            };
            if (sp <= 8) by_st(std::integral_constant<int, 8>{});
            else if (sp <= 16) by_st(std::integral_constant<int, 16>{});
            else if (sp <= 24) by_st(std::integral_constant<int, 24>{});
            else by_st(std::integral_constant<int, 32>{});
        };
        switch (mt_all) {
            case 1: by_sp(std::integral_constant<int, 1>{}); break;
            case 2: by_sp(std::integral_constant<int, 2>{}); break;
            case 3: by_sp(std::integral_constant<int, 3>{}); break;
            case 4: by_sp(std::integral_constant<int, 4>{}); break;
            case 5: by_sp(std::integral_constant<int, 5>{}); break;
            case 6: by_sp(std::integral_constant<int, 6>{}); break;
            case 7: by_sp(std::integral_constant<int, 7>{}); break;
            default: by_sp(std::integral_constant<int, 8>{}); break;
        }
    } else if (msmem <= device_info().smem_optin - 1024) {
        const int ctas = std::min(ceil_div(K, 4 * 8 * kResNI), 8 * device_info().sms);
        const int mt = std::min(8, ceil_div(M, 8));  // m-tiles of the first (largest) slice
        auto go = [&](auto kern) {
            ensure_dynamic_smem(reinterpret_cast<const void*>(kern), msmem);
            FDS_LAUNCH(kern, dim3(ctas, ceil_div(M, 64)), 128, msmem, st, J, K, M, P, values_dev, dW, res_dev, hf);
        };
        if (PF == 5) {
            if (mt <= 2) go(vf_residue_mma_kernel<2, 5>);
            else if (mt <= 4) go(vf_residue_mma_kernel<4, 5>);
            else if (mt <= 6) go(vf_residue_mma_kernel<6, 5>);
            else go(vf_residue_mma_kernel<8, 5>);
        } else {
            if (mt <= 2) go(vf_residue_mma_kernel<2, 4>);
            else if (mt <= 4) go(vf_residue_mma_kernel<4, 4>);
            else if (mt <= 6) go(vf_residue_mma_kernel<6, 4>);
            else go(vf_residue_mma_kernel<8, 4>);
        }
    } else {
        dim3 g(ceil_div(K, kResThreads), ceil_div(M, kResChunk));
        FDS_LAUNCH(vf_residue_kernel, g, kResThreads, smem, st, J, K, M, P, values_dev, dW, res_dev, hf);
    }
    // bytes moved: values 16 J + residues 16 M (all rows) or 8 M (pair heads + reals) per channel
    profiler().end(st, pe, kProfVfResidue, static_cast<double>(K) * (16.0 * J + (heads_only ? 8.0 : 16.0) * M));
    if (rms_dev) {
        std::vector<Cx> invd(static_cast<size_t>(M) * J);
        for (int m = 0; m < M; ++m)
            for (int j = 0; j < J; ++j) invd[static_cast<size_t>(m) * J + j] = 1.0 / (s[j] - poles[m]);
        cplx* dinv = dev<cplx>(cx.phi, invd.size());
        FDS_CUDA(cudaMemcpyAsync(dinv, invd.data(), invd.size() * sizeof(cplx), cudaMemcpyHostToDevice, st));
        if (K < 4 * device_info().sms * 128 / 16)  // fewer channels than ~1/16 of a thread per SM slot
            FDS_LAUNCH(vf_rms_cta_kernel, K, 128, 0, st, J, K, M, values_dev, res_dev, dinv, rms_dev);
        else
            FDS_LAUNCH(vf_rms_kernel, ceil_div(K, 128), 128, 0, st, J, K, M, values_dev, res_dev, dinv, rms_dev);
    }
}

namespace {

// vecfit.cpp:410-462: validation, starting poles and the relocation loop on the
// ORF channels (host values ov [j][KO]); returns the relocated poles.
std::vector<Cx> fit_poles(const std::vector<Cx>& s, const Cx* ov, int KO, int order, int n_reloc, FitReportC& r) {
    double band = 0.0;
    for (Cx x : s) band = std::max(band, std::abs(x.imag()));
    if (band == 0.0)
        for (Cx x : s) band = std::max(band, std::abs(x));
    if (band == 0.0) throw ValidationError("vector_fit: samples carry no frequency band");
    std::vector<Cx> poles = start_poles(band, order);
    RelocResult rr;
    for (int it = 0; it < n_reloc; ++it) {
        rr = vf_relocate(s, ov, KO, poles);
        poles = rr.poles;
        r.iterations = it + 1;
        r.movement = rr.movement;
        if (rr.movement < 1e-8) break;
    }
    r.reloc_rms = rr.rms;
    return poles;
}

void check_fit_args(int J, int K, const std::vector<int>& orf, int order, int n_reloc) {
    if (J == 0) throw ValidationError("vector_fit: no samples");
    if (order < 1) throw ValidationError("vector_fit: order must be >= 1");
    if (order >= 2 * J) throw ValidationError("vector_fit: order too high for the sample count");
    if (n_reloc < 1) throw ValidationError("vector_fit: n_relocations must be >= 1");
    if (orf.empty()) throw ValidationError("vector_fit: ORF channel set is empty");
    for (int k : orf)
        if (k < 0 || k >= K) throw ValidationError("vector_fit: ORF channel index out of range");
}

}  // namespace

std::vector<Cx> vf_vector_fit_device(const std::vector<Cx>& s, const Cx* values_orf, const cplx* values_dev, int K,
                                     const std::vector<int>& orf, int order, int n_reloc, cplx* res_dev,
                                     cudaStream_t st) {
    const int J = static_cast<int>(s.size());
    check_fit_args(J, K, orf, order, n_reloc);
    FitReportC r;
    const std::vector<Cx> canon = canonical_order(fit_poles(s, values_orf, static_cast<int>(orf.size()), order, n_reloc, r));
    vf_residues_device(s, values_dev, K, canon, res_dev, nullptr, st);
    return canon;
}

void vf_vector_fit(const std::vector<Cx>& s, const Cx* values, int K, const std::vector<int>& orf, int order,
                   int n_reloc, std::vector<Cx>& poles, std::vector<Cx>& res_km, FitReportC* rep) {
    // vecfit.cpp:410-488
    const int J = static_cast<int>(s.size());
    check_fit_args(J, K, orf, order, n_reloc);
    const int KO = static_cast<int>(orf.size());
    std::vector<Cx> ov(static_cast<size_t>(J) * KO);
    for (int j = 0; j < J; ++j)
        for (int q = 0; q < KO; ++q) ov[static_cast<size_t>(j) * KO + q] = values[static_cast<size_t>(j) * K + orf[q]];
    FitReportC r;
    poles = fit_poles(s, ov.data(), KO, order, n_reloc, r);
    // residues for every channel on the device
    const std::vector<Cx> canon = canonical_order(poles);
    auto& cx = VfContext::get();
    cplx* dvals = dev<cplx>(cx.values, static_cast<size_t>(J) * K);
    cplx* dres = dev<cplx>(cx.out, static_cast<size_t>(order) * K);
    double* drms = dev<double>(cx.rms, K);
    FDS_CUDA(cudaMemcpyAsync(dvals, values, sizeof(cplx) * J * K, cudaMemcpyHostToDevice, cx.st));
    vf_residues_device(s, dvals, K, canon, dres, drms, cx.st);
    std::vector<Cx> rmk(static_cast<size_t>(order) * K);
    r.rms.assign(K, 0.0);
    FDS_CUDA(cudaMemcpyAsync(rmk.data(), dres, rmk.size() * sizeof(cplx), cudaMemcpyDeviceToHost, cx.st));
    FDS_CUDA(cudaMemcpyAsync(r.rms.data(), drms, K * sizeof(double), cudaMemcpyDeviceToHost, cx.st));
    FDS_CUDA(cudaStreamSynchronize(cx.st));
    // The reference keeps the relocation's pole order (heads in eigenvalue order),
    // and identify_residues canonicalises internally: for VF output they coincide.
    poles = canon;
    res_km.assign(static_cast<size_t>(K) * order, Cx(0, 0));
    for (int k = 0; k < K; ++k)
        for (int m = 0; m < order; ++m) res_km[static_cast<size_t>(k) * order + m] = rmk[static_cast<size_t>(m) * K + k];
    for (Cx p : poles) r.unstable += p.real() > 0.0;
    if (rep) *rep = std::move(r);
}

std::vector<double> vf_channel_errors(const std::vector<Cx>& ph, const std::vector<Cx>& rh, const std::vector<Cx>& pl,
                                      const std::vector<Cx>& rl, int K, const std::vector<Cx>& grid) {
    // afs.cpp:118-145
    if (grid.empty()) throw ValidationError("channel_errors: empty grid");
    const int G = static_cast<int>(grid.size()), MH = static_cast<int>(ph.size()), ML = static_cast<int>(pl.size());
    if (grid_hits_pole(grid, ph, pl)) throw NumericError("eval_model: s coincides with a pole");
    auto& cx = VfContext::get();
    cplx* dgrid = dev<cplx>(cx.misc2, G + MH + ML);
    cplx* dph = dgrid + G;
    cplx* dpl = dph + MH;
    cplx* dinv = dev<cplx>(cx.tab, static_cast<size_t>(G) * (MH + ML));
    cplx* dr = dev<cplx>(cx.resid, static_cast<size_t>(K) * (MH + ML));
    double* dout = dev<double>(cx.rms, 2 * static_cast<size_t>(K));
    FDS_CUDA(cudaMemcpyAsync(dgrid, grid.data(), G * sizeof(cplx), cudaMemcpyHostToDevice, cx.st));
    FDS_CUDA(cudaMemcpyAsync(dph, ph.data(), MH * sizeof(cplx), cudaMemcpyHostToDevice, cx.st));
    FDS_CUDA(cudaMemcpyAsync(dpl, pl.data(), ML * sizeof(cplx), cudaMemcpyHostToDevice, cx.st));
    FDS_CUDA(cudaMemcpyAsync(dr, rh.data(), static_cast<size_t>(K) * MH * sizeof(cplx), cudaMemcpyHostToDevice, cx.st));
    FDS_CUDA(cudaMemcpyAsync(dr + static_cast<size_t>(K) * MH, rl.data(), static_cast<size_t>(K) * ML * sizeof(cplx),
                             cudaMemcpyHostToDevice, cx.st));
    FDS_LAUNCH(vf_inv_table_kernel, ceil_div(G * MH, 256), 256, 0, cx.st, G, MH, dgrid, dph, dinv);
    FDS_LAUNCH(vf_inv_table_kernel, ceil_div(G * ML, 256), 256, 0, cx.st, G, ML, dgrid, dpl,
               dinv + static_cast<size_t>(G) * MH);
    cudaEvent_t pe;
    profiler().begin(cx.st, kProfChanErr, 0.0, pe);
    chanerr_run(cx, cx.st, G, MH, ML, K, dr, dr + static_cast<size_t>(K) * MH, size_t(MH), size_t(1), size_t(ML),
                size_t(1), dinv, dinv + static_cast<size_t>(G) * MH, dout);
    profiler().end(cx.st, pe, kProfChanErr, 8.0 * G * static_cast<double>(K) * (MH + ML));
    std::vector<double> h(2 * static_cast<size_t>(K));
    FDS_CUDA(cudaMemcpyAsync(h.data(), dout, h.size() * sizeof(double), cudaMemcpyDeviceToHost, cx.st));
    FDS_CUDA(cudaStreamSynchronize(cx.st));
    std::vector<double> e(K);
    for (int k = 0; k < K; ++k) {
        if (h[2 * k + 1] == 0.0)
            throw NumericError("channel_errors: channel " + std::to_string(k) + " has identically zero high-order fit");
        e[k] = h[2 * k] / h[2 * k + 1];
    }
    return e;
}

void vf_channel_errors_device(const std::vector<Cx>& ph, const cplx* rh_mk, const std::vector<Cx>& pl,
                              const cplx* rl_mk, int K, const std::vector<Cx>& grid, const int* test_pos_dev, int KT,
                              const int* orf_pos_dev, int KO, double* ce_dev, AfsErrReduce* red_dev,
                              cudaStream_t st) {
    // afs.cpp:118-145 with residues [m][k] in HBM; the per-channel ratios are
    // reduced on the device (E2, worst ORF channel, first zero-energy channel).
    if (grid.empty()) throw ValidationError("channel_errors: empty grid");
    const int G = static_cast<int>(grid.size()), MH = static_cast<int>(ph.size()), ML = static_cast<int>(pl.size());
    if (grid_hits_pole(grid, ph, pl)) throw NumericError("eval_model: s coincides with a pole");
    auto& cx = VfContext::get();
    std::vector<Cx> tabs(grid);
    tabs.insert(tabs.end(), ph.begin(), ph.end());
    tabs.insert(tabs.end(), pl.begin(), pl.end());
    cplx* dgrid = dev<cplx>(cx.misc2, G + MH + ML);
    cplx* dph = dgrid + G;
    cplx* dpl = dph + MH;
    cplx* dinv = dev<cplx>(cx.tab, static_cast<size_t>(G) * (MH + ML));
    FDS_CUDA(cudaMemcpyAsync(dgrid, tabs.data(), tabs.size() * sizeof(cplx), cudaMemcpyHostToDevice, st));
    FDS_LAUNCH(vf_inv_table_kernel, ceil_div(G * MH, 256), 256, 0, st, G, MH, dgrid, dph, dinv);
    FDS_LAUNCH(vf_inv_table_kernel, ceil_div(G * ML, 256), 256, 0, st, G, ML, dgrid, dpl,
               dinv + static_cast<size_t>(G) * MH);
    cudaEvent_t pe;
    profiler().begin(st, kProfChanErr, 0.0, pe);
    chanerr_run(cx, st, G, MH, ML, K, rh_mk, rl_mk, size_t(1), size_t(K), size_t(1), size_t(K), dinv,
                dinv + static_cast<size_t>(G) * MH, ce_dev);
    profiler().end(st, pe, kProfChanErr, 8.0 * G * static_cast<double>(K) * (MH + ML));
    FDS_LAUNCH(afs_reduce_errors_kernel, 1, 1024, 0, st, K, ce_dev, KT, test_pos_dev, KO, orf_pos_dev, red_dev);
    // tabs is read by the async copy above
    FDS_CUDA(cudaStreamSynchronize(st));
}

int vf_select_device(const std::vector<Cx>& ph, const cplx* rh_k, const std::vector<Cx>& pl, const cplx* rl_k,
                     size_t mstride, const std::vector<Cx>& grid, const std::vector<Cx>& existing, double radius,
                     cudaStream_t st) {
    // afs.cpp:162-187 for the worst ORF channel whose residues sit at rh_k[m*mstride]
    const int G = static_cast<int>(grid.size()), MH = static_cast<int>(ph.size()), ML = static_cast<int>(pl.size());
    if (MH + ML > 512) throw ValidationError("select_new_frequency: model order too large");
    auto& cx = VfContext::get();
    std::vector<Cx> tabs(grid);
    tabs.insert(tabs.end(), ph.begin(), ph.end());
    tabs.insert(tabs.end(), pl.begin(), pl.end());
    cplx* dgrid = dev<cplx>(cx.misc2, G + MH + ML);
    cplx* dph = dgrid + G;
    cplx* dpl = dph + MH;
    cplx* dinv = dev<cplx>(cx.tab, static_cast<size_t>(G) * (MH + ML));
    std::vector<double> exim(existing.size());
    for (size_t i = 0; i < existing.size(); ++i) exim[i] = existing[i].imag();
    double* dex = dev<double>(cx.misc, std::max<size_t>(exim.size(), 1) + 2);
    int* dsel = reinterpret_cast<int*>(dex + std::max<size_t>(exim.size(), 1));
    FDS_CUDA(cudaMemcpyAsync(dgrid, tabs.data(), tabs.size() * sizeof(cplx), cudaMemcpyHostToDevice, st));
    if (!exim.empty())
        FDS_CUDA(cudaMemcpyAsync(dex, exim.data(), exim.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    FDS_LAUNCH(vf_inv_table_kernel, ceil_div(G * MH, 256), 256, 0, st, G, MH, dgrid, dph, dinv);
    FDS_LAUNCH(vf_inv_table_kernel, ceil_div(G * ML, 256), 256, 0, st, G, ML, dgrid, dpl,
               dinv + static_cast<size_t>(G) * MH);
    const int nex = static_cast<int>(exim.size());
    const size_t smem = std::max<size_t>(nex, 1) * sizeof(double);
    if (smem > 48 * 1024) {
        FDS_CUDA(cudaFuncSetAttribute(vf_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(std::min(smem, device_info().smem_optin - 16 * 1024))));
    }
    FDS_LAUNCH(vf_select_kernel, 1, 1024, smem, st, G, MH, ML, rh_k, rl_k, mstride, mstride, dinv,
               dinv + static_cast<size_t>(G) * MH, dgrid, nex, dex, radius, dsel);
    int sel = -1;
    FDS_CUDA(cudaMemcpyAsync(&sel, dsel, sizeof(int), cudaMemcpyDeviceToHost, st));
    FDS_CUDA(cudaStreamSynchronize(st));
    if (sel < 0) throw NumericError("select_new_frequency: every grid point is excluded");
    return sel;
}

void vf_gather_channels(const cplx* src_mk, int K, int M, const int* pos_dev, int KT, cplx* dst_mk, cudaStream_t st) {
    const size_t n = static_cast<size_t>(M) * KT;
    if (n == 0) return;
    FDS_LAUNCH(vf_gather_channels_kernel, static_cast<int>((n + 255) / 256), 256, 0, st, K, M, KT, src_mk, pos_dev,
               dst_mk);
}

Cx vf_select_new_frequency(const std::vector<Cx>& ph, const std::vector<Cx>& rh, const std::vector<Cx>& pl,
                           const std::vector<Cx>& rl, int K, const std::vector<Cx>& grid,
                           const std::vector<Cx>& existing, const std::vector<int>& orf_pos, double radius,
                           const std::vector<double>* errors_in) {
    // afs.cpp:147-187
    if (orf_pos.empty()) throw ValidationError("select_new_frequency: empty ORF set");
    const std::vector<double> errors = errors_in ? *errors_in : vf_channel_errors(ph, rh, pl, rl, K, grid);
    int kmax = orf_pos[0];
    double worst = -1.0;
    for (int k : orf_pos) {
        if (k < 0 || k >= K) throw ValidationError("select_new_frequency: ORF position out of range");
        if (errors[k] > worst) { worst = errors[k]; kmax = k; }
    }
    const int G = static_cast<int>(grid.size()), MH = static_cast<int>(ph.size()), ML = static_cast<int>(pl.size());
    if (MH + ML > 512) throw ValidationError("select_new_frequency: model order too large");
    auto& cx = VfContext::get();
    // (re)build the inverse tables — cheap, keeps the function self-contained
    cplx* dgrid = dev<cplx>(cx.misc2, G + MH + ML);
    cplx* dph = dgrid + G;
    cplx* dpl = dph + MH;
    cplx* dinv = dev<cplx>(cx.tab, static_cast<size_t>(G) * (MH + ML));
    cplx* dr = dev<cplx>(cx.tab2, MH + ML);
    std::vector<double> exim(existing.size());
    for (size_t i = 0; i < existing.size(); ++i) exim[i] = existing[i].imag();
    double* dex = dev<double>(cx.misc, std::max<size_t>(exim.size(), 1) + 2);
    int* dsel = reinterpret_cast<int*>(dex + std::max<size_t>(exim.size(), 1));
    FDS_CUDA(cudaMemcpyAsync(dgrid, grid.data(), G * sizeof(cplx), cudaMemcpyHostToDevice, cx.st));
    FDS_CUDA(cudaMemcpyAsync(dph, ph.data(), MH * sizeof(cplx), cudaMemcpyHostToDevice, cx.st));
    FDS_CUDA(cudaMemcpyAsync(dpl, pl.data(), ML * sizeof(cplx), cudaMemcpyHostToDevice, cx.st));
    FDS_CUDA(cudaMemcpyAsync(dr, rh.data() + static_cast<size_t>(kmax) * MH, MH * sizeof(cplx), cudaMemcpyHostToDevice, cx.st));
    FDS_CUDA(cudaMemcpyAsync(dr + MH, rl.data() + static_cast<size_t>(kmax) * ML, ML * sizeof(cplx), cudaMemcpyHostToDevice, cx.st));
    if (!exim.empty())
        FDS_CUDA(cudaMemcpyAsync(dex, exim.data(), exim.size() * sizeof(double), cudaMemcpyHostToDevice, cx.st));
    FDS_LAUNCH(vf_inv_table_kernel, ceil_div(G * MH, 256), 256, 0, cx.st, G, MH, dgrid, dph, dinv);
    FDS_LAUNCH(vf_inv_table_kernel, ceil_div(G * ML, 256), 256, 0, cx.st, G, ML, dgrid, dpl,
               dinv + static_cast<size_t>(G) * MH);
    const int nex = static_cast<int>(exim.size());
    const size_t smem = std::max<size_t>(nex, 1) * sizeof(double);
    if (smem > 48 * 1024) {
        FDS_CUDA(cudaFuncSetAttribute(vf_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(std::min(smem, device_info().smem_optin - 16 * 1024))));
    }
    FDS_LAUNCH(vf_select_kernel, 1, 1024, smem, cx.st, G, MH, ML, dr, dr + MH, size_t(1), size_t(1), dinv,
               dinv + static_cast<size_t>(G) * MH, dgrid, nex, dex, radius, dsel);
    int sel = -1;
    FDS_CUDA(cudaMemcpyAsync(&sel, dsel, sizeof(int), cudaMemcpyDeviceToHost, cx.st));
    FDS_CUDA(cudaStreamSynchronize(cx.st));
    if (sel < 0) throw NumericError("select_new_frequency: every grid point is excluded");
    return grid[sel];
}

}  // namespace fdsb
