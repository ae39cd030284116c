// Laplace-domain 3D elastodynamic collocation BEM assembly on sm_100a (FP64).
//
// Behind FrequencySystem::evaluate (proj/include/fdsweep/systems.hpp:34-42); the
// reference has no BEM. Formulation shared with the CPU oracle
// (oracle/bem_oracle.cpp):
//   U*_ij = (A δij − B e_i e_j)/(4πμ r)
//   4π r² T*_ij = (C−B)(δij r,n + e_j n_i) − 2B(e_i n_j − 2 e_i e_j r,n) − 2D e_i e_j r,n
//                 + (λ/μ)(C−D−2B) e_i n_j
//   A=rψ, B=rχ, C=r²ψ', D=r²χ' of z = s r/c_s (16-term Taylor branch for |z|<0.3).
//
// Kernels (all deterministic — no float atomics, fixed reduction orders):
//   bem_far_kernel   one thread per (collocation point c, 64-element source
//                    chunk, frequency): 7-point Dunavant rule on every pair
//                    e != c; writes the 3x3 T̂ block of A (planar, column-major)
//                    and a per-chunk partial of b = Û t.
//   bem_near_kernel  one warp per listed near/self pair (host-built CSR, same
//                    d/h rule as the oracle) and 32 frequencies (lane = frequency):
//                    4^L x 7 subdivided points or the polar self rule
//                    (3 x 10 x 10 + exact ln-CPV), summed sequentially per lane;
//                    overwrites the A block and emits the b correction
//                    U_near·t − U_7pt·t.
//   bem_rhs_kernel   b[3c+i] = p(s)·(Σ_chunks partial + Σ_near corrections).
#include "bem.cuh"

namespace fdsb {

namespace {

constexpr double kPi = 3.14159265358979323846;

// Frequency-dependent scalars of one kernel evaluation: A, B and the three
// combinations the traction kernel needs, CB = C−B, G = C−D−2B, B4 = 4B−2D.
// Far branch in closed form with E2 = e^{−z}, E1 = k² e^{−kz}, P2 = 1/z + 1/z²,
// P1 = 1/x + 1/x² (x = kz):
//   A  = (1+P2)E2 − P1 E1            B  = (1+3P2)E2 − (1+3P1)E1
//   CB = 2(1+3P1)E1 − (z+3+6P2)E2     G  = −(1+x)E1   (the E2 terms cancel exactly)
//   B4 = (2z+12+30P2)E2 − (2x+12+30P1)E1
// which is the oracle's A..D algebra regrouped (one complex reciprocal instead
// of two, and the G cancellation done symbolically).
struct KTerms {
    cplx A, B, CB, G, B4;
};

// sincos without the Payne-Hanek slow path: Cody-Waite reduction by pi/2 in
// three FMA steps (fdlibm's 33-bit split of pi/2; with FMA each step rounds
// once, so the reduced argument stays within a few ulp of exact for |x| up to
// ~2^30, where the rounding already carried by x = Im(s) r / c_s dominates)
// and fdlibm's __kernel_sin/__kernel_cos minimax polynomials on |r| <= pi/4.
// Keeping CUDA's sincos out of the quadrature loops removes its local-memory
// reduction array and slow-path registers.
__device__ __forceinline__ void sincos_b(double x, double& s, double& c) {
    const double q = rint(x * 6.36619772367581382433e-01);
    double r = fma(-q, 1.57079632673412561417e+00, x);
    r = fma(-q, 6.07710050630396597660e-11, r);
    r = fma(-q, 2.02226624871116645580e-21, r);
    const double z = r * r;
    const double ps = fma(z, fma(z, fma(z, fma(z, fma(z, 1.58969099521155010221e-10, -2.50507602534068634195e-08),
                                                2.75573137070700676789e-06),
                                         -1.98412698298579493134e-04),
                                  8.33333333332248946124e-03),
                           -1.66666666666666324348e-01);
    const double pc = fma(z, fma(z, fma(z, fma(z, fma(z, -1.13596475577881948265e-11, 2.08757232129817482790e-09),
                                                -2.75573143513906633035e-07),
                                         2.48015872894767294178e-05),
                                  -1.38888888888741095749e-03),
                           4.16666666666666019037e-02);
    const double sr = fma(r * z, ps, r);
    const double hz = 0.5 * z, w = 1.0 - hz;
    const double cr = w + (((1.0 - w) - hz) + z * z * pc);
    const long long iq = static_cast<long long>(q);
    double ss = (iq & 1) ? cr : sr;
    double cc = (iq & 1) ? sr : cr;
    if (iq & 2) ss = -ss;
    if ((iq + 1) & 2) cc = -cc;
    s = ss;
    c = cc;
}

// e^{-(a + i b)}
__device__ __forceinline__ cplx cexp_neg(double a, double b) {
    double sn, cs;
    sincos_b(b, sn, cs);
    const double e = exp(-a);
    return mk(e * cs, -e * sn);
}

// Per-thread constants of one frequency s: z = s r / c_s = (za + i zb) r and
// 1/z = w / r, so the quadrature loops need no complex division.
struct FreqK {
    double za, zb;   // s / c_s
    cplx w, w2;      // c_s / s and its square
    cplx wk, wk2;    // (c_s / s) / k and its square (1/x1 = wk / r)
    double r2ser;    // r^2 below which |z|^2 < kSeriesR2 (Taylor branch)
};

__device__ __forceinline__ FreqK freq_consts(const BemParams& P, cplx s) {
    FreqK F;
    F.za = s.re * P.inv_cs;
    F.zb = s.im * P.inv_cs;
    F.w = crecip(mk(F.za, F.zb));
    F.w2 = F.w * F.w;
    F.wk = F.w * P.inv_k;
    F.wk2 = F.wk * F.wk;
    const double zz = F.za * F.za + F.zb * F.zb;
    F.r2ser = BemParams::kSeriesR2 / zz;
    return F;
}

// Taylor branch (|z| < 0.3): A, B, C, D as power series in z.
__device__ __forceinline__ KTerms kterms_series(const BemParams& P, cplx z) {
    KTerms o;
    cplx A = mk(0.0, 0.0), B = A, C = A, D = A;
#pragma unroll
    for (int m = BemParams::kTerms - 1; m >= 0; --m) {
        A = A * z + P.ta[m];
        B = B * z + P.tb[m];
        C = C * z + P.tc[m];
        D = D * z + P.td[m];
    }
    o.A = A;
    o.B = B;
    o.CB = C - B;
    o.G = C - D - 2.0 * B;
    o.B4 = 4.0 * B - 2.0 * D;
    return o;
}

// Closed form given P2 = 1/z + 1/z^2, P1 = 1/x + 1/x^2, E2 = e^{-z}, E1 = k^2 e^{-x}.
__device__ __forceinline__ KTerms kterms_closed(cplx z, cplx x1, cplx P2, cplx P1, cplx E2, cplx E1) {
    KTerms o;
    const cplx q1E1 = (3.0 * P1 + 1.0) * E1;
    o.A = (P2 + 1.0) * E2 - P1 * E1;
    o.B = (3.0 * P2 + 1.0) * E2 - q1E1;
    o.CB = 2.0 * q1E1 - (z + 6.0 * P2 + 3.0) * E2;
    o.G = -((x1 + 1.0) * E1);
    o.B4 = (2.0 * z + 30.0 * P2 + 12.0) * E2 - (2.0 * x1 + 30.0 * P1 + 12.0) * E1;
    return o;
}

__device__ __forceinline__ KTerms kterms(const BemParams& P, cplx z) {
    if (abs2(z) < BemParams::kSeriesR2) return kterms_series(P, z);
    const double k = P.k, ik = P.inv_k;
    const cplx x1 = z * k;
    const double d = 1.0 / abs2(z);
    const cplx iz = mk(z.re * d, -z.im * d);
    const cplx iz2 = iz * iz;
    const cplx E2 = cexp_neg(z.re, z.im);
    const cplx E1 = cexp_neg(x1.re, x1.im) * (k * k);
    return kterms_closed(z, x1, iz + iz2, iz * ik + iz2 * (ik * ik), E2, E1);
}

// Same terms at distance r (1/r = ir, 1/r^2 = ir2) from the per-thread
// frequency constants: no complex division per point.
__device__ __forceinline__ KTerms kterms_r(const BemParams& P, const FreqK& F, double r, double ir, double ir2) {
    const cplx z = mk(F.za * r, F.zb * r);
    if (r * r < F.r2ser) return kterms_series(P, z);
    const double k = P.k;
    const cplx x1 = z * k;
    const cplx P2 = F.w * ir + F.w2 * ir2;
    const cplx P1 = F.wk * ir + F.wk2 * ir2;
    const cplx E2 = cexp_neg(z.re, z.im);
    const cplx E1 = cexp_neg(x1.re, x1.im) * (k * k);
    return kterms_closed(z, x1, P2, P1, E2, E1);
}

// Quadrature-point sums over one flat source element (n constant):
//   T_ij = δij S0 + n_i Sj + Ei n_j + Bij,   (U·t)_i = SA t_i − SB_i
// with S0 = Σ cb r,n, Sj = Σ cb e_j, Ei = Σ e4 e_i, Bij = Σ b4 r,n e_i e_j,
// SA = Σ A fu, SB_i = Σ B fu (e·t) e_i — 17 complex sums per point instead of
// the 12 complex 3-term updates of the assembled blocks.
struct KAcc {
    cplx s0, sj[3], ei[3], bij[6], sa, sb[3];
    __device__ __forceinline__ void zero() {
        s0 = sa = mk(0.0, 0.0);
#pragma unroll
        for (int i = 0; i < 3; ++i) sj[i] = ei[i] = sb[i] = mk(0.0, 0.0);
#pragma unroll
        for (int i = 0; i < 6; ++i) bij[i] = mk(0.0, 0.0);
    }
    // displacement part: A, B with weight fu, unit vector e, e·t
    __device__ __forceinline__ void add_u(const KTerms& k, const double e[3], double fu, double et) {
        sa = sa + k.A * fu;
        const cplx bf = k.B * (fu * et);
#pragma unroll
        for (int i = 0; i < 3; ++i) sb[i] = sb[i] + bf * e[i];
    }
    __device__ __forceinline__ void add(const BemParams& P, const KTerms& k, const double e[3], double rn,
                                        double fu, double ft, double et) {
        const cplx cb = k.CB * ft;
        const cplx e4 = (P.lam_over_mu * k.G - 2.0 * k.B) * ft;
        const cplx b4 = k.B4 * (ft * rn);
        s0 = s0 + cb * rn;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            sj[i] = sj[i] + cb * e[i];
            ei[i] = ei[i] + e4 * e[i];
        }
        bij[0] = bij[0] + b4 * (e[0] * e[0]);
        bij[1] = bij[1] + b4 * (e[0] * e[1]);
        bij[2] = bij[2] + b4 * (e[0] * e[2]);
        bij[3] = bij[3] + b4 * (e[1] * e[1]);
        bij[4] = bij[4] + b4 * (e[1] * e[2]);
        bij[5] = bij[5] + b4 * (e[2] * e[2]);
        add_u(k, e, fu, et);
    }
    // T (row-major i*3+j) and U·t of the element
    __device__ __forceinline__ void finish(const double n[3], const double t[3], cplx T[9], cplx Ut[3]) const {
        constexpr int bidx[3][3] = {{0, 1, 2}, {1, 3, 4}, {2, 4, 5}};
#pragma unroll
        for (int i = 0; i < 3; ++i) {
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                cplx v = sj[j] * n[i] + ei[i] * n[j] + bij[bidx[i][j]];
                if (i == j) v = v + s0;
                T[3 * i + j] = v;
            }
            Ut[i] = sa * t[i] - sb[i];
        }
    }
};

// One regular quadrature point y (relative position r = y − x) of weight w.
__device__ __forceinline__ void kpoint(const BemParams& P, KAcc& acc, double rx, double ry, double rz,
                                       const double n[3], const double t[3], const FreqK& F, double w) {
    const double r2 = rx * rx + ry * ry + rz * rz;
    const double r = sqrt(r2);
    const double ir = 1.0 / r;
    const double ir2 = ir * ir;
    const double e[3] = {rx * ir, ry * ir, rz * ir};
    const double rn = e[0] * n[0] + e[1] * n[1] + e[2] * n[2];
    const KTerms k = kterms_r(P, F, r, ir, ir2);
    const double fu = w * ir * P.inv_4pi_mu;
    const double ft = w * ir2 * (1.0 / (4.0 * kPi));
    const double et = e[0] * t[0] + e[1] * t[1] + e[2] * t[2];
    acc.add(P, k, e, rn, fu, ft, et);
}

// Displacement-only point (the far 7-point U·t a near pair must cancel).
__device__ __forceinline__ void kpoint_u(const BemParams& P, KAcc& acc, double rx, double ry, double rz,
                                         const double t[3], const FreqK& F, double w) {
    const double r = sqrt(rx * rx + ry * ry + rz * rz);
    const double ir = 1.0 / r;
    const double e[3] = {rx * ir, ry * ir, rz * ir};
    const KTerms k = kterms_r(P, F, r, ir, ir * ir);
    acc.add_u(k, e, w * ir * P.inv_4pi_mu, e[0] * t[0] + e[1] * t[1] + e[2] * t[2]);
}

// Self-element polar point: the static CPV part E10/E20 is integrated exactly
// elsewhere, so only the dynamic remainder (CB − E10, λ/μ G − 2B − E20) is summed.
__device__ __forceinline__ void kpoint_self(const BemParams& P, KAcc& acc, const KTerms& k, const double ev[3],
                                            double fu, double ft, double et) {
    const cplx dE1 = (k.CB - mk(P.E10, 0.0)) * ft;
    const cplx dE2 = (P.lam_over_mu * k.G - 2.0 * k.B - mk(P.E20, 0.0)) * ft;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        acc.sj[i] = acc.sj[i] + dE1 * ev[i];
        acc.ei[i] = acc.ei[i] + dE2 * ev[i];
    }
    acc.add_u(k, ev, fu, et);
}

// Exact ln-CPV static part along one polar ray: T += (E10 e_j n_i + E20 e_i n_j) lnR.
__device__ __forceinline__ void kpoint_cpv(const BemParams& P, KAcc& acc, const double ev[3], double lnR) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        acc.sj[i].re += P.E10 * lnR * ev[i];
        acc.ei[i].re += P.E20 * lnR * ev[i];
    }
}

}  // namespace

// ------------------------------------------------------------------ far field
__global__ void __launch_bounds__(kFarThreads, 2)
bem_far_kernel(BemParams P, const double* __restrict__ geo, const double* __restrict__ trac,
               int ne, const cplx* __restrict__ svec, double* __restrict__ A, size_t mstride,
               size_t plane, int ld, cplx* __restrict__ partial, size_t pstride) {
    __shared__ double sg[kFarChunk][16];
    __shared__ double st[kFarChunk][3];
    const int c = blockIdx.x * kFarThreads + threadIdx.x;
    const int chunk = blockIdx.y;
    const int b = blockIdx.z;
    const int e0 = chunk * kFarChunk;
    const int ecount = min(kFarChunk, ne - e0);
    for (int i = threadIdx.x; i < ecount * 16; i += kFarThreads) sg[i / 16][i % 16] = geo[(size_t)e0 * 16 + i];
    for (int i = threadIdx.x; i < ecount * 3; i += kFarThreads) st[i / 3][i % 3] = trac[(size_t)e0 * 3 + i];
    __syncthreads();
    if (c >= ne) return;
    const cplx s = svec[b];
    const FreqK F = freq_consts(P, s);
    const double x0 = geo[(size_t)c * 16 + 9], x1 = geo[(size_t)c * 16 + 10], x2 = geo[(size_t)c * 16 + 11];
    double* Are = A + (size_t)b * mstride;
    double* Aim = Are + plane;
    cplx Ut[3] = {mk(0, 0), mk(0, 0), mk(0, 0)};
    for (int el = 0; el < ecount; ++el) {
        const int e = e0 + el;
        if (e == c) continue;
        const double* g = sg[el];
        const double n[3] = {g[12], g[13], g[14]};
        const double t[3] = {st[el][0], st[el][1], st[el][2]};
        KAcc acc;
        acc.zero();
        // two quadrature points in flight (independent transcendental chains);
        // at 2 CTAs/SM the kernel keeps 255 registers (measured: cfg2 far
        // stage 35.1 -> 32.8 ms; full unrolling or 3 CTAs/SM spill heavily)
#pragma unroll 2
        for (int q = 0; q < 7; ++q) {
            const double l0 = P.r7l[q][0], l1 = P.r7l[q][1], l2 = P.r7l[q][2];
            const double yx = l0 * g[0] + l1 * g[3] + l2 * g[6];
            const double yy = l0 * g[1] + l1 * g[4] + l2 * g[7];
            const double yz = l0 * g[2] + l1 * g[5] + l2 * g[8];
            kpoint(P, acc, yx - x0, yy - x1, yz - x2, n, t, F, P.r7w[q] * g[15]);
        }
        cplx T[9], Ue[3];
        acc.finish(n, t, T, Ue);
#pragma unroll
        for (int i = 0; i < 3; ++i) Ut[i] = Ut[i] + Ue[i];
        // A[(3e+j)*ld + 3c+i]
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const size_t col = (size_t)(3 * e + j) * ld + 3 * c;
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                Are[col + i] = T[3 * i + j].re;
                Aim[col + i] = T[3 * i + j].im;
            }
        }
    }
    cplx* pp = partial + (size_t)b * pstride + (size_t)chunk * 3 * ne + 3 * c;
    pp[0] = Ut[0];
    pp[1] = Ut[1];
    pp[2] = Ut[2];
}

// ------------------------------------------------------------------ near / self
// One warp per listed near/self pair and 32 frequencies: lane b integrates the
// whole pair for frequency b (the quadrature geometry is warp-uniform), so
// there is no cross-lane reduction and all 32 lanes do useful work.
__global__ void __launch_bounds__(128, 3)
bem_near_kernel(BemParams P, const double* __restrict__ geo, const double* __restrict__ trac,
                int ne, const int* __restrict__ pairs, const int* __restrict__ order, int npairs,
                const cplx* __restrict__ svec, int B, double* __restrict__ A, size_t mstride, size_t plane, int ld,
                cplx* __restrict__ corr, size_t cstride) {
    const int slot = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.y * 32 + lane;
    if (slot >= npairs) return;
    const int pair = order[slot];
    const bool active = b < B;
    const int c = pairs[3 * pair], e = pairs[3 * pair + 1], level = pairs[3 * pair + 2];
    const cplx s = svec[active ? b : 0];
    const FreqK F = freq_consts(P, s);
    const double* g = geo + (size_t)e * 16;
    const double x0 = geo[(size_t)c * 16 + 9], x1 = geo[(size_t)c * 16 + 10], x2 = geo[(size_t)c * 16 + 11];
    const double n[3] = {g[12], g[13], g[14]};
    const double t[3] = {trac[3 * e], trac[3 * e + 1], trac[3 * e + 2]};
    cplx T[9], Ut[3];
    KAcc acc;
    acc.zero();

    if (level < 0) {
        // Self element: polar quadrature about the centroid over the 3 edge
        // sub-triangles; static antisymmetric T part as the exact CPV.
        const int NG = BemParams::kSelfGauss;
        for (int edge = 0; edge < 3; ++edge) {
            const int ia = edge, ib = (edge + 1) % 3;
            const double Px = g[3 * ia], Py = g[3 * ia + 1], Pz = g[3 * ia + 2];
            const double Qx = g[3 * ib] - Px, Qy = g[3 * ib + 1] - Py, Qz = g[3 * ib + 2] - Pz;
            const double L = sqrt(Qx * Qx + Qy * Qy + Qz * Qz);
            const double cx = g[9], cy = g[10], cz = g[11];
            const double wx = Px - cx, wy = Py - cy, wz = Pz - cz;
            const double crx = wy * Qz - wz * Qy, cry = wz * Qx - wx * Qz, crz = wx * Qy - wy * Qx;
            const double hperp = sqrt(crx * crx + cry * cry + crz * crz) / L;
            for (int a = 0; a < NG; ++a) {
                const double ta = P.glx[a];
                const double dx = wx + ta * Qx, dy = wy + ta * Qy, dz = wz + ta * Qz;
                const double R = sqrt(dx * dx + dy * dy + dz * dz);
                const double ev[3] = {dx / R, dy / R, dz / R};
                const double jt = hperp * L * P.glw[a];
                const double lnR = log(R) / (R * R) * jt * (1.0 / (4.0 * kPi));
                kpoint_cpv(P, acc, ev, lnR);
                const double et = ev[0] * t[0] + ev[1] * t[1] + ev[2] * t[2];
#pragma unroll 1
                for (int bq = 0; bq < NG; ++bq) {
                    const double u = P.glx[bq];
                    const double rho = R * u;
                    const KTerms k = kterms(P, s * (rho * P.inv_cs));
                    const double w = jt * P.glw[bq];
                    kpoint_self(P, acc, k, ev, w * u / rho * P.inv_4pi_mu, w * u / (rho * rho) * (1.0 / (4.0 * kPi)),
                                et);
                }
            }
        }
        acc.finish(n, t, T, Ut);
    } else {
        // Near element: 4^level sub-triangles (recursive midpoint split, children
        // (p0,m01,m20), (m01,p1,m12), (m20,m12,p2), (m01,m12,m20)), 7 points each.
        const int nsub = 1 << (2 * level);
        for (int sub = 0; sub < nsub; ++sub) {
            double p[3][3];
#pragma unroll
            for (int v = 0; v < 3; ++v)
#pragma unroll
                for (int d = 0; d < 3; ++d) p[v][d] = g[3 * v + d];
            for (int lv = level - 1; lv >= 0; --lv) {
                const int child = (sub >> (2 * lv)) & 3;
                double m01[3], m12[3], m20[3];
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    m01[d] = 0.5 * (p[0][d] + p[1][d]);
                    m12[d] = 0.5 * (p[1][d] + p[2][d]);
                    m20[d] = 0.5 * (p[2][d] + p[0][d]);
                }
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    if (child == 0) { p[1][d] = m01[d]; p[2][d] = m20[d]; }
                    else if (child == 1) { p[0][d] = m01[d]; p[2][d] = m12[d]; }
                    else if (child == 2) { p[0][d] = m20[d]; p[1][d] = m12[d]; }
                    else { p[0][d] = m01[d]; p[1][d] = m12[d]; p[2][d] = m20[d]; }
                }
            }
            const double ux = p[1][0] - p[0][0], uy = p[1][1] - p[0][1], uz = p[1][2] - p[0][2];
            const double vx = p[2][0] - p[0][0], vy = p[2][1] - p[0][1], vz = p[2][2] - p[0][2];
            const double cx = uy * vz - uz * vy, cy = uz * vx - ux * vz, cz = ux * vy - uy * vx;
            const double area = 0.5 * sqrt(cx * cx + cy * cy + cz * cz);
#pragma unroll 1
            for (int gq = 0; gq < 7; ++gq) {
                const double l0 = P.r7l[gq][0], l1 = P.r7l[gq][1], l2 = P.r7l[gq][2];
                const double yx = l0 * p[0][0] + l1 * p[1][0] + l2 * p[2][0];
                const double yy = l0 * p[0][1] + l1 * p[1][1] + l2 * p[2][1];
                const double yz = l0 * p[0][2] + l1 * p[1][2] + l2 * p[2][2];
                kpoint(P, acc, yx - x0, yy - x1, yz - x2, n, t, F, P.r7w[gq] * area);
            }
        }
        // subtract the far kernel's 7-point U·t for this pair (it is in the partials)
        KAcc accf;
        accf.zero();
#pragma unroll 1
        for (int gq = 0; gq < 7; ++gq) {
            const double l0 = P.r7l[gq][0], l1 = P.r7l[gq][1], l2 = P.r7l[gq][2];
            const double yx = l0 * g[0] + l1 * g[3] + l2 * g[6];
            const double yy = l0 * g[1] + l1 * g[4] + l2 * g[7];
            const double yz = l0 * g[2] + l1 * g[5] + l2 * g[8];
            kpoint_u(P, accf, yx - x0, yy - x1, yz - x2, t, F, P.r7w[gq] * g[15]);
        }
        acc.finish(n, t, T, Ut);
#pragma unroll
        for (int i = 0; i < 3; ++i) Ut[i] = Ut[i] - (accf.sa * t[i] - accf.sb[i]);
    }
    if (!active) return;
    double* Are = A + (size_t)b * mstride;
    double* Aim = Are + plane;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        const size_t col = (size_t)(3 * e + j) * ld + 3 * c;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            cplx v = T[3 * i + j];
            if (level < 0 && i == j) v.re += 0.5;
            Are[col + i] = v.re;
            Aim[col + i] = v.im;
        }
    }
    cplx* cp = corr + (size_t)b * cstride + (size_t)pair * 3;
    cp[0] = Ut[0];
    cp[1] = Ut[1];
    cp[2] = Ut[2];
}

// Few frequencies (B < 8): one warp per (pair, frequency), lanes split the
// quadrature points and reduce with shuffles in a fixed tree.
namespace {

__device__ __forceinline__ void warp_sum(cplx* v, int count) {
    for (int i = 0; i < count; ++i) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            v[i].re += __shfl_xor_sync(0xffffffffu, v[i].re, off);
            v[i].im += __shfl_xor_sync(0xffffffffu, v[i].im, off);
        }
    }
}

}  // namespace

__global__ void __launch_bounds__(128)
bem_near_pts_kernel(BemParams P, const double* __restrict__ geo, const double* __restrict__ trac,
                int ne, const int* __restrict__ pairs, int npairs, const cplx* __restrict__ svec,
                double* __restrict__ A, size_t mstride, size_t plane, int ld,
                cplx* __restrict__ corr, size_t cstride) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.y;
    if (warp >= npairs) return;
    const int c = pairs[3 * warp], e = pairs[3 * warp + 1], level = pairs[3 * warp + 2];
    const cplx s = svec[b];
    const FreqK F = freq_consts(P, s);
    const double* g = geo + (size_t)e * 16;
    const double x0 = geo[(size_t)c * 16 + 9], x1 = geo[(size_t)c * 16 + 10], x2 = geo[(size_t)c * 16 + 11];
    const double n[3] = {g[12], g[13], g[14]};
    const double t[3] = {trac[3 * e], trac[3 * e + 1], trac[3 * e + 2]};
    cplx T[9], Ut[3];
    KAcc acc;
    acc.zero();

    if (level < 0) {
        // Self element: polar quadrature about the centroid over the 3 edge
        // sub-triangles; static antisymmetric T part as the exact CPV.
        const int NG = BemParams::kSelfGauss;
        const int npts = 3 * NG * NG;
        for (int q = lane; q < npts; q += 32) {
            const int edge = q / (NG * NG), a = (q / NG) % NG, bq = q % NG;
            const int ia = edge, ib = (edge + 1) % 3;
            const double Px = g[3 * ia], Py = g[3 * ia + 1], Pz = g[3 * ia + 2];
            const double Qx = g[3 * ib] - Px, Qy = g[3 * ib + 1] - Py, Qz = g[3 * ib + 2] - Pz;
            const double L = sqrt(Qx * Qx + Qy * Qy + Qz * Qz);
            const double cx = g[9], cy = g[10], cz = g[11];
            const double wx = Px - cx, wy = Py - cy, wz = Pz - cz;
            const double crx = wy * Qz - wz * Qy, cry = wz * Qx - wx * Qz, crz = wx * Qy - wy * Qx;
            const double hperp = sqrt(crx * crx + cry * cry + crz * crz) / L;
            const double ta = P.glx[a];
            const double dx = wx + ta * Qx, dy = wy + ta * Qy, dz = wz + ta * Qz;
            const double R = sqrt(dx * dx + dy * dy + dz * dz);
            const double ev[3] = {dx / R, dy / R, dz / R};
            const double jt = hperp * L * P.glw[a];
            if (bq == 0) kpoint_cpv(P, acc, ev, log(R) / (R * R) * jt * (1.0 / (4.0 * kPi)));
            const double u = P.glx[bq];
            const double rho = R * u;
            const KTerms k = kterms(P, s * (rho * P.inv_cs));
            const double w = jt * P.glw[bq];
            const double et = ev[0] * t[0] + ev[1] * t[1] + ev[2] * t[2];
            kpoint_self(P, acc, k, ev, w * u / rho * P.inv_4pi_mu, w * u / (rho * rho) * (1.0 / (4.0 * kPi)), et);
        }
        acc.finish(n, t, T, Ut);
    } else {
        // Near element: 4^level sub-triangles (recursive midpoint split, children
        // (p0,m01,m20), (m01,p1,m12), (m20,m12,p2), (m01,m12,m20)), 7 points each.
        const int nsub = 1 << (2 * level);
        const int npts = nsub * 7;
        for (int q = lane; q < npts; q += 32) {
            int sub = q / 7;
            const int gq = q % 7;
            double p[3][3];
#pragma unroll
            for (int v = 0; v < 3; ++v)
#pragma unroll
                for (int d = 0; d < 3; ++d) p[v][d] = g[3 * v + d];
            for (int lv = level - 1; lv >= 0; --lv) {
                const int child = (sub >> (2 * lv)) & 3;
                double m01[3], m12[3], m20[3];
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    m01[d] = 0.5 * (p[0][d] + p[1][d]);
                    m12[d] = 0.5 * (p[1][d] + p[2][d]);
                    m20[d] = 0.5 * (p[2][d] + p[0][d]);
                }
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    if (child == 0) { p[1][d] = m01[d]; p[2][d] = m20[d]; }
                    else if (child == 1) { p[0][d] = m01[d]; p[2][d] = m12[d]; }
                    else if (child == 2) { p[0][d] = m20[d]; p[1][d] = m12[d]; }
                    else { p[0][d] = m01[d]; p[1][d] = m12[d]; p[2][d] = m20[d]; }
                }
            }
            const double ux = p[1][0] - p[0][0], uy = p[1][1] - p[0][1], uz = p[1][2] - p[0][2];
            const double vx = p[2][0] - p[0][0], vy = p[2][1] - p[0][1], vz = p[2][2] - p[0][2];
            const double cx = uy * vz - uz * vy, cy = uz * vx - ux * vz, cz = ux * vy - uy * vx;
            const double area = 0.5 * sqrt(cx * cx + cy * cy + cz * cz);
            const double l0 = P.r7l[gq][0], l1 = P.r7l[gq][1], l2 = P.r7l[gq][2];
            const double yx = l0 * p[0][0] + l1 * p[1][0] + l2 * p[2][0];
            const double yy = l0 * p[0][1] + l1 * p[1][1] + l2 * p[2][1];
            const double yz = l0 * p[0][2] + l1 * p[1][2] + l2 * p[2][2];
            kpoint(P, acc, yx - x0, yy - x1, yz - x2, n, t, F, P.r7w[gq] * area);
        }
        acc.finish(n, t, T, Ut);
        // subtract the far kernel's 7-point U·t for this pair (it is in the partials)
        if (lane < 7) {
            KAcc accf;
            accf.zero();
            const double l0 = P.r7l[lane][0], l1 = P.r7l[lane][1], l2 = P.r7l[lane][2];
            const double yx = l0 * g[0] + l1 * g[3] + l2 * g[6];
            const double yy = l0 * g[1] + l1 * g[4] + l2 * g[7];
            const double yz = l0 * g[2] + l1 * g[5] + l2 * g[8];
            kpoint_u(P, accf, yx - x0, yy - x1, yz - x2, t, F, P.r7w[lane] * g[15]);
#pragma unroll
            for (int i = 0; i < 3; ++i) Ut[i] = Ut[i] - (accf.sa * t[i] - accf.sb[i]);
        }
    }
    warp_sum(T, 9);
    warp_sum(Ut, 3);
    if (lane == 0) {
        double* Are = A + (size_t)b * mstride;
        double* Aim = Are + plane;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const size_t col = (size_t)(3 * e + j) * ld + 3 * c;
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                cplx v = T[3 * i + j];
                if (level < 0 && i == j) v.re += 0.5;
                Are[col + i] = v.re;
                Aim[col + i] = v.im;
            }
        }
        cplx* cp = corr + (size_t)b * cstride + (size_t)warp * 3;
        cp[0] = Ut[0];
        cp[1] = Ut[1];
        cp[2] = Ut[2];
    }
}

// ------------------------------------------------------------------ rhs
__global__ void bem_rhs_kernel(int ne, int nchunks, const cplx* __restrict__ partial, size_t pstride,
                               const int* __restrict__ near_ptr, const cplx* __restrict__ corr,
                               size_t cstride, const cplx* __restrict__ svec, cplx* __restrict__ rhs,
                               size_t rstride) {
    const int dof = blockIdx.x * blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    if (dof >= 3 * ne) return;
    const int c = dof / 3, i = dof % 3;
    const cplx* pp = partial + (size_t)b * pstride;
    cplx acc = mk(0.0, 0.0);
    for (int ch = 0; ch < nchunks; ++ch) acc = acc + pp[(size_t)ch * 3 * ne + dof];
    const cplx* cp = corr + (size_t)b * cstride;
    for (int q = near_ptr[c]; q < near_ptr[c + 1]; ++q) acc = acc + cp[(size_t)q * 3 + i];
    rhs[(size_t)b * rstride + dof] = acc * crecip(svec[b]);  // Heaviside p(s) = 1/s
}

void bem_assemble(const BemDevice& d, const cplx* svec_dev, int B, double* A, size_t mstride,
                  size_t plane, int ld, cplx* rhs, size_t rstride, cudaStream_t st) {
    const int ne = d.ne;
    const int nchunks = ceil_div(ne, kFarChunk);
    dim3 gf(ceil_div(ne, kFarThreads), nchunks, B);
    cudaEvent_t pe;
    profiler().begin(st, kProfAsmFar, 0.0, pe);
    FDS_LAUNCH(bem_far_kernel, gf, kFarThreads, 0, st, d.params, d.geo, d.trac, ne, svec_dev, A,
               mstride, plane, ld, d.partial, d.pstride);
    // work unit: kernel evaluations (7 points per far pair and frequency)
    profiler().end(st, pe, kProfAsmFar, 7.0 * ne * (ne - 1.0) * B);
    profiler().begin(st, kProfAsmNear, 0.0, pe);
    if (B >= 8) {
        dim3 gn(ceil_div(d.npairs, 4), ceil_div(B, 32));
        FDS_LAUNCH(bem_near_kernel, gn, 128, 0, st, d.params, d.geo, d.trac, ne, d.pairs, d.order, d.npairs,
                   svec_dev, B, A, mstride, plane, ld, d.corr, d.cstride);
    } else {
        dim3 gn(ceil_div(d.npairs * 32, 128), B);
        FDS_LAUNCH(bem_near_pts_kernel, gn, 128, 0, st, d.params, d.geo, d.trac, ne, d.pairs, d.npairs,
                   svec_dev, A, mstride, plane, ld, d.corr, d.cstride);
    }
    profiler().end(st, pe, kProfAsmNear, static_cast<double>(d.npairs) * B);
    dim3 gr(ceil_div(3 * ne, 128), B);
    FDS_LAUNCH(bem_rhs_kernel, gr, 128, 0, st, ne, nchunks, d.partial, d.pstride, d.near_ptr, d.corr,
               d.cstride, svec_dev, rhs, rstride);
}

}  // namespace fdsb
