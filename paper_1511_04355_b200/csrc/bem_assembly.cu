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

__device__ __forceinline__ void abcd(const BemParams& P, cplx z, cplx& A, cplx& B, cplx& C, cplx& D) {
    if (abs2(z) < BemParams::kSeriesR2) {
        A = B = C = D = mk(0.0, 0.0);
#pragma unroll
        for (int m = BemParams::kTerms - 1; m >= 0; --m) {
            A = A * z + P.ta[m];
            B = B * z + P.tb[m];
            C = C * z + P.tc[m];
            D = D * z + P.td[m];
        }
        return;
    }
    const cplx x1 = z * P.k;
    const cplx e2 = cexpd(-z), e1 = cexpd(-x1);
    const cplx iz = crecip(z), iz2 = iz * iz;
    const cplx ix = crecip(x1), ix2 = ix * ix;
    const double k2 = P.k * P.k;
    A = (mk(1.0, 0.0) + iz + iz2) * e2 - k2 * ((ix + ix2) * e1);
    const cplx q2 = mk(1.0, 0.0) + 3.0 * iz + 3.0 * iz2;
    const cplx q1 = mk(1.0, 0.0) + 3.0 * ix + 3.0 * ix2;
    B = q2 * e2 - k2 * (q1 * e1);
    C = -((z + 2.0 + 3.0 * iz + 3.0 * iz2) * e2) + k2 * (q1 * e1);
    D = -((z + 4.0 + 9.0 * iz + 9.0 * iz2) * e2) + k2 * ((x1 + 4.0 + 9.0 * ix + 9.0 * ix2) * e1);
}

// Accumulates w*T (9 complex, row-major i*3+j) and w*(U·t) (3 complex).
__device__ __forceinline__ void accumulate_ut(const BemParams& P, double rx, double ry, double rz,
                                              const double n[3], const double t[3], cplx s,
                                              double w, cplx T[9], cplx Ut[3]) {
    const double r2 = rx * rx + ry * ry + rz * rz;
    const double r = sqrt(r2);
    const double ir = 1.0 / r;
    const double e[3] = {rx * ir, ry * ir, rz * ir};
    const double rn = e[0] * n[0] + e[1] * n[1] + e[2] * n[2];
    cplx A, B, C, D;
    abcd(P, s * (r * P.inv_cs), A, B, C, D);
    const double fu = w * ir * P.inv_4pi_mu;
    const double ft = w * ir * ir * (1.0 / (4.0 * kPi));
    const cplx cb = (C - B) * ft;
    const cplx e4 = (P.lam_over_mu * (C - D - 2.0 * B) - 2.0 * B) * ft;  // coefficient of e_i n_j
    const cplx b4 = (4.0 * B - 2.0 * D) * ft;                              // of e_i e_j r,n
    // U·t = (A t − B e (e·t)) fu
    const double et = e[0] * t[0] + e[1] * t[1] + e[2] * t[2];
#pragma unroll
    for (int i = 0; i < 3; ++i) Ut[i] = Ut[i] + (A * t[i] - B * (e[i] * et)) * fu;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const double dij = (i == j) ? rn : 0.0;
            T[3 * i + j] = T[3 * i + j] + cb * (dij + e[j] * n[i]) + e4 * (e[i] * n[j]) +
                           b4 * (e[i] * e[j] * rn);
        }
    }
}

}  // namespace

// ------------------------------------------------------------------ far field
__global__ void __launch_bounds__(kFarThreads)
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
        cplx T[9];
#pragma unroll
        for (int i = 0; i < 9; ++i) T[i] = mk(0.0, 0.0);
#pragma unroll
        for (int q = 0; q < 7; ++q) {
            const double l0 = P.r7l[q][0], l1 = P.r7l[q][1], l2 = P.r7l[q][2];
            const double yx = l0 * g[0] + l1 * g[3] + l2 * g[6];
            const double yy = l0 * g[1] + l1 * g[4] + l2 * g[7];
            const double yz = l0 * g[2] + l1 * g[5] + l2 * g[8];
            accumulate_ut(P, yx - x0, yy - x1, yz - x2, n, t, s, P.r7w[q] * g[15], T, Ut);
        }
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
__global__ void __launch_bounds__(128)
bem_near_kernel(BemParams P, const double* __restrict__ geo, const double* __restrict__ trac,
                int ne, const int* __restrict__ pairs, int npairs, const cplx* __restrict__ svec, int B,
                double* __restrict__ A, size_t mstride, size_t plane, int ld,
                cplx* __restrict__ corr, size_t cstride) {
    const int pair = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    const int b = blockIdx.y * 32 + lane;
    if (pair >= npairs) return;
    const bool active = b < B;
    const int c = pairs[3 * pair], e = pairs[3 * pair + 1], level = pairs[3 * pair + 2];
    const cplx s = svec[active ? b : 0];
    const double* g = geo + (size_t)e * 16;
    const double x0 = geo[(size_t)c * 16 + 9], x1 = geo[(size_t)c * 16 + 10], x2 = geo[(size_t)c * 16 + 11];
    const double n[3] = {g[12], g[13], g[14]};
    const double t[3] = {trac[3 * e], trac[3 * e + 1], trac[3 * e + 2]};
    cplx T[9], Ut[3];
#pragma unroll
    for (int i = 0; i < 9; ++i) T[i] = mk(0.0, 0.0);
    Ut[0] = Ut[1] = Ut[2] = mk(0.0, 0.0);

    if (level < 0) {
        // Self element: polar quadrature about the centroid over the 3 edge
        // sub-triangles; static antisymmetric T part as the exact CPV.
        const int NG = BemParams::kSelfGauss;
        const cplx E10 = mk(P.E10, 0.0), E20 = mk(P.E20, 0.0);
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
#pragma unroll
                for (int i = 0; i < 3; ++i)
#pragma unroll
                    for (int j = 0; j < 3; ++j)
                        T[3 * i + j] = T[3 * i + j] + (E10 * (ev[j] * n[i]) + E20 * (ev[i] * n[j])) * lnR;
                const double et = ev[0] * t[0] + ev[1] * t[1] + ev[2] * t[2];
                for (int bq = 0; bq < NG; ++bq) {
                    const double u = P.glx[bq];
                    const double rho = R * u;
                    cplx Aa, Bb, Cc, Dd;
                    abcd(P, s * (rho * P.inv_cs), Aa, Bb, Cc, Dd);
                    const double w = jt * P.glw[bq];
                    const double fu = w * u / rho * P.inv_4pi_mu;
                    const double ft = w * u / (rho * rho) * (1.0 / (4.0 * kPi));
                    const cplx dE1 = (Cc - Bb) - E10;
                    const cplx dE2 = P.lam_over_mu * (Cc - Dd - 2.0 * Bb) - 2.0 * Bb - E20;
#pragma unroll
                    for (int i = 0; i < 3; ++i) Ut[i] = Ut[i] + (Aa * t[i] - Bb * (ev[i] * et)) * fu;
#pragma unroll
                    for (int i = 0; i < 3; ++i)
#pragma unroll
                        for (int j = 0; j < 3; ++j)
                            T[3 * i + j] = T[3 * i + j] + (dE1 * (ev[j] * n[i]) + dE2 * (ev[i] * n[j])) * ft;
                }
            }
        }
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
            for (int gq = 0; gq < 7; ++gq) {
                const double l0 = P.r7l[gq][0], l1 = P.r7l[gq][1], l2 = P.r7l[gq][2];
                const double yx = l0 * p[0][0] + l1 * p[1][0] + l2 * p[2][0];
                const double yy = l0 * p[0][1] + l1 * p[1][1] + l2 * p[2][1];
                const double yz = l0 * p[0][2] + l1 * p[1][2] + l2 * p[2][2];
                accumulate_ut(P, yx - x0, yy - x1, yz - x2, n, t, s, P.r7w[gq] * area, T, Ut);
            }
        }
        // subtract the far kernel's 7-point U·t for this pair (it is in the partials)
        cplx Tdummy[9];
        cplx Uf[3] = {mk(0, 0), mk(0, 0), mk(0, 0)};
#pragma unroll
        for (int i = 0; i < 9; ++i) Tdummy[i] = mk(0.0, 0.0);
        for (int gq = 0; gq < 7; ++gq) {
            const double l0 = P.r7l[gq][0], l1 = P.r7l[gq][1], l2 = P.r7l[gq][2];
            const double yx = l0 * g[0] + l1 * g[3] + l2 * g[6];
            const double yy = l0 * g[1] + l1 * g[4] + l2 * g[7];
            const double yz = l0 * g[2] + l1 * g[5] + l2 * g[8];
            accumulate_ut(P, yx - x0, yy - x1, yz - x2, n, t, s, P.r7w[gq] * g[15], Tdummy, Uf);
        }
        Ut[0] = Ut[0] - Uf[0];
        Ut[1] = Ut[1] - Uf[1];
        Ut[2] = Ut[2] - Uf[2];
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
    const double* g = geo + (size_t)e * 16;
    const double x0 = geo[(size_t)c * 16 + 9], x1 = geo[(size_t)c * 16 + 10], x2 = geo[(size_t)c * 16 + 11];
    const double n[3] = {g[12], g[13], g[14]};
    const double t[3] = {trac[3 * e], trac[3 * e + 1], trac[3 * e + 2]};
    cplx T[9], Ut[3];
#pragma unroll
    for (int i = 0; i < 9; ++i) T[i] = mk(0.0, 0.0);
    Ut[0] = Ut[1] = Ut[2] = mk(0.0, 0.0);

    if (level < 0) {
        // Self element: polar quadrature about the centroid over the 3 edge
        // sub-triangles; static antisymmetric T part as the exact CPV.
        const int NG = BemParams::kSelfGauss;
        const int npts = 3 * NG * NG;
        const cplx E10 = mk(P.E10, 0.0), E20 = mk(P.E20, 0.0);
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
            if (bq == 0) {
                const double lnR = log(R) / (R * R) * jt * (1.0 / (4.0 * kPi));
#pragma unroll
                for (int i = 0; i < 3; ++i)
#pragma unroll
                    for (int j = 0; j < 3; ++j)
                        T[3 * i + j] = T[3 * i + j] + (E10 * (ev[j] * n[i]) + E20 * (ev[i] * n[j])) * lnR;
            }
            const double u = P.glx[bq];
            const double rho = R * u;
            cplx Aa, Bb, Cc, Dd;
            abcd(P, s * (rho * P.inv_cs), Aa, Bb, Cc, Dd);
            const double w = jt * P.glw[bq];
            const double fu = w * u / rho * P.inv_4pi_mu;
            const double ft = w * u / (rho * rho) * (1.0 / (4.0 * kPi));
            const cplx dE1 = (Cc - Bb) - E10;
            const cplx dE2 = P.lam_over_mu * (Cc - Dd - 2.0 * Bb) - 2.0 * Bb - E20;
            const double et = ev[0] * t[0] + ev[1] * t[1] + ev[2] * t[2];
#pragma unroll
            for (int i = 0; i < 3; ++i) Ut[i] = Ut[i] + (Aa * t[i] - Bb * (ev[i] * et)) * fu;
#pragma unroll
            for (int i = 0; i < 3; ++i)
#pragma unroll
                for (int j = 0; j < 3; ++j)
                    T[3 * i + j] = T[3 * i + j] + (dE1 * (ev[j] * n[i]) + dE2 * (ev[i] * n[j])) * ft;
        }
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
            accumulate_ut(P, yx - x0, yy - x1, yz - x2, n, t, s, P.r7w[gq] * area, T, Ut);
        }
        // subtract the far kernel's 7-point U·t for this pair (it is in the partials)
        if (lane < 7) {
            cplx Tdummy[9];
            cplx Uf[3] = {mk(0, 0), mk(0, 0), mk(0, 0)};
            const double l0 = P.r7l[lane][0], l1 = P.r7l[lane][1], l2 = P.r7l[lane][2];
            const double yx = l0 * g[0] + l1 * g[3] + l2 * g[6];
            const double yy = l0 * g[1] + l1 * g[4] + l2 * g[7];
            const double yz = l0 * g[2] + l1 * g[5] + l2 * g[8];
#pragma unroll
            for (int i = 0; i < 9; ++i) Tdummy[i] = mk(0.0, 0.0);
            accumulate_ut(P, yx - x0, yy - x1, yz - x2, n, t, s, P.r7w[lane] * g[15], Tdummy, Uf);
            Ut[0] = Ut[0] - Uf[0];
            Ut[1] = Ut[1] - Uf[1];
            Ut[2] = Ut[2] - Uf[2];
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
    FDS_LAUNCH(bem_far_kernel, gf, kFarThreads, 0, st, d.params, d.geo, d.trac, ne, svec_dev, A,
               mstride, plane, ld, d.partial, d.pstride);
    if (B >= 8) {
        dim3 gn(ceil_div(d.npairs, 4), ceil_div(B, 32));
        FDS_LAUNCH(bem_near_kernel, gn, 128, 0, st, d.params, d.geo, d.trac, ne, d.pairs, d.npairs,
                   svec_dev, B, A, mstride, plane, ld, d.corr, d.cstride);
    } else {
        dim3 gn(ceil_div(d.npairs * 32, 128), B);
        FDS_LAUNCH(bem_near_pts_kernel, gn, 128, 0, st, d.params, d.geo, d.trac, ne, d.pairs, d.npairs,
                   svec_dev, A, mstride, plane, ld, d.corr, d.cstride);
    }
    dim3 gr(ceil_div(3 * ne, 128), B);
    FDS_LAUNCH(bem_rhs_kernel, gr, 128, 0, st, ne, nchunks, d.partial, d.pstride, d.near_ptr, d.corr,
               d.cstride, svec_dev, rhs, rstride);
}

}  // namespace fdsb
