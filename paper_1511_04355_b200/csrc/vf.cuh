// Vector fitting on sm_100a: shared declarations (vf.cu, laplace.cu, afs.cpp).
#pragma once

#include <complex>
#include <vector>

#include "common.cuh"

namespace fdsb {

using Cx = std::complex<double>;

// Thread-local device workspace shared by the VF / Laplace / AFS entry points
// (growable buffers, one non-blocking stream). Avoids per-call cudaMalloc in
// the AFS loop.
struct VfContext {
    cudaStream_t st = nullptr;
    struct Buf {
        void* p = nullptr;
        size_t bytes = 0;
        void* get(size_t need);
    };
    Buf values, resid, W, phi, rms, tab, tab2, out, misc, misc2, qr, lsq, lsq_io, chanerr;
    std::vector<double> w_key;  // (J, M, s, poles) of the solve operator held in W
    bool w_valid = false;
    void release();  // frees every buffer (and forgets the cached solve operator)
    static VfContext& get();
};

// ------------------------------------------------------------------ device least squares (vf_lsq.cu)
struct VfLsqStatus {
    int rank, nonzero;
    double maxpivot;
};
// Column-pivoted QR least squares of the m x n system in(i, j) = in[i*rs + j*cs]
// on one CTA: x_out = solution for rhs, or w_out[c*m + i] = wscale[c] W(c, i)
// (explicit solve operator). status->rank < n means rank-deficient (no output).
void vf_lsq_launch(int m, int n, const double* in, long long rs, long long cs, const double* rhs, double* x_out,
                   double* w_out, const double* wscale, VfLsqStatus* status, cudaStream_t st, int m_thr = 0);
// The stacked sigma system of relocate_poles (K blocks of red rows x M, row-major
// r22[(k red + i) M + c], rhs beta): solved directly when it fits on chip, else
// folded to M x M first (vf_stack_fold_kernel). y receives the M-vector.
void vf_lsq_stacked_launch(int K, int red, int M, const double* r22, const double* beta, double* y,
                           VfLsqStatus* status, cudaStream_t st);
// Does the m x n system (with one or kLsqCols right-hand sides) fit one CTA?
bool vf_lsq_fits(int m, int n, bool single_rhs);
// Explicit solve operator of a system too large for one CTA (column-major a,
// m x n): folded QR -> pivoted QR of the n x n factor (Eigen's rank rule with
// the original m) -> W by triangular solves against R (see vf_lsq.cu).
void vf_lsq_operator_large(int m, int n, const double* a, const double* wscale, double* w_out, VfLsqStatus* status,
                           cudaStream_t st);
void vf_reloc_rms_launch(int K, int red, int M, int J, const double* r22, const double* beta, const double* tail,
                         const double* y, double* rms, cudaStream_t st);

// ------------------------------------------------------------------ host helpers
std::vector<Cx> canonical_order(const std::vector<Cx>& poles);  // vecfit.cpp:134-169
bool conj_closed(const std::vector<Cx>& poles, double tol = 1e-9);  // vecfit.cpp:116-132
void require_distinct(const std::vector<Cx>& s);                 // vecfit.cpp:20-30
std::vector<Cx> start_poles(double omega_max, int order);        // vecfit.cpp:171-186

struct RelocResult {
    std::vector<Cx> poles;
    std::vector<double> rms;
    double movement = 0.0;
};

// relocate_poles on K channels of host samples (values [j][k]).
RelocResult vf_relocate(const std::vector<Cx>& s, const Cx* values, int K, const std::vector<Cx>& poles_in);

// identify_residues for K channels whose values live on the device as
// [j][k] complex (values_dev); residues written on the device as [m][k];
// rms_dev (K doubles) optional. Poles must already be canonical. heads_only:
// the conjugate row m+1 of each pole pair is not written (its values are
// conj(row m); consumers that use the pair symmetry never read it).
void vf_residues_device(const std::vector<Cx>& s, const cplx* values_dev, int K,
                        const std::vector<Cx>& poles, cplx* res_dev, double* rms_dev, cudaStream_t st,
                        bool heads_only = false);

// eval_model (vecfit.cpp:490-509) on the device: out[g*K + k], residues [k][m].
void vf_eval_model(const std::vector<Cx>& poles, const Cx* res_km, int K, const std::vector<Cx>& s, Cx* out);
// fit_error_evf (vecfit.cpp:511-526) of one channel: residues res_k[m], data[j*dstride].
double vf_fit_error_evf(const std::vector<Cx>& poles, const Cx* res_k, const std::vector<Cx>& s, const Cx* data,
                        int dstride);

struct FitReportC {
    int iterations = 0;
    double movement = 0.0;
    int unstable = 0;
    std::vector<double> rms, reloc_rms;
};

// vector_fit over host samples; residues returned [k][m].
void vf_vector_fit(const std::vector<Cx>& s, const Cx* values, int K, const std::vector<int>& orf, int order,
                   int n_reloc, std::vector<Cx>& poles, std::vector<Cx>& residues_km, FitReportC* rep);

// channel_errors (afs.cpp:118-145) for two models over a grid; residues [k][m].
std::vector<double> vf_channel_errors(const std::vector<Cx>& ph, const std::vector<Cx>& rh,
                                      const std::vector<Cx>& pl, const std::vector<Cx>& rl, int K,
                                      const std::vector<Cx>& grid);
// select_new_frequency (afs.cpp:147-187) given precomputed channel errors.
Cx vf_select_new_frequency(const std::vector<Cx>& ph, const std::vector<Cx>& rh, const std::vector<Cx>& pl,
                           const std::vector<Cx>& rl, int K, const std::vector<Cx>& grid,
                           const std::vector<Cx>& existing, const std::vector<int>& orf_pos, double radius,
                           const std::vector<double>* errors);

// ---- device-resident AFS iteration
// vector_fit whose residue step reads samples [j][k] already in HBM and leaves
// residues [m][k] in HBM; relocation runs on the ORF values (host, [j][|orf|]).
// Returns the canonical poles.
std::vector<Cx> vf_vector_fit_device(const std::vector<Cx>& s, const Cx* values_orf, const cplx* values_dev, int K,
                                     const std::vector<int>& orf, int order, int n_reloc, cplx* res_dev,
                                     cudaStream_t st);
struct AfsErrReduce {
    double e2;   // max over the test positions of e_k
    int kmax;    // worst ORF channel position (first strict max in ORF order)
    int zero_k;  // first channel with an identically zero high-order fit, or -1
};
// channel_errors of two device-resident models (residues [m][k]) into ce_dev
// [k][2] = (max|fH-fL|, max|fH|), reduced into *red_dev; synchronises st.
void vf_channel_errors_device(const std::vector<Cx>& ph, const cplx* rh_mk, const std::vector<Cx>& pl,
                              const cplx* rl_mk, int K, const std::vector<Cx>& grid, const int* test_pos_dev, int KT,
                              const int* orf_pos_dev, int KO, double* ce_dev, AfsErrReduce* red_dev,
                              cudaStream_t st);
// select_new_frequency's grid scan for one channel whose residues sit at
// rh_k[m*mstride], rl_k[m*mstride] on the device; returns the grid index.
int vf_select_device(const std::vector<Cx>& ph, const cplx* rh_k, const std::vector<Cx>& pl, const cplx* rl_k,
                     size_t mstride, const std::vector<Cx>& grid, const std::vector<Cx>& existing, double radius,
                     cudaStream_t st);
// dst[m][q] = src[m][pos[q]] for q < KT (channel subset of a [m][K] residue block)
void vf_gather_channels(const cplx* src_mk, int K, int M, const int* pos_dev, int KT, cplx* dst_mk, cudaStream_t st);
// rational_invert of a device-resident model (residues [m][k], exact conjugate
// pairs as the residue kernels write them) into out_dev [k][t], with
// rational_invert's validation.
void rat_invert_mk_device(const std::vector<Cx>& poles, const cplx* res_mk_dev, int K, const std::vector<double>& t,
                          double* out_dev, cudaStream_t st);

// rational_invert (laplace.cpp:127-164): host model -> host out[k][t].
void rat_invert_host(const std::vector<Cx>& poles, const std::vector<Cx>& res_km, int K,
                     const std::vector<double>& t, double* out);
// host model -> series left in HBM (out_dev, [k][t]).
void rat_invert_to_device(const std::vector<Cx>& poles, const std::vector<Cx>& res_km, int K,
                          const std::vector<double>& t, double* out_dev, cudaStream_t st);
// error_e1 (afs.cpp:189-216) of two device-resident series [k][t]; bit-identical to the host sums.
double afs_error_e1_device(const std::vector<double>& t, const double* cur_dev, const double* prev_dev, int K,
                           cudaStream_t st);
// device variant: residues on device [m][k]; paired = residues exactly conjugate per pair.
void rat_invert_device(const std::vector<Cx>& poles, const cplx* res_mk_dev, int K, const std::vector<double>& t,
                       double* out_dev, bool paired, cudaStream_t st);

// fsm_invert (laplace.cpp:89-125): half spectra element (k, i) at half[k*sk + i*si] (device).
void fsm_invert_device(double period, int Ns, double eta, int K, const cplx* half_dev, size_t sk, size_t si,
                       bool hanning, double* out_dev, cudaStream_t st);

}  // namespace fdsb
