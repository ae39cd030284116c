/*
 * fdsweep_b200 — C-ABI of the B200-native hot path behind the reference
 * toolkit's solver/fitting/inversion API (arxiv 1511.04355, `fdsweep`).
 *
 * Plain pointers and sizes only; no CUDA or torch types. Complex numbers are
 * `fds_c64` = two doubles (re, im), layout-identical to std::complex<double>
 * (proj/include/fdsweep/types.hpp:10) so a C++ caller passes
 * reinterpret_cast<const fds_c64*>(vec.data()).
 *
 * Status codes map one-to-one onto the reference's exception classes
 * (proj/include/fdsweep/types.hpp:14-36): FDS_EVALIDATION -> ValidationError,
 * FDS_ENUMERIC -> NumericError, FDS_EIO -> IoError, FDS_ECONVERGENCE ->
 * ConvergenceError. FDS_ECUDA means the device path failed (no fallback
 * exists). fds_last_error() returns the thread-local message of the last
 * failing call on this thread.
 *
 * Host layouts follow the reference: samples are per-frequency AoS
 * values[j*K + k] (FrequencySample::values, types.hpp:40-45), residues are
 * channel-major res[k*M + m] (RationalModel::residues, vecfit.hpp:21-30),
 * time series are channel-major out[k*T + n] (TimeSeries::values, types.hpp:48-56).
 */
#ifndef FDSWEEP_B200_H
#define FDSWEEP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef struct {
    double re, im;
} fds_c64;

enum {
    FDS_OK = 0,
    FDS_EVALIDATION = 1,
    FDS_ENUMERIC = 2,
    FDS_EIO = 3,
    FDS_ECONVERGENCE = 4,
    FDS_ECUDA = 5
};

const char* fds_last_error(void);
/* Version string of the library ("fdsweep_b200 <semver> sm_100a"). */
const char* fds_version(void);
/* Select the CUDA device for subsequent calls on this thread. */
int fds_set_device(int device);

/* ------------------------------------------------------------------------
 * BEM frequency system — replaces FrequencySystem::evaluate(Complex s)
 * (proj/include/fdsweep/systems.hpp:34-42; called by run_afs at
 * proj/src/afs.cpp:293 and by the FSM sweep).
 * Laplace-domain 3D elastodynamic collocation BEM on constant flat
 * triangles; unknowns element-major u[3e + {x,y,z}]; load = per-element
 * traction vector x Heaviside factor 1/s. The handle is immutable after
 * create; evaluate is reentrant (calls are serialised per handle on its own
 * stream; factorizations of different handles in one process are serialised
 * per device) and deterministic: a frequency solved in a batch of the same
 * size gives bit-identical results on every call (all reductions have a fixed
 * order; the batch chunk size of a handle with max_batch = 0 is fixed at its
 * first evaluate). Across batch sizes the 3M trailing update groups its
 * rank-64 (single matrix) or rank-128 (batch) updates differently, so the
 * same s agrees to rounding (~1e-15 relative), not bit for bit;
 * FDSWEEP_GEMM=4m restores bit-identity across batch sizes.
 * ---------------------------------------------------------------------- */
typedef struct fds_bem fds_bem;

typedef struct {
    int n_vertices;
    const double* vertices;   /* [n_vertices][3] */
    int n_elements;
    const int* triangles;     /* [n_elements][3]; (v1-v0)x(v2-v0) = domain-outward normal */
    double shear_modulus;     /* mu */
    double poisson_ratio;     /* nu */
    double density;           /* rho */
    const double* traction;   /* [n_elements][3], multiplied by p(s) = 1/s */
    int n_channels;           /* output DOFs; 0 => all 3*n_elements */
    const int* channels;      /* DOF indices into u */
    int max_batch;            /* frequencies solved concurrently; 0 => from the free HBM at the first evaluate */
} fds_bem_desc;

int fds_bem_create(const fds_bem_desc* desc, fds_bem** out);
int fds_bem_destroy(fds_bem* bem);
int fds_bem_channels(const fds_bem* bem);
int fds_bem_unknowns(const fds_bem* bem);
/* One solve: out[k] = u_channel_k(s). Host buffers. */
int fds_bem_evaluate(fds_bem* bem, fds_c64 s, fds_c64* out);
/* B independent solves (batched assembly + LU + solve): out[b*K + k]. Host buffers. */
int fds_bem_evaluate_batch(fds_bem* bem, const fds_c64* s, int B, fds_c64* out);
/* Same, device-resident result (pointer to B*K fds_c64 in HBM, valid until the
 * next call on this handle); used by the bench to time the path without copies. */
int fds_bem_evaluate_batch_device(fds_bem* bem, const fds_c64* s, int B, const fds_c64** dev_out);
/* Debug / parity: assembled A(s) (column-major N x N) and b(s) to host. */
int fds_bem_assemble_host(fds_bem* bem, fds_c64 s, fds_c64* A, fds_c64* b);
/* Verification at sizes where A(s) should not cross PCIe: assembles A(s), b(s)
 * on the device and returns A[rows[i], cols[i]] for i < count (and b if
 * non-NULL, n entries). Pins the assembly kernels against the CPU oracle's
 * BemOracle::assemble entrywise (no reference counterpart: SPEC.md:9). */
int fds_bem_assemble_entries(fds_bem* bem, fds_c64 s, int count, const int* rows, const int* cols,
                             fds_c64* A_entries, fds_c64* b);
/* Backward error of a solution u (n unknowns, host): assembles A(s), b(s) on
 * the device; norms[0..3] = ||A u - b||_2, ||A||_inf, ||u||_2, ||b||_2. */
int fds_bem_residual(fds_bem* bem, fds_c64 s, const fds_c64* u, double* norms);
/* Per-stage device times of the last evaluate_batch call (ms): assembly, LU, solve;
 * and the number of kernel launches it issued. */
int fds_bem_last_timing(const fds_bem* bem, double* assembly_ms, double* lu_ms, double* solve_ms,
                        int* launches);

/* Solver of subsequent evaluate calls: kind 0 = batched LU with partial
 * pivoting (default); kind 1 = restarted GMRES on the assembled dense A (all
 * frequencies of a batch in lockstep, right block-Jacobi on the 3x3 element
 * blocks), stopping at ||b - A u|| <= tol ||b||. A frequency whose GMRES misses
 * tol within max_iter (e.g. near an interior resonance) is solved by LU
 * instead. For large N one O(N^2) product per iteration beats the O(N^3)
 * factorization. */
/* Device stage times summed over every solve since create (or the last reset):
 * out[0..3] = assembly ms, LU (or GMRES) ms, solve ms, frequencies solved. */
int fds_bem_cumulative_timing(fds_bem* bem, double* out, int reset);
int fds_bem_set_solver(fds_bem* bem, int kind, double tol, int restart, int max_iter);
/* Of the last evaluate: largest GMRES iteration count, largest true relative
 * residual of the GMRES-solved frequencies, number of LU fallbacks. */
int fds_bem_last_gmres(const fds_bem* bem, int* iterations, double* rel_residual, int* lu_fallbacks);

/* Dense complex LU + solve on the device for caller-provided host matrices
 * (column-major, B matrices of order n): x[b] = A[b]^{-1} rhs[b]. */
int fds_zgesv_batch(int n, int B, const fds_c64* A, const fds_c64* rhs, fds_c64* x);
/* Device-resident variant: A (planar: re plane then im plane,
 * column-major, B consecutive matrices) is factored in place; returns ms. */
int fds_lu_factor_device(int n, int B, double* A_planar, int* ipiv, int* info, double* ms);

/* ------------------------------------------------------------------------
 * Vector fitting — replaces proj/src/vecfit.cpp (vecfit.hpp:48-86).
 * ---------------------------------------------------------------------- */
/* relocate_poles (vecfit.cpp:188-354): samples restricted to K channels. */
int fds_vf_relocate(int J, int K, const fds_c64* s, const fds_c64* values, int M,
                    const fds_c64* poles_in, fds_c64* poles_out, double* per_channel_rms,
                    double* movement);
/* identify_residues for K channels at once (vecfit.cpp:356-408 applied per channel;
 * the LS matrix is shared): res[k*M + m], rms[k] (may be NULL). */
int fds_vf_identify_residues(int J, int K, const fds_c64* s, const fds_c64* values, int M,
                             const fds_c64* poles, fds_c64* residues, double* rms);
/* vector_fit (vecfit.cpp:410-488). report_i = {iterations_used, unstable_pole_count},
 * report_d = {pole_movement}; per_channel_rms[K], relocation_rms[n_orf] may be NULL. */
int fds_vector_fit(int J, int K, const fds_c64* s, const fds_c64* values, int n_orf,
                   const int* orf, int order, int n_relocations, fds_c64* poles_out,
                   fds_c64* residues_out, int* report_i, double* report_d,
                   double* per_channel_rms, double* relocation_rms);
/* eval_model (vecfit.cpp:503-509) at G points: out[g*K + k]. */
/* Frees the calling thread's VF / Laplace device workspaces, including the
 * cached identify_residues solve operator (reused while (s, poles) repeat). */
int fds_vf_release_workspace(void);
int fds_eval_model(int M, const fds_c64* poles, int K, const fds_c64* residues, int G,
                   const fds_c64* s, fds_c64* out);
/* fit_error_evf (vecfit.cpp:511-526): E_vf of one channel of the model
 * (residues [K][M]) against samples values[j*K + k] at s[J]; on the device. */
int fds_fit_error_evf(int M, const fds_c64* poles, int K, const fds_c64* residues, int channel, int J,
                      const fds_c64* s, const fds_c64* values, double* out);
/* channel_errors (afs.cpp:118-145): e[k] = max_g|fH-fL| / max_g|fH|. */
int fds_channel_errors(int MH, const fds_c64* poles_h, const fds_c64* res_h, int ML,
                       const fds_c64* poles_l, const fds_c64* res_l, int K, int G,
                       const fds_c64* grid, double* errors);
/* select_new_frequency (afs.cpp:147-187). */
int fds_select_new_frequency(int MH, const fds_c64* poles_h, const fds_c64* res_h, int ML,
                             const fds_c64* poles_l, const fds_c64* res_l, int K, int G,
                             const fds_c64* grid, int n_existing, const fds_c64* existing,
                             int n_orf, const int* orf_positions, double exclusion_radius,
                             fds_c64* s_new);

/* ------------------------------------------------------------------------
 * Time reconstruction — replaces proj/src/laplace.cpp (laplace.hpp:40-59).
 * ---------------------------------------------------------------------- */
/* fsm_invert (laplace.cpp:89-125): half[k*(Ns/2+1) + i] -> out[k*Ns + n]. */
int fds_fsm_invert(double period, int Ns, double eta, int K, const fds_c64* half, int hanning,
                   double* out);
/* rational_invert (laplace.cpp:127-164): out[k*T + n]. */
int fds_rational_invert(int M, const fds_c64* poles, int K, const fds_c64* residues, int T,
                        const double* t, double* out);

/* Device-resident VF/FSM stage (config 5): data pointers are HBM, the small
 * s / poles / t vectors host. residues: [m*K + k] (canonical pole order);
 * values: [j*K + k]; half: [i*K + k] (frequency-major); out: [k*Ns + n] /
 * [k*T + n]. ms (optional) = device time of the whole call (CUDA events on the
 * library stream around every launch the call makes, shared QR included). */
int fds_vf_identify_residues_device(int J, int K, const fds_c64* s_host, const fds_c64* values_dev,
                                    int M, const fds_c64* poles_host, fds_c64* residues_dev,
                                    double* ms);
/* Same, but the conjugate row m+1 of every pole pair (canonical order: pairs
 * adjacent, +Im first) is left unwritten — it equals conj(row m). For
 * consumers that use the pair symmetry (fds_rational_invert_device reads only
 * the pair heads and the real poles); saves 8 M bytes of HBM writes per DOF. */
int fds_vf_identify_residues_device_heads(int J, int K, const fds_c64* s_host, const fds_c64* values_dev,
                                          int M, const fds_c64* poles_host, fds_c64* residues_dev,
                                          double* ms);
int fds_rational_invert_device(int M, const fds_c64* poles_host, int K, const fds_c64* residues_dev,
                               int T, const double* t_host, double* out_dev, double* ms);
int fds_fsm_invert_device(double period, int Ns, double eta, int K, const fds_c64* half_dev,
                          int hanning, double* out_dev, double* ms);
/* Same with explicit element strides: half[k*stride_k + i*stride_i] (stride_k =
 * Ns/2+1, stride_i = 1 is the per-channel layout of fsm_invert). */
int fds_fsm_invert_device_strided(double period, int Ns, double eta, int K, const fds_c64* half_dev,
                                  long long stride_k, long long stride_i, int hanning, double* out_dev,
                                  double* ms);

/* ------------------------------------------------------------------------
 * AFS driver — replaces run_afs (proj/src/afs.cpp:226-396) for a BEM system
 * or a rational/modal closed-form system (evaluated on the host).
 * ---------------------------------------------------------------------- */
typedef struct {
    int initial_count;      /* J0 */
    double alpha_high, alpha_low;
    double e1_threshold, e2_threshold;
    int validation_steps;   /* J_c */
    int n_orf;
    const int* orf_indices; /* NULL/0 => draw 5 with seed */
    int n_test;
    const int* test_indices; /* NULL/0 => all channels */
    double omega_max, eta, period;
    int grid_points, time_points, max_iterations;
    uint64_t seed;
    int n_relocations;
} fds_afs_config;

typedef struct {
    int n_c;
    int converged;
    int solver_calls;
    int n_history;
    int order;              /* M_H of the final model */
    int n_orf;              /* ORF channels the driver used (drawn with the seed when cfg->n_orf == 0, */
    int orf_indices[8];     /* afs.cpp:234-236); the first min(n_orf, 8) are listed */
} fds_afs_summary;

/* Callback system for non-BEM systems: fills out[K] at s; returns 0 on success. */
typedef int (*fds_system_fn)(void* user, fds_c64 s, fds_c64* out);

/* samples_s[cap], history[cap*8] rows {J, MH, ML, has_s_new, re, im, E1, E2},
 * poles[cap], residues[K*cap] (final model over all channels, [k*order+m]).
 * On an error status (the reference's exception classes) the samples, sample
 * values, history and summary (order = 0) still hold the iterations completed
 * before the failure, so a caller can report where the sweep stopped. */
int fds_run_afs_bem(fds_bem* bem, const fds_afs_config* cfg, int cap, fds_c64* samples_s,
                    fds_c64* sample_values, double* history, fds_c64* poles, fds_c64* residues,
                    fds_afs_summary* summary);
int fds_run_afs_callback(fds_system_fn fn, void* user, int channels, const fds_afs_config* cfg,
                         int cap, fds_c64* samples_s, fds_c64* sample_values, double* history,
                         fds_c64* poles, fds_c64* residues, fds_afs_summary* summary);

/* Count of kernels this library launched since load (evidence for the bench). */
int64_t fds_kernel_launches(void);
/* Per-kernel device timing for roofline reporting. enable(1) clears and starts
 * recording (CUDA events around each launch of the profiled kernels on their
 * own stream); read() sums launches of one kind: 0 LU GEMM (work = FP64 flops),
 * 1 LU panel, 2 LU swap+TRSM, 3 assembly far field, 4 assembly near field,
 * 5 VF residue apply (work = bytes), 6 rational invert, 7 FSM, 8 channel errors. */
int fds_profile_enable(int on);
int fds_profile_read(int kind, int* count, double* total_ms, double* total_work);

/* Debug: red-zone check of the library's device allocations (no reference
 * counterpart; stands in for compute-sanitizer memcheck, which this GPU pool
 * does not allow). With FDSWEEP_REDZONE set in the environment before the
 * library loads, every cudaMalloc carries a 4 KB guard zone on each side;
 * this call synchronises the device, compares the zones of all live
 * allocations and returns the bytes found overwritten so far (freed
 * allocations included), the number of zone checks made and the live
 * allocation count. enabled = 0 and zeros when the mode is off. */
int fds_debug_redzone_check(int* enabled, long long* overwritten_bytes, long long* checks, long long* live);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif

#endif /* FDSWEEP_B200_H */
