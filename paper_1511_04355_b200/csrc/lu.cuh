// Batched / blocked complex LU with partial pivoting on sm_100a.
#pragma once

#include <mutex>

#include "common.cuh"

namespace fdsb {

// B matrices of order n, planar FP64 (re plane then im plane, each ld x ld,
// column-major); matrix b starts at A + b*mstride, im plane at +plane.
struct LuProblem {
    double* A = nullptr;
    size_t mstride = 0;
    size_t plane = 0;
    int n = 0;
    int ld = 0;
    int batch = 0;
    int* ipiv = nullptr;  // [batch][n], 0-based row swapped with row c at step c
    int* info = nullptr;  // [batch], 0 = ok, c+1 = first zero pivot
};

struct LuWorkspace {
    // side stream + events of the look-ahead schedule (per workspace, so
    // concurrent handles never share them)
    cudaStream_t side = nullptr;
    cudaEvent_t ev[8] = {};
    void ensure_side();
    double* linv_buf = nullptr;  // [batch][2][64][64] L11^{-1} per panel
    int linv_cap = 0;
    double* linv(int batch);
    // 3M trailing update: pre-formed operand planes (Re+Im, Re-Im of L21 [batch][2][128][ld];
    // Re+Im of U12 [batch][ld][kG3Rows]) and the (A, ld, batch) they were encoded for
    double* g3 = nullptr;
    size_t g3_cap = 0;
    double* g3_planes(const LuProblem& pb);
    const double* g3_key_A = nullptr;  // L21 planes currently formed for (A, k, w)
    int g3_key_k = -1, g3_key_w = -1;
    // row-interchange groups of the last factorization: columns [0, super_end)
    // were factored as 128-column super-panels (LAPACK order inside each), the
    // rest as nb-column panels; LINPACK order across groups
    int super_end = 0;
    int super256_end = 0;  // columns [0, super256_end) were factored as 256-column super-panels
    // dataflow solve: forward results [batch][n], per-panel pivot flags, block flags, tickets
    cplx* ybuf = nullptr;
    size_t ybuf_cap = 0;
    int* sflags = nullptr;
    size_t sflag_cap = 0;
    void ensure_solve(int batch, int n, int nblk);
    double* slots = nullptr;
    unsigned* counters = nullptr;
    size_t slot_bytes = 0;
    int counter_count = 0;
    void ensure(int groups, int P, int nb);
    void release();
    LuWorkspace() = default;
    LuWorkspace(const LuWorkspace&) = delete;
    LuWorkspace& operator=(const LuWorkspace&) = delete;
    ~LuWorkspace() { release(); }
};

inline int lu_ld(int n) { return (n + 63) / 64 * 64; }
inline size_t lu_plane(int n) { return static_cast<size_t>(lu_ld(n)) * lu_ld(n); }

// Process-wide, per-device gate held by every caller of lu_factor from the
// enqueue until the factorization has completed on the device. The
// single-matrix look-ahead schedule launches its software-barrier panel kernel
// (lu_panel_kernel, CTAs spin on a global counter) next to its own trailing
// GEMM on a second stream; that is safe because the GEMM's CTAs retire, but
// panels of two handles running at once could fill the SMs with spinning CTAs.
// Holding the gate serialises factorizations of different handles/threads in
// one process. (Other processes on the same GPU — MPS — are not covered: run
// one process per GPU, as the bench and the driver do.)
std::unique_lock<std::mutex> lu_device_gate();

// Per-step timings are not taken here; the caller brackets with events.
void lu_factor(const LuProblem& pb, LuWorkspace& ws, cudaStream_t st);
// rhs[b*rstride + i], complex interleaved, overwritten with the solution
// (dataflow substitution; FDSWEEP_SOLVE=blocked selects the per-panel launches).
void lu_solve(const LuProblem& pb, cplx* rhs, size_t rstride, LuWorkspace& ws, cudaStream_t st);
int lu_panel_width(int n);

}  // namespace fdsb
