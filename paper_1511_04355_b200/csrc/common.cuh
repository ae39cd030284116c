// Shared device/host helpers for the fdsweep_b200 sm_100a library.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "fdsweep_b200.h"

namespace fdsb {

// Error classes mirror proj/include/fdsweep/types.hpp:14-36; the C-ABI maps
// each onto its FDS_E* status.
struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct ValidationError : Error { using Error::Error; };
struct NumericError : Error { using Error::Error; };
struct IoError : Error { using Error::Error; };
struct ConvergenceError : Error { using Error::Error; };
struct CudaError : Error { using Error::Error; };

extern std::atomic<int64_t> g_launches;

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------- red-zone allocations (debug)
// compute-sanitizer is closed on this GPU pool, so out-of-bounds WRITES are
// looked for here instead: with FDSWEEP_REDZONE set (read once), every
// cudaMalloc of the library is widened by a 4 KB zone on each side filled with
// 0xA5, the back zone starting at the first byte past the requested size; the
// zones are compared on cudaFree and by fds_debug_redzone_check (all live
// allocations). The allocation itself is pre-filled with 0xFF (NaN / -1). Off by default: the macros below then forward unchanged.
struct RedzoneRegistry {
    struct Rec { void* base; size_t bytes; };
    std::mutex mu;
    std::map<void*, Rec> live;
    long long violations = 0, checked = 0;
    static constexpr size_t kZone = 4096;
    static constexpr unsigned char kFill = 0xA5;
    static bool enabled() {
        static const bool on = std::getenv("FDSWEEP_REDZONE") != nullptr;
        return on;
    }
    static RedzoneRegistry& get() {
        static RedzoneRegistry r;
        return r;
    }
    static size_t back_bytes(size_t bytes) { return kZone + (256 - bytes % 256) % 256; }
    // caller holds mu; the device must be idle with respect to the allocation
    long long check_one(void* user, const Rec& rec) {
        const size_t back = back_bytes(rec.bytes);
        std::vector<unsigned char> h(kZone + back);
        if (::cudaMemcpy(h.data(), rec.base, kZone, cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
        if (::cudaMemcpy(h.data() + kZone, static_cast<char*>(user) + rec.bytes, back, cudaMemcpyDeviceToHost) !=
            cudaSuccess)
            return 0;
        long long bad = 0;
        for (unsigned char c : h) bad += c != kFill;
        ++checked;
        if (bad)
            std::fprintf(stderr, "fdsweep_b200 redzone: %lld bytes overwritten around a %zu-byte allocation\n", bad,
                         rec.bytes);
        return bad;
    }
};

template <class T>
inline cudaError_t rz_malloc(T** out, size_t bytes) {
    if (!RedzoneRegistry::enabled()) return ::cudaMalloc(reinterpret_cast<void**>(out), bytes);
    auto& rz = RedzoneRegistry::get();
    const size_t back = RedzoneRegistry::back_bytes(bytes);
    void* base = nullptr;
    const cudaError_t e = ::cudaMalloc(&base, RedzoneRegistry::kZone + bytes + back);
    if (e != cudaSuccess) return e;
    char* user = static_cast<char*>(base) + RedzoneRegistry::kZone;
    ::cudaMemset(base, RedzoneRegistry::kFill, RedzoneRegistry::kZone);
    ::cudaMemset(user + bytes, RedzoneRegistry::kFill, back);
    // initcheck stand-in: fresh memory reads as NaN doubles / -1 ints, so a result that
    // depends on bytes the library never wrote fails the parity tests run in this mode
    ::cudaMemset(user, 0xFF, bytes);
    // the fills run on the legacy stream; the library's streams are non-blocking, so
    // finish them before the allocation is handed out
    ::cudaDeviceSynchronize();
    std::lock_guard<std::mutex> lk(rz.mu);
    rz.live[user] = {base, bytes};
    *out = reinterpret_cast<T*>(user);
    return cudaSuccess;
}

inline cudaError_t rz_free(void* p) {
    if (!RedzoneRegistry::enabled() || !p) return ::cudaFree(p);
    auto& rz = RedzoneRegistry::get();
    std::lock_guard<std::mutex> lk(rz.mu);
    auto it = rz.live.find(p);
    if (it == rz.live.end()) return ::cudaFree(p);
    ::cudaDeviceSynchronize();
    rz.violations += rz.check_one(p, it->second);
    void* base = it->second.base;
    rz.live.erase(it);
    return ::cudaFree(base);
}
#define FDS_CUDA(x) ::fdsb::cuda_check((x), #x)

// Opt a kernel into `bytes` of dynamic shared memory (> 48 KB needs the
// attribute), tracked per (device, kernel) — several template instances
// launched from one generic lambda must not share one "already set" flag, and
// the attribute is per device context.
inline void ensure_dynamic_smem(const void* fn, size_t bytes) {
    if (bytes <= 48 * 1024) return;
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> done;
    std::lock_guard<std::mutex> lk(mu);
    size_t& have = done[{dev, fn}];
    if (bytes <= have) return;
    cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)),
               "cudaFuncSetAttribute(MaxDynamicSharedMemorySize)");
    have = bytes;
}
// Once-per-(device, key) initialisation (constant-memory tables, occupancy queries).
template <class F>
inline void once_per_device(const void* key, F init) {
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, bool> done;
    std::lock_guard<std::mutex> lk(mu);
    bool& d = done[{dev, key}];
    if (!d) {
        init();
        d = true;
    }
}
// Every kernel launch of the library goes through this (launch accounting +
// immediate launch-error check).
// FDSWEEP_SYNC_LAUNCH (debug): synchronise after every launch so a faulting kernel is named
inline bool sync_launches() {
    static const bool on = std::getenv("FDSWEEP_SYNC_LAUNCH") != nullptr;
    return on;
}
#define FDS_LAUNCH(kernel, grid, block, smem, stream, ...)                        \
    do {                                                                           \
        kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);               \
        ::fdsb::g_launches.fetch_add(1, std::memory_order_relaxed);               \
        ::fdsb::cuda_check(cudaGetLastError(), #kernel);                           \
        if (::fdsb::sync_launches())                                               \
            ::fdsb::cuda_check(cudaStreamSynchronize(stream), #kernel " (FDSWEEP_SYNC_LAUNCH)"); \
    } while (0)

// ---------------------------------------------------------------- complex
struct cplx {
    double re, im;
};
__host__ __device__ __forceinline__ cplx mk(double r, double i) { return {r, i}; }
__host__ __device__ __forceinline__ cplx operator+(cplx a, cplx b) { return {a.re + b.re, a.im + b.im}; }
__host__ __device__ __forceinline__ cplx operator-(cplx a, cplx b) { return {a.re - b.re, a.im - b.im}; }
__host__ __device__ __forceinline__ cplx operator-(cplx a) { return {-a.re, -a.im}; }
__host__ __device__ __forceinline__ cplx operator*(cplx a, cplx b) {
    return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
__host__ __device__ __forceinline__ cplx operator*(cplx a, double s) { return {a.re * s, a.im * s}; }
__host__ __device__ __forceinline__ cplx operator*(double s, cplx a) { return {a.re * s, a.im * s}; }
__host__ __device__ __forceinline__ cplx operator+(cplx a, double s) { return {a.re + s, a.im}; }
__host__ __device__ __forceinline__ cplx conjg(cplx a) { return {a.re, -a.im}; }
__host__ __device__ __forceinline__ double abs2(cplx a) { return a.re * a.re + a.im * a.im; }
// Smith's algorithm (scaled), robust for the magnitudes met here.
__host__ __device__ __forceinline__ cplx cdiv(cplx a, cplx b) {
    if (fabs(b.re) >= fabs(b.im)) {
        const double r = b.im / b.re, d = b.re + b.im * r;
        return {(a.re + a.im * r) / d, (a.im - a.re * r) / d};
    }
    const double r = b.re / b.im, d = b.re * r + b.im;
    return {(a.re * r + a.im) / d, (a.im * r - a.re) / d};
}
__host__ __device__ __forceinline__ cplx crecip(cplx b) { return cdiv(mk(1.0, 0.0), b); }
__device__ __forceinline__ cplx cexpd(cplx z) {
    double s, c;
    sincos(z.im, &s, &c);
    const double e = exp(z.re);
    return {e * c, e * s};
}

inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
inline PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        cuda_check(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q),
                   "cudaGetDriverEntryPoint(cuTensorMapEncodeTiled)");
        if (!fn || q != cudaDriverEntryPointSuccess) throw CudaError("cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    return encode;
}

// Timing-perturbation points for the race stress test (tests/test_gpu_race_stress.py):
// compiled to nothing in the product library; the FDS_JITTER build
// (libfdsweep_b200_jitter.so) sleeps a pseudo-random 0-8 us at every point, so
// a missing fence or barrier in a hand-rolled synchronisation protocol shows
// up as results that are no longer bit-identical to the product library's.
#ifdef FDS_JITTER
__device__ __forceinline__ void fds_jitter(unsigned salt) {
    unsigned h = (blockIdx.x * 73856093u) ^ (blockIdx.y * 2654435761u) ^ (blockIdx.z * 40503u) ^
                 (threadIdx.x * 19349663u) ^ (salt * 83492791u) ^ static_cast<unsigned>(clock64());
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    h ^= h >> 15;
    if ((h & 3u) == 0u) __nanosleep(h % 8192u);
}
#else
__device__ __forceinline__ void fds_jitter(unsigned) {}
#endif

// ---------------------------------------------------------------- mbarrier / TMA (sm_90+ async proxy)
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(bar))),
                 "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n"
                 ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(bar))), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
        ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0),
        "r"(c1), "r"(c2), "r"(static_cast<unsigned>(__cvta_generic_to_shared(bar)))
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
        ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0),
        "r"(c1), "r"(static_cast<unsigned>(__cvta_generic_to_shared(bar)))
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n"
                 ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(bar))) : "memory");
}
// 1-D bulk copy global -> shared (16 B aligned addresses, size a multiple of 16),
// completion counted on the mbarrier's transaction bytes.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
        ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))), "l"(src), "r"(bytes),
        "r"(static_cast<unsigned>(__cvta_generic_to_shared(bar)))
        : "memory");
}

// Optional per-kernel timing (bench roofline): when enabled, selected launches
// are bracketed by CUDA events on their stream; totals are read back with
// fds_profile_read(). Disabled by default (zero overhead).
struct KernelProfile {
    bool enabled = false;
    struct Rec { cudaEvent_t a, b; double work; int kind; };
    std::vector<Rec> recs;
    std::mutex mu;  // the AFS driver fits its two models on two host threads
    void begin(cudaStream_t st, int kind, double work, cudaEvent_t& a);
    void end(cudaStream_t st, cudaEvent_t a, int kind, double work);
};
KernelProfile& profiler();
enum ProfKind { kProfLuGemm = 0, kProfLuPanel = 1, kProfLuTrsm = 2, kProfAsmFar = 3, kProfAsmNear = 4,
                kProfVfResidue = 5, kProfRatInv = 6, kProfFsm = 7, kProfChanErr = 8, kProfCount = 9 };

struct DeviceInfo {
    int device = 0;
    int sms = 148;
    size_t smem_optin = 227 * 1024;
};
const DeviceInfo& device_info();

}  // namespace fdsb


// every cudaMalloc / cudaFree of the library goes through the red-zone wrappers
#define cudaMalloc(p, n) ::fdsb::rz_malloc((p), (n))
#define cudaFree(p) ::fdsb::rz_free(p)
