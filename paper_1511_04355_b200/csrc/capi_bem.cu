// C-ABI for the BEM frequency system and the batched complex LU
// (include/fdsweep_b200.h). Replaces FrequencySystem::evaluate
// (proj/include/fdsweep/systems.hpp:34-42) with a CUDA path; there is no CPU
// fallback — every entry point fails with FDS_ECUDA if the device path fails.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>

#include "bem.cuh"
#include "capi_util.h"
#include "gmres.cuh"
#include "lu.cuh"

namespace fdsb {

std::atomic<int64_t> g_launches{0};

const DeviceInfo& device_info() {
    // per device (fds_set_device may switch the calling thread's device)
    int dev = 0;
    FDS_CUDA(cudaGetDevice(&dev));
    static std::mutex mu;
    static std::map<int, DeviceInfo> infos;
    std::lock_guard<std::mutex> lk(mu);
    auto it = infos.find(dev);
    if (it != infos.end()) return it->second;
    cudaDeviceProp p;
    FDS_CUDA(cudaGetDeviceProperties(&p, dev));
    if (p.major != 10) throw CudaError("fdsweep_b200 is built for sm_100a (B200); found sm_" +
                                       std::to_string(p.major) + std::to_string(p.minor));
    DeviceInfo info;
    info.device = dev;
    info.sms = p.multiProcessorCount;
    info.smem_optin = p.sharedMemPerBlockOptin;
    return infos.emplace(dev, info).first->second;
}

thread_local std::string g_error;

KernelProfile& profiler() {
    static KernelProfile p;
    return p;
}

void KernelProfile::begin(cudaStream_t st, int, double, cudaEvent_t& a) {
    a = nullptr;
    if (!enabled) return;
    FDS_CUDA(cudaEventCreate(&a));
    FDS_CUDA(cudaEventRecord(a, st));
}

void KernelProfile::end(cudaStream_t st, cudaEvent_t a, int kind, double work) {
    if (!enabled || !a) return;
    cudaEvent_t b;
    FDS_CUDA(cudaEventCreate(&b));
    FDS_CUDA(cudaEventRecord(b, st));
    std::lock_guard<std::mutex> lk(mu);
    recs.push_back({a, b, work, kind});
}

// A[rows[i], cols[i]] from the planar column-major matrix (verification entry point).
__global__ void gather_entries_kernel(const double* __restrict__ A, size_t plane, int ld, const int* __restrict__ rc,
                                      int count, cplx* __restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const size_t g = static_cast<size_t>(rc[count + i]) * ld + rc[i];
    out[i] = {A[g], A[plane + g]};
}

// Residual r = A u - b, partial over a slice of columns: one thread per row,
// CTA (row block, column slice), u slice staged in shared memory. Writes the
// slice's partial sums and partial |A_ij| row sums; a second kernel reduces.
constexpr int kResRows = 256, kResCols = 512;
__global__ void __launch_bounds__(kResRows) residual_partial_kernel(const double* __restrict__ A, size_t plane,
                                                                    int ld, int n, const cplx* __restrict__ u,
                                                                    cplx* __restrict__ part,
                                                                    double* __restrict__ absrow) {
    __shared__ cplx us[kResCols];
    const int i = blockIdx.x * kResRows + threadIdx.x;
    const int j0 = blockIdx.y * kResCols, j1 = min(n, j0 + kResCols);
    for (int j = j0 + threadIdx.x; j < j1; j += kResRows) us[j - j0] = u[j];
    __syncthreads();
    if (i >= n) return;
    cplx acc = {0.0, 0.0};
    double ab = 0.0;
    for (int j = j0; j < j1; ++j) {
        const size_t g = static_cast<size_t>(j) * ld + i;
        const cplx a = {A[g], A[plane + g]};
        acc = acc + a * us[j - j0];
        ab += sqrt(abs2(a));
    }
    part[static_cast<size_t>(blockIdx.y) * n + i] = acc;
    absrow[static_cast<size_t>(blockIdx.y) * n + i] = ab;
}

// One CTA: norms[0] = ||A u - b||_2, [1] = ||A||_inf, [2] = ||u||_2, [3] = ||b||_2 (fixed order).
__global__ void residual_reduce_kernel(const cplx* __restrict__ part, const double* __restrict__ absrow, int slices,
                                       int n, const cplx* __restrict__ b, const cplx* __restrict__ u,
                                       double* __restrict__ norms) {
    __shared__ double red[4][256];
    double rr = 0.0, am = 0.0, uu = 0.0, bb = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        cplx r = {-b[i].re, -b[i].im};
        double ab = 0.0;
        for (int q = 0; q < slices; ++q) {
            r = r + part[static_cast<size_t>(q) * n + i];
            ab += absrow[static_cast<size_t>(q) * n + i];
        }
        rr += abs2(r);
        am = fmax(am, ab);
        uu += abs2(u[i]);
        bb += abs2(b[i]);
    }
    red[0][threadIdx.x] = rr; red[1][threadIdx.x] = am; red[2][threadIdx.x] = uu; red[3][threadIdx.x] = bb;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            red[0][threadIdx.x] += red[0][threadIdx.x + w];
            red[1][threadIdx.x] = fmax(red[1][threadIdx.x], red[1][threadIdx.x + w]);
            red[2][threadIdx.x] += red[2][threadIdx.x + w];
            red[3][threadIdx.x] += red[3][threadIdx.x + w];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        norms[0] = sqrt(red[0][0]);
        norms[1] = red[1][0];
        norms[2] = sqrt(red[2][0]);
        norms[3] = sqrt(red[3][0]);
    }
}

__global__ void gather_channels_kernel(const cplx* __restrict__ rhs, size_t rstride, const int* __restrict__ ch,
                                       int K, int B, cplx* __restrict__ out) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= K * B) return;
    const int b = idx / K, k = idx % K;
    out[idx] = rhs[static_cast<size_t>(b) * rstride + ch[k]];
}

}  // namespace fdsb

using namespace fdsb;

struct fds_bem {
    std::mutex mu;
    cudaStream_t st = nullptr;
    BemDevice dev;
    int ne = 0, n = 0, ld = 0;
    size_t plane = 0, mstride = 0;
    int K = 0;
    int* chan = nullptr;
    int cap = 0, max_batch = 0;
    double* A = nullptr;
    int* ipiv = nullptr;
    int* info = nullptr;
    cplx* rhs = nullptr;
    cplx* svec = nullptr;
    cplx* out = nullptr;
    LuWorkspace ws;
    // solver: 0 = batched LU (default), 1 = restarted GMRES per frequency
    int solver = 0;
    GmresParams gp;
    GmresWorkspace gws;
    int gm_iters = 0;
    double gm_resid = 0.0;
    int gm_fallbacks = 0;
    cudaEvent_t ev[4] = {};
    double t_asm = 0, t_lu = 0, t_solve = 0;
    int launches = 0;
    double cum[4] = {0, 0, 0, 0};  // assembly / LU / solve ms and frequencies since create or reset

    void ensure(int B) {
        if (B <= cap) return;
        auto fr = [](void* p) { if (p) cudaFree(p); };
        fr(A); fr(ipiv); fr(info); fr(rhs); fr(svec); fr(out); fr(dev.partial); fr(dev.corr);
        FDS_CUDA(cudaMalloc(&A, mstride * B * sizeof(double)));
        FDS_CUDA(cudaMemsetAsync(A, 0, mstride * B * sizeof(double), st));  // padding stays zero
        FDS_CUDA(cudaMalloc(&ipiv, static_cast<size_t>(B) * n * sizeof(int)));
        FDS_CUDA(cudaMalloc(&info, B * sizeof(int)));
        FDS_CUDA(cudaMalloc(&rhs, static_cast<size_t>(B) * ld * sizeof(cplx)));
        FDS_CUDA(cudaMalloc(&svec, B * sizeof(cplx)));
        FDS_CUDA(cudaMalloc(&out, static_cast<size_t>(B) * K * sizeof(cplx)));
        const int nchunks = ceil_div(ne, kFarChunk);
        dev.pstride = static_cast<size_t>(nchunks) * 3 * ne;
        FDS_CUDA(cudaMalloc(&dev.partial, dev.pstride * B * sizeof(cplx)));
        dev.cstride = static_cast<size_t>(dev.npairs) * 3;
        FDS_CUDA(cudaMalloc(&dev.corr, std::max<size_t>(dev.cstride, 3) * B * sizeof(cplx)));
        cap = B;
    }

    int auto_batch = 0;  // max_batch == 0: fixed at the first evaluate (deterministic chunking)
    int chunk_limit() {
        if (max_batch > 0) return max_batch;
        if (auto_batch > 0) return auto_batch;
        size_t fr = 0, tot = 0;
        cudaMemGetInfo(&fr, &tot);
        // matrix + b-partials + the 3M update's operand planes (LuWorkspace::g3_planes) + slack
        const size_t per = mstride * sizeof(double) + dev.pstride * sizeof(cplx) +
                           static_cast<size_t>(ld) * (2 * 128 + 136) * sizeof(double) + 4096 * 64;
        const size_t budget = static_cast<size_t>(0.85 * (fr + static_cast<size_t>(cap) * per));
        auto_batch = std::max<int>(1, static_cast<int>(budget / std::max<size_t>(per, 1)));
        return auto_batch;
    }

    // Solves B frequencies already in svec_host; result (B x K) left in `out` on device.
    void run(const fds_c64* s_host, int B) {
        for (int b = 0; b < B; ++b) {
            const fds_c64 z = s_host[b];
            if (!std::isfinite(z.re) || !std::isfinite(z.im))
                throw ValidationError("bem: contour frequency must be finite");
            if (z.re == 0.0 && z.im == 0.0)
                throw ValidationError("bem: s = 0 is the pole of the Heaviside load p(s) = 1/s");
        }
        launches = 0;
        t_asm = t_lu = t_solve = 0;
        const int64_t l0 = g_launches.load();
        const auto gate = lu_device_gate();  // held until the stream synchronises below
        ensure(B);
        FDS_CUDA(cudaMemcpyAsync(svec, s_host, B * sizeof(cplx), cudaMemcpyHostToDevice, st));
        FDS_CUDA(cudaEventRecord(ev[0], st));
        bem_assemble(dev, svec, B, A, mstride, plane, ld, rhs, ld, st);
        FDS_CUDA(cudaEventRecord(ev[1], st));
        LuProblem pb;
        pb.A = A;
        pb.mstride = mstride;
        pb.plane = plane;
        pb.n = n;
        pb.ld = ld;
        pb.batch = B;
        pb.ipiv = ipiv;
        pb.info = info;
        if (solver == 1) {
            FDS_CUDA(cudaMemsetAsync(info, 0, B * sizeof(int), st));
            gm_iters = 0;
            gm_resid = 0.0;
            gm_fallbacks = 0;
            const std::vector<GmresStats> gst = gmres_solve_batch(A, mstride, plane, n, ld, B, rhs, ld, gp, gws, st);
            for (int b = 0; b < B; ++b) {
                gm_iters = std::max(gm_iters, gst[b].iterations);
                if (gst[b].converged) {
                    gm_resid = std::max(gm_resid, gst[b].rel_residual);
                    continue;
                }
                // GMRES stagnated (e.g. near an interior resonance of the cavity): this
                // frequency is solved by the LU path instead, from its saved right-hand side
                ++gm_fallbacks;
                FDS_CUDA(cudaMemcpyAsync(rhs + static_cast<size_t>(b) * ld, gws.bsave + 2 * static_cast<size_t>(b) * n,
                                         n * sizeof(cplx), cudaMemcpyDeviceToDevice, st));
                LuProblem one = pb;
                one.A = A + static_cast<size_t>(b) * mstride;
                one.batch = 1;
                one.ipiv = ipiv + static_cast<size_t>(b) * n;
                one.info = info + b;
                lu_factor(one, ws, st);
                lu_solve(one, rhs + static_cast<size_t>(b) * ld, ld, ws, st);
            }
            FDS_CUDA(cudaEventRecord(ev[2], st));
        } else {
            lu_factor(pb, ws, st);
            FDS_CUDA(cudaEventRecord(ev[2], st));
            lu_solve(pb, rhs, ld, ws, st);
        }
        FDS_LAUNCH(gather_channels_kernel, ceil_div(K * B, 256), 256, 0, st, rhs, static_cast<size_t>(ld),
                   chan, K, B, out);
        FDS_CUDA(cudaEventRecord(ev[3], st));
        std::vector<int> hinfo(B);
        FDS_CUDA(cudaMemcpyAsync(hinfo.data(), info, B * sizeof(int), cudaMemcpyDeviceToHost, st));
        FDS_CUDA(cudaStreamSynchronize(st));
        for (int b = 0; b < B; ++b)
            if (hinfo[b] != 0) throw NumericError("bem: singular system matrix (zero pivot at column " +
                                                  std::to_string(hinfo[b] - 1) + ")");
        float ms;
        FDS_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
        t_asm = ms;
        FDS_CUDA(cudaEventElapsedTime(&ms, ev[1], ev[2]));
        t_lu = ms;
        FDS_CUDA(cudaEventElapsedTime(&ms, ev[2], ev[3]));
        t_solve = ms;
        launches = static_cast<int>(g_launches.load() - l0);
        cum[0] += t_asm;
        cum[1] += t_lu;
        cum[2] += t_solve;
        cum[3] += B;
    }
};

extern "C" {

const char* fds_last_error(void) { return g_error.c_str(); }
const char* fds_version(void) { return "fdsweep_b200 0.1.0 sm_100a"; }
int64_t fds_kernel_launches(void) { return g_launches.load(); }

int fds_profile_enable(int on) {
    return fds_guard([&] {
        auto& p = profiler();
        std::lock_guard<std::mutex> lk(p.mu);
        for (auto& r : p.recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
        p.recs.clear();
        p.enabled = on != 0;
    });
}

int fds_debug_redzone_check(int* enabled, long long* overwritten_bytes, long long* checks, long long* live) {
    return fds_guard([&] {
        const bool on = RedzoneRegistry::enabled();
        long long bad = 0, chk = 0, nlive = 0;
        if (on) {
            FDS_CUDA(cudaDeviceSynchronize());
            auto& rz = RedzoneRegistry::get();
            std::lock_guard<std::mutex> lk(rz.mu);
            long long now = 0;
            for (auto& kv : rz.live) now += rz.check_one(kv.first, kv.second);
            bad = rz.violations + now;  // live zones are re-counted on every call, freed ones once
            chk = rz.checked;
            nlive = static_cast<long long>(rz.live.size());
        }
        if (enabled) *enabled = on ? 1 : 0;
        if (overwritten_bytes) *overwritten_bytes = bad;
        if (checks) *checks = chk;
        if (live) *live = nlive;
    });
}

int fds_profile_read(int kind, int* count, double* total_ms, double* total_work) {
    return fds_guard([&] {
        auto& p = profiler();
        std::lock_guard<std::mutex> lk(p.mu);
        int c = 0;
        double ms = 0, w = 0;
        for (auto& r : p.recs) {
            if (r.kind != kind) continue;
            FDS_CUDA(cudaEventSynchronize(r.b));
            float t;
            FDS_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
            ++c;
            ms += t;
            w += r.work;
        }
        if (count) *count = c;
        if (total_ms) *total_ms = ms;
        if (total_work) *total_work = w;
    });
}

int fds_set_device(int device) {
    return fds_guard([&] { FDS_CUDA(cudaSetDevice(device)); });
}

int fds_bem_create(const fds_bem_desc* d, fds_bem** out) {
    return fds_guard([&] {
        if (!d || !out) throw ValidationError("fds_bem_create: null argument");
        if (d->n_elements < 1 || d->n_vertices < 3 || !d->vertices || !d->triangles || !d->traction)
            throw ValidationError("fds_bem_create: empty mesh or load");
        if (d->n_channels > 0 && !d->channels) throw ValidationError("fds_bem_create: null channel list");
        if (d->max_batch < 0) throw ValidationError("fds_bem_create: max_batch must be >= 0");
        // host-side validation first: bad input is reported as such, GPU or not
        const int n = 3 * d->n_elements;
        const BemParams params = make_bem_params(d->shear_modulus, d->poisson_ratio, d->density);
        for (int i = 0; i < 3 * d->n_vertices; ++i)
            if (!std::isfinite(d->vertices[i])) throw ValidationError("fds_bem_create: non-finite vertex coordinate");
        for (int i = 0; i < n; ++i)
            if (!std::isfinite(d->traction[i])) throw ValidationError("fds_bem_create: non-finite traction");
        std::vector<double> geo;
        std::vector<int> pairs, ptr;
        bem_build_geometry(d->vertices, d->n_vertices, d->triangles, d->n_elements, geo, pairs, ptr);
        std::vector<int> chans;
        if (d->n_channels > 0) {
            for (int i = 0; i < d->n_channels; ++i) {
                if (d->channels[i] < 0 || d->channels[i] >= n)
                    throw ValidationError("fds_bem_create: channel DOF out of range");
                chans.push_back(d->channels[i]);
            }
        } else {
            for (int i = 0; i < n; ++i) chans.push_back(i);
        }
        device_info();
        auto* h = new fds_bem;
        try {
            h->ne = d->n_elements;
            h->n = n;
            h->ld = lu_ld(h->n);
            h->plane = lu_plane(h->n);
            h->mstride = 2 * h->plane;
            h->max_batch = d->max_batch;
            h->dev.ne = h->ne;
            h->dev.params = params;
            h->dev.npairs = static_cast<int>(pairs.size() / 3);
            h->K = static_cast<int>(chans.size());
            FDS_CUDA(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking));
            for (auto& e : h->ev) FDS_CUDA(cudaEventCreate(&e));
            FDS_CUDA(cudaMalloc(&h->dev.geo, geo.size() * sizeof(double)));
            FDS_CUDA(cudaMalloc(&h->dev.trac, 3 * h->ne * sizeof(double)));
            FDS_CUDA(cudaMalloc(&h->dev.pairs, std::max<size_t>(pairs.size(), 3) * sizeof(int)));
            FDS_CUDA(cudaMalloc(&h->dev.near_ptr, ptr.size() * sizeof(int)));
            FDS_CUDA(cudaMalloc(&h->chan, chans.size() * sizeof(int)));
            FDS_CUDA(cudaMemcpy(h->dev.geo, geo.data(), geo.size() * sizeof(double), cudaMemcpyHostToDevice));
            FDS_CUDA(cudaMemcpy(h->dev.trac, d->traction, 3 * h->ne * sizeof(double), cudaMemcpyHostToDevice));
            FDS_CUDA(cudaMemcpy(h->dev.pairs, pairs.data(), pairs.size() * sizeof(int), cudaMemcpyHostToDevice));
            FDS_CUDA(cudaMemcpy(h->dev.near_ptr, ptr.data(), ptr.size() * sizeof(int), cudaMemcpyHostToDevice));
            // near-kernel processing order: costliest pairs first (self polar rule,
            // then deepest subdivision), so warps sharing a CTA carry equal work
            {
                const int np = h->dev.npairs;
                std::vector<int> order(np);
                for (int q = 0; q < np; ++q) order[q] = q;
                auto cost = [&](int q) { const int lv = pairs[3 * q + 2]; return lv < 0 ? 1 << 20 : 1 << (2 * lv); };
                std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost(a) > cost(b); });
                FDS_CUDA(cudaMalloc(&h->dev.order, std::max(np, 1) * sizeof(int)));
                FDS_CUDA(cudaMemcpy(h->dev.order, order.data(), np * sizeof(int), cudaMemcpyHostToDevice));
            }
            FDS_CUDA(cudaMemcpy(h->chan, chans.data(), chans.size() * sizeof(int), cudaMemcpyHostToDevice));
        } catch (...) {
            fds_bem_destroy(h);
            throw;
        }
        *out = h;
    });
}

int fds_bem_destroy(fds_bem* h) {
    if (!h) return FDS_OK;
    auto fr = [](void* p) { if (p) cudaFree(p); };
    if (h->st) cudaStreamSynchronize(h->st);
    fr(h->A); fr(h->ipiv); fr(h->info); fr(h->rhs); fr(h->svec); fr(h->out); fr(h->chan);
    fr(h->dev.geo); fr(h->dev.trac); fr(h->dev.pairs); fr(h->dev.order); fr(h->dev.near_ptr); fr(h->dev.partial); fr(h->dev.corr);
    h->ws.release();
    for (auto e : h->ev) if (e) cudaEventDestroy(e);
    if (h->st) cudaStreamDestroy(h->st);
    delete h;
    return FDS_OK;
}

int fds_bem_channels(const fds_bem* h) { return h ? h->K : -1; }
int fds_bem_unknowns(const fds_bem* h) { return h ? h->n : -1; }

int fds_bem_evaluate_batch(fds_bem* h, const fds_c64* s, int B, fds_c64* out) {
    return fds_guard([&] {
        if (!h || (B > 0 && (!s || !out))) throw ValidationError("fds_bem_evaluate_batch: null argument");
        if (B < 0) throw ValidationError("fds_bem_evaluate_batch: negative batch");
        for (int b = 0; b < B; ++b)
            if (s[b].re == 0.0 && s[b].im == 0.0)
                throw ValidationError("bem: s = 0 is the pole of the Heaviside load");
        std::lock_guard<std::mutex> lk(h->mu);
        const int lim = h->chunk_limit();
        double ta = 0, tl = 0, ts = 0;
        int nl = 0;
        for (int b0 = 0; b0 < B; b0 += lim) {
            const int nb = std::min(lim, B - b0);
            h->run(s + b0, nb);
            FDS_CUDA(cudaMemcpyAsync(out + static_cast<size_t>(b0) * h->K, h->out,
                                     static_cast<size_t>(nb) * h->K * sizeof(cplx), cudaMemcpyDeviceToHost, h->st));
            FDS_CUDA(cudaStreamSynchronize(h->st));
            ta += h->t_asm;
            tl += h->t_lu;
            ts += h->t_solve;
            nl += h->launches;
        }
        h->t_asm = ta;
        h->t_lu = tl;
        h->t_solve = ts;
        h->launches = nl;
    });
}

int fds_bem_evaluate(fds_bem* h, fds_c64 s, fds_c64* out) { return fds_bem_evaluate_batch(h, &s, 1, out); }

int fds_bem_evaluate_batch_device(fds_bem* h, const fds_c64* s, int B, const fds_c64** dev_out) {
    return fds_guard([&] {
        if (!h || !s || !dev_out || B < 1) throw ValidationError("fds_bem_evaluate_batch_device: bad argument");
        std::lock_guard<std::mutex> lk(h->mu);
        if (h->max_batch > 0 && B > h->max_batch)
            throw ValidationError("fds_bem_evaluate_batch_device: B exceeds max_batch");
        h->run(s, B);
        *dev_out = reinterpret_cast<const fds_c64*>(h->out);
    });
}

int fds_bem_assemble_host(fds_bem* h, fds_c64 s, fds_c64* A, fds_c64* b) {
    return fds_guard([&] {
        std::lock_guard<std::mutex> lk(h->mu);
        h->ensure(1);
        FDS_CUDA(cudaMemcpyAsync(h->svec, &s, sizeof(cplx), cudaMemcpyHostToDevice, h->st));
        bem_assemble(h->dev, h->svec, 1, h->A, h->mstride, h->plane, h->ld, h->rhs, h->ld, h->st);
        std::vector<double> re(h->plane), im(h->plane);
        FDS_CUDA(cudaMemcpyAsync(re.data(), h->A, h->plane * sizeof(double), cudaMemcpyDeviceToHost, h->st));
        FDS_CUDA(cudaMemcpyAsync(im.data(), h->A + h->plane, h->plane * sizeof(double), cudaMemcpyDeviceToHost, h->st));
        FDS_CUDA(cudaMemcpyAsync(b, h->rhs, h->n * sizeof(cplx), cudaMemcpyDeviceToHost, h->st));
        FDS_CUDA(cudaStreamSynchronize(h->st));
        for (int j = 0; j < h->n; ++j)
            for (int i = 0; i < h->n; ++i) {
                const size_t gi = static_cast<size_t>(j) * h->ld + i;
                A[static_cast<size_t>(j) * h->n + i] = {re[gi], im[gi]};
            }
    });
}

int fds_bem_assemble_entries(fds_bem* h, fds_c64 s, int count, const int* rows, const int* cols, fds_c64* out,
                             fds_c64* b) {
    return fds_guard([&] {
        if (!h || count < 0 || (count > 0 && (!rows || !cols || !out)))
            throw ValidationError("fds_bem_assemble_entries: bad argument");
        for (int i = 0; i < count; ++i)
            if (rows[i] < 0 || rows[i] >= h->n || cols[i] < 0 || cols[i] >= h->n)
                throw ValidationError("fds_bem_assemble_entries: index out of range");
        std::lock_guard<std::mutex> lk(h->mu);
        h->ensure(1);
        FDS_CUDA(cudaMemcpyAsync(h->svec, &s, sizeof(cplx), cudaMemcpyHostToDevice, h->st));
        bem_assemble(h->dev, h->svec, 1, h->A, h->mstride, h->plane, h->ld, h->rhs, h->ld, h->st);
        if (count > 0) {
            int* drc = nullptr;
            cplx* dout = nullptr;
            FDS_CUDA(cudaMallocAsync(&drc, 2 * static_cast<size_t>(count) * sizeof(int), h->st));
            FDS_CUDA(cudaMallocAsync(&dout, static_cast<size_t>(count) * sizeof(cplx), h->st));
            FDS_CUDA(cudaMemcpyAsync(drc, rows, count * sizeof(int), cudaMemcpyHostToDevice, h->st));
            FDS_CUDA(cudaMemcpyAsync(drc + count, cols, count * sizeof(int), cudaMemcpyHostToDevice, h->st));
            FDS_LAUNCH(gather_entries_kernel, ceil_div(count, 256), 256, 0, h->st, h->A, h->plane, h->ld, drc, count,
                       dout);
            FDS_CUDA(cudaMemcpyAsync(out, dout, count * sizeof(cplx), cudaMemcpyDeviceToHost, h->st));
            FDS_CUDA(cudaFreeAsync(drc, h->st));
            FDS_CUDA(cudaFreeAsync(dout, h->st));
        }
        if (b) FDS_CUDA(cudaMemcpyAsync(b, h->rhs, h->n * sizeof(cplx), cudaMemcpyDeviceToHost, h->st));
        FDS_CUDA(cudaStreamSynchronize(h->st));
    });
}

int fds_bem_residual(fds_bem* h, fds_c64 s, const fds_c64* u, double* norms) {
    return fds_guard([&] {
        if (!h || !u || !norms) throw ValidationError("fds_bem_residual: null argument");
        std::lock_guard<std::mutex> lk(h->mu);
        h->ensure(1);
        FDS_CUDA(cudaMemcpyAsync(h->svec, &s, sizeof(cplx), cudaMemcpyHostToDevice, h->st));
        bem_assemble(h->dev, h->svec, 1, h->A, h->mstride, h->plane, h->ld, h->rhs, h->ld, h->st);
        const int n = h->n, slices = ceil_div(n, kResCols);
        cplx *du = nullptr, *part = nullptr;
        double *absrow = nullptr, *dn = nullptr;
        FDS_CUDA(cudaMallocAsync(&du, n * sizeof(cplx), h->st));
        FDS_CUDA(cudaMallocAsync(&part, static_cast<size_t>(slices) * n * sizeof(cplx), h->st));
        FDS_CUDA(cudaMallocAsync(&absrow, static_cast<size_t>(slices) * n * sizeof(double), h->st));
        FDS_CUDA(cudaMallocAsync(&dn, 4 * sizeof(double), h->st));
        FDS_CUDA(cudaMemcpyAsync(du, u, n * sizeof(cplx), cudaMemcpyHostToDevice, h->st));
        FDS_LAUNCH(residual_partial_kernel, dim3(ceil_div(n, kResRows), slices), kResRows, 0, h->st, h->A, h->plane,
                   h->ld, n, du, part, absrow);
        FDS_LAUNCH(residual_reduce_kernel, 1, 256, 0, h->st, part, absrow, slices, n, h->rhs, du, dn);
        FDS_CUDA(cudaMemcpyAsync(norms, dn, 4 * sizeof(double), cudaMemcpyDeviceToHost, h->st));
        FDS_CUDA(cudaFreeAsync(du, h->st));
        FDS_CUDA(cudaFreeAsync(part, h->st));
        FDS_CUDA(cudaFreeAsync(absrow, h->st));
        FDS_CUDA(cudaFreeAsync(dn, h->st));
        FDS_CUDA(cudaStreamSynchronize(h->st));
    });
}

int fds_bem_last_timing(const fds_bem* h, double* a, double* l, double* s, int* launches) {
    if (!h) return FDS_EVALIDATION;
    if (a) *a = h->t_asm;
    if (l) *l = h->t_lu;
    if (s) *s = h->t_solve;
    if (launches) *launches = h->launches;
    return FDS_OK;
}

int fds_bem_cumulative_timing(fds_bem* h, double* out, int reset) {
    return fds_guard([&] {
        if (!h || !out) throw ValidationError("fds_bem_cumulative_timing: null argument");
        std::lock_guard<std::mutex> lk(h->mu);
        for (int i = 0; i < 4; ++i) out[i] = h->cum[i];
        if (reset)
            for (double& c : h->cum) c = 0.0;
    });
}

int fds_bem_set_solver(fds_bem* h, int kind, double tol, int restart, int max_iter) {
    return fds_guard([&] {
        if (!h) throw ValidationError("fds_bem_set_solver: null handle");
        if (kind != 0 && kind != 1) throw ValidationError("fds_bem_set_solver: kind must be 0 (LU) or 1 (GMRES)");
        if (kind == 1 && (!(tol > 0.0) || restart < 1 || max_iter < 1))
            throw ValidationError("fds_bem_set_solver: GMRES needs tol > 0, restart >= 1, max_iter >= 1");
        std::lock_guard<std::mutex> lk(h->mu);
        h->solver = kind;
        if (kind == 1) {
            h->gp.tol = tol;
            h->gp.restart = restart;
            h->gp.max_iter = max_iter;
        }
    });
}

int fds_bem_last_gmres(const fds_bem* h, int* iterations, double* rel_residual, int* lu_fallbacks) {
    return fds_guard([&] {
        if (!h) throw ValidationError("fds_bem_last_gmres: null handle");
        if (iterations) *iterations = h->gm_iters;
        if (rel_residual) *rel_residual = h->gm_resid;
        if (lu_fallbacks) *lu_fallbacks = h->gm_fallbacks;
    });
}

// ------------------------------------------------------------------ batched zgesv
int fds_zgesv_batch(int n, int B, const fds_c64* A, const fds_c64* rhs, fds_c64* x) {
    return fds_guard([&] {
        if (n < 1 || B < 1 || !A || !rhs || !x) throw ValidationError("fds_zgesv_batch: bad argument");
        device_info();
        const int ld = lu_ld(n);
        const size_t plane = lu_plane(n), mstride = 2 * plane;
        std::vector<double> h(mstride * B, 0.0);
        for (int b = 0; b < B; ++b)
            for (int j = 0; j < n; ++j)
                for (int i = 0; i < n; ++i) {
                    const fds_c64 v = A[static_cast<size_t>(b) * n * n + static_cast<size_t>(j) * n + i];
                    h[b * mstride + static_cast<size_t>(j) * ld + i] = v.re;
                    h[b * mstride + plane + static_cast<size_t>(j) * ld + i] = v.im;
                }
        DeviceBuffer<double> dA(mstride * B);
        DeviceBuffer<int> dp(static_cast<size_t>(n) * B), di(B);
        DeviceBuffer<cplx> dr(static_cast<size_t>(ld) * B);
        cudaStream_t st = nullptr;
        FDS_CUDA(cudaMemcpy(dA.p, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice));
        for (int b = 0; b < B; ++b)
            FDS_CUDA(cudaMemcpy(dr.p + static_cast<size_t>(b) * ld, rhs + static_cast<size_t>(b) * n,
                                n * sizeof(cplx), cudaMemcpyHostToDevice));
        LuProblem pb;
        pb.A = dA.p;
        pb.mstride = mstride;
        pb.plane = plane;
        pb.n = n;
        pb.ld = ld;
        pb.batch = B;
        pb.ipiv = dp.p;
        pb.info = di.p;
        LuWorkspace ws;
        {
            const auto gate = lu_device_gate();
            lu_factor(pb, ws, st);
            lu_solve(pb, dr.p, ld, ws, st);
            FDS_CUDA(cudaStreamSynchronize(st));
        }
        ws.release();
        std::vector<int> info(B);
        FDS_CUDA(cudaMemcpy(info.data(), di.p, B * sizeof(int), cudaMemcpyDeviceToHost));
        for (int b = 0; b < B; ++b)
            if (info[b]) throw NumericError("zgesv: singular matrix");
        for (int b = 0; b < B; ++b)
            FDS_CUDA(cudaMemcpy(x + static_cast<size_t>(b) * n, dr.p + static_cast<size_t>(b) * ld, n * sizeof(cplx),
                                cudaMemcpyDeviceToHost));
    });
}

int fds_lu_factor_device(int n, int B, double* A_planar, int* ipiv, int* info, double* ms) {
    return fds_guard([&] {
        LuProblem pb;
        pb.A = A_planar;
        pb.plane = lu_plane(n);
        pb.mstride = 2 * pb.plane;
        pb.n = n;
        pb.ld = lu_ld(n);
        pb.batch = B;
        pb.ipiv = ipiv;
        pb.info = info;
        static thread_local LuWorkspace ws;
        cudaEvent_t e0, e1;
        FDS_CUDA(cudaEventCreate(&e0));
        FDS_CUDA(cudaEventCreate(&e1));
        const auto gate = lu_device_gate();
        FDS_CUDA(cudaEventRecord(e0, nullptr));
        lu_factor(pb, ws, nullptr);
        FDS_CUDA(cudaEventRecord(e1, nullptr));
        FDS_CUDA(cudaEventSynchronize(e1));
        float t;
        FDS_CUDA(cudaEventElapsedTime(&t, e0, e1));
        if (ms) *ms = t;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    });
}

}  // extern "C"
