// standalone panel trace: factor diagonally dominant random matrices with the GEPP panel, dump per-phase clocks
#define FDS_PANEL_TRACE
#include "../paper_1511_04355_b200/csrc/lu.cu"
#include <cstdio>
#include <vector>
#include <random>
#include <chrono>
namespace fdsb { std::atomic<int64_t> g_launches{0}; const DeviceInfo& device_info(){ static DeviceInfo d; static bool i=false; if(!i){cudaDeviceProp p; cudaGetDeviceProperties(&p,0); d.sms=p.multiProcessorCount; d.smem_optin=p.sharedMemPerBlockOptin; i=true;} return d;}
KernelProfile& profiler(){ static KernelProfile p; return p;} void KernelProfile::begin(cudaStream_t, int, double, cudaEvent_t& a){a=nullptr;} void KernelProfile::end(cudaStream_t, cudaEvent_t, int, double){}
void calu_panel_step(const LuProblem&, CaluWorkspace&, int, int, cudaStream_t){} void CaluWorkspace::release(){} void CaluWorkspace::ensure(int,int){} }
using namespace fdsb;
int main(int argc, char** argv){
  int n = atoi(argv[1]), B = atoi(argv[2]);
  LuProblem pb; pb.n=n; pb.ld=lu_ld(n); pb.plane=lu_plane(n); pb.mstride=2*pb.plane; pb.batch=B;
  std::vector<double> h(pb.mstride*B); std::mt19937_64 g(1); std::normal_distribution<double> d;
  for(auto& x: h) x=d(g) / std::sqrt((double)n);
  for(int bb=0;bb<B;bb++) for(int i=0;i<n;i++) h[bb*pb.mstride + (size_t)i*pb.ld + i] += 4.0;
  cudaMalloc(&pb.A, h.size()*8); cudaMemcpy(pb.A,h.data(),h.size()*8,cudaMemcpyHostToDevice);
  cudaMalloc(&pb.ipiv, (size_t)n*B*4); cudaMalloc(&pb.info, B*4);

  LuWorkspace ws; cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  lu_factor(pb, ws, nullptr); cudaDeviceSynchronize();
  cudaMemcpy(pb.A,h.data(),h.size()*8,cudaMemcpyHostToDevice);
  auto h0 = std::chrono::steady_clock::now();
  cudaEventRecord(a); lu_factor(pb, ws, nullptr); cudaEventRecord(b);
  auto h1 = std::chrono::steady_clock::now();
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms,a,b);
  printf("host enqueue %.2f ms\n", std::chrono::duration<double, std::milli>(h1-h0).count());

  printf("n=%d B=%d lu %.2f ms err=%s\n", n, B, ms, cudaGetErrorString(cudaGetLastError()));
  unsigned long long* tr; cudaMalloc(&tr, 8*1024*8); cudaMemset(tr,0,8*1024*8);
  cudaMemcpyToSymbol(g_trace, &tr, sizeof(tr));
  cudaMemcpy(pb.A,h.data(),h.size()*8,cudaMemcpyHostToDevice);
  lu_factor(pb, ws, nullptr); cudaDeviceSynchronize();
  std::vector<unsigned long long> t(8*1024); cudaMemcpy(t.data(),tr,t.size()*8,cudaMemcpyDeviceToHost);
  for(int c=0;c<3;c++) if(t[8*c+4]) printf("cta %d: cols %llu: argmax+stage %.0f | publish %.0f | poll+winner %.0f | update %.0f cycles/column\n", c, t[8*c+4], (double)t[8*c]/t[8*c+4], (double)t[8*c+1]/t[8*c+4], (double)t[8*c+2]/t[8*c+4], (double)t[8*c+3]/t[8*c+4]);

}
