// Probe: green-context SM partitions on B200.
//  1. split the device's SMs into {8k} + rest for several k;
//  2. create a green context + stream per group;
//  3. launch runtime-API kernels (memory from the primary context) on those
//     streams and record which SMs the CTAs ran on (%smid);
//  4. run two partitions concurrently and time them.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <set>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)
#define DK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; pfn_err(r, &s); printf("CU %s @%d: %d %s\n", #x, __LINE__, (int)r, s); exit(1);} } while (0)

static PFN_cuGetErrorString pfn_err;

__global__ void who(int* out, long spin) {
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x == 0) out[blockIdx.x] = smid;
  long long t0 = clock64();
  while (clock64() - t0 < spin) {}
}

template <class T>
T sym(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q));
  if (!p) { printf("missing %s\n", name); exit(1); }
  return reinterpret_cast<T>(p);
}

int main() {
  CK(cudaSetDevice(0));
  CK(cudaFree(0));
  pfn_err = sym<PFN_cuGetErrorString>("cuGetErrorString");
  auto getRes = sym<PFN_cuDeviceGetDevResource>("cuDeviceGetDevResource");
  auto split = sym<PFN_cuDevSmResourceSplitByCount>("cuDevSmResourceSplitByCount");
  auto gen = sym<PFN_cuDevResourceGenerateDesc>("cuDevResourceGenerateDesc");
  auto create = sym<PFN_cuGreenCtxCreate>("cuGreenCtxCreate");
  auto mkstream = sym<PFN_cuGreenCtxStreamCreate>("cuGreenCtxStreamCreate");
  CUdevice dev;
  auto getdev = sym<PFN_cuDeviceGet>("cuDeviceGet");
  DK(getdev(&dev, 0));
  CUdevResource all;
  DK(getRes(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("device SMs: %u\n", all.sm.smCount);
  int* d_out;
  CK(cudaMalloc(&d_out, 4096 * sizeof(int)));
  for (int k : {1, 4, 9, 17}) {
    CUdevResource grp, rest;
    unsigned n = 1;
    DK(split(&grp, &n, &all, &rest, 0, 8 * k));
    printf("k=%d: group %u SMs, rest %u SMs (n=%u)\n", k, grp.sm.smCount, rest.sm.smCount, n);
    CUdevResourceDesc dg, dr;
    DK(gen(&dg, &grp, 1));
    DK(gen(&dr, &rest, 1));
    CUgreenCtx gg, gr;
    DK(create(&gg, dg, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    DK(create(&gr, dr, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream sg, sr;
    DK(mkstream(&sg, gg, CU_STREAM_NON_BLOCKING, 0));
    DK(mkstream(&sr, gr, CU_STREAM_NON_BLOCKING, 0));
    for (int which = 0; which < 2; ++which) {
      CUstream s = which ? sr : sg;
      CK(cudaMemset(d_out, 0xff, 4096 * sizeof(int)));
      who<<<1024, 128, 0, (cudaStream_t)s>>>(d_out, 2000);
      CK(cudaGetLastError());
      CK(cudaStreamSynchronize((cudaStream_t)s));
      std::vector<int> h(1024);
      CK(cudaMemcpy(h.data(), d_out, 1024 * sizeof(int), cudaMemcpyDeviceToHost));
      std::set<int> sms(h.begin(), h.end());
      printf("  %s partition: CTAs landed on %zu distinct SMs (min %d max %d)\n",
             which ? "rest " : "group", sms.size(), *sms.begin(), *sms.rbegin());
    }
    // concurrency: both partitions busy at once.
    cudaEvent_t a0, a1, b0, b1;
    CK(cudaEventCreate(&a0)); CK(cudaEventCreate(&a1)); CK(cudaEventCreate(&b0)); CK(cudaEventCreate(&b1));
    int *o1, *o2;
    CK(cudaMalloc(&o1, 100000 * 4)); CK(cudaMalloc(&o2, 100000 * 4));
    CK(cudaEventRecord(a0, (cudaStream_t)sg));
    who<<<grp.sm.smCount * 4, 128, 0, (cudaStream_t)sg>>>(o1, 2000000);
    CK(cudaEventRecord(a1, (cudaStream_t)sg));
    CK(cudaEventRecord(b0, (cudaStream_t)sr));
    who<<<rest.sm.smCount * 4, 128, 0, (cudaStream_t)sr>>>(o2, 2000000);
    CK(cudaEventRecord(b1, (cudaStream_t)sr));
    CK(cudaDeviceSynchronize());
    float ta, tb, tab;
    CK(cudaEventElapsedTime(&ta, a0, a1));
    CK(cudaEventElapsedTime(&tb, b0, b1));
    CK(cudaEventElapsedTime(&tab, a0, b1));
    printf("  concurrent: group %.3f ms, rest %.3f ms, span %.3f ms\n", ta, tb, tab);
  }
  printf("OK\n");
  return 0;
}
