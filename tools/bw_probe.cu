// Streaming-bandwidth probe: how fast can one CTA per SM pull bytes from
// HBM into shared memory on B200 with (a) 2D TMA boxes (64 x 128 rows,
// 128B swizzle: the GEMM's weight tile) vs (b) 1D cp.async.bulk copies of
// contiguous chunks (pre-packed weight tiles), for several stage counts and
// SM counts. Consumer = an arrive on the empty barrier (no math).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 10000000;\n@!p bra W_%=;\n}" :: "r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma2d(const CUtensorMap* m, uint64_t* bar, void* dst, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
               :: "r"(su32(dst)), "l"((uint64_t)m), "r"(su32(bar)), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void bulk1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(su32(dst)), "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}

// mode 0: 2D TMA 64x128 boxes; mode 1: 1D bulk chunk bytes
__global__ void stream_kernel(const __grid_constant__ CUtensorMap map, const char* base, int mode, int stages,
                              int chunk, long long total_chunks, int rows) {
  extern __shared__ __align__(1024) char smem[];
  uint64_t* full = (uint64_t*)(smem + stages * chunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  long long my0 = total_chunks * blockIdx.x / gridDim.x, my1 = total_chunks * (blockIdx.x + 1) / gridDim.x;
  int stage = 0; uint32_t phase = 0;
  long long issued = my0, done = my0;
  // prime
  for (int s = 0; s < stages && issued < my1; ++s, ++issued) {
    mbar_expect(&full[s], chunk);
    if (mode == 0) { long long kb = issued % 64, mb = issued / 64; tma2d(&map, &full[s], smem + s * chunk, (int)kb * 64, (int)(mb * 128) % rows); }
    else if (mode == 1) bulk1d(smem + s * chunk, base + (issued * chunk) % (1ll << 33), chunk, &full[s]);
    else for (int j = 0; j < chunk / 4096; ++j)  // mode 2: 4 KB pieces 32 KB apart (KV pages)
      bulk1d(smem + s * chunk + j * 4096, base + ((issued * (chunk / 4096) + j) * 32768ll) % (1ll << 33), 4096, &full[s]);
  }
  while (done < my1) {
    mbar_wait(&full[stage], phase);
    ++done;
    if (issued < my1) {
      mbar_expect(&full[stage], chunk);
      if (mode == 0) { long long kb = issued % 64, mb = issued / 64; tma2d(&map, &full[stage], smem + stage * chunk, (int)kb * 64, (int)(mb * 128) % rows); }
      else if (mode == 1) bulk1d(smem + stage * chunk, base + (issued * chunk) % (1ll << 33), chunk, &full[stage]);
      else for (int j = 0; j < chunk / 4096; ++j)
        bulk1d(smem + stage * chunk + j * 4096, base + ((issued * (chunk / 4096) + j) * 32768ll) % (1ll << 33), 4096, &full[stage]);
      ++issued;
    }
    if (++stage == stages) { stage = 0; phase ^= 1; }
  }
}

int main() {
  CK(cudaSetDevice(0));
  const size_t bytes = 8ull << 30;
  char* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 1, bytes));
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  auto encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  const int K = 4096; const int rows = (int)(bytes / (K * 2));
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows}; cuuint64_t str[1] = {(cuuint64_t)K * 2};
  cuuint32_t box[2] = {64, 128}; cuuint32_t es[2] = {1, 1};
  if (encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("encode fail\n"); return 1; }
  CK(cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  // BW_GREEN=contig|spread: launch into a green-context partition of
  // BW_GREEN_SMS SMs (the first 8k SMs of a split, or k of the 8-SM groups
  // spaced evenly over the split) instead of a plain stream
  cudaStream_t gstream = 0;
  const char* gmode = getenv("BW_GREEN");
  if (gmode) {
    auto sym = [](const char* name) {
      void* p = nullptr; cudaDriverEntryPointQueryResult qq;
      CK(cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &qq));
      return p;
    };
    auto get_res = (PFN_cuDeviceGetDevResource)sym("cuDeviceGetDevResource");
    auto split = (PFN_cuDevSmResourceSplitByCount)sym("cuDevSmResourceSplitByCount");
    auto gen = (PFN_cuDevResourceGenerateDesc)sym("cuDevResourceGenerateDesc");
    auto create = (PFN_cuGreenCtxCreate)sym("cuGreenCtxCreate");
    auto mkstream = (PFN_cuGreenCtxStreamCreate)sym("cuGreenCtxStreamCreate");
    CUdevice dev = 0;
    CUdevResource all; get_res(dev, &all, CU_DEV_RESOURCE_TYPE_SM);
    const int want = getenv("BW_GREEN_SMS") ? atoi(getenv("BW_GREEN_SMS")) : 32;
    std::vector<CUdevResource> pick;
    if (gmode[0] == 's') {
      unsigned n = all.sm.smCount / 8; std::vector<CUdevResource> grp(n); CUdevResource rest;
      if (split(grp.data(), &n, &all, &rest, 0, 8) != CUDA_SUCCESS) { printf("split fail\n"); return 1; }
      const unsigned k = want / 8;
      for (unsigned i = 0; i < k; ++i) pick.push_back(grp[(2 * i + 1) * n / (2 * k)]);
    } else {
      unsigned n = 1; CUdevResource grp, rest;
      if (split(&grp, &n, &all, &rest, 0, want) != CUDA_SUCCESS) { printf("split fail\n"); return 1; }
      pick.push_back(grp);
    }
    CUdevResourceDesc d; CUgreenCtx g; CUstream st;
    if (gen(&d, pick.data(), (unsigned)pick.size()) != CUDA_SUCCESS || create(&g, d, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
        mkstream(&st, g, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS) { printf("green ctx fail\n"); return 1; }
    gstream = (cudaStream_t)st;
  }
  struct Cfg { int mode, chunk, stages; };
  std::vector<Cfg> cfgs = {{1, 16384, 12}, {1, 4096, 48}, {1, 4096, 12}, {2, 16384, 12}, {2, 16384, 6}, {1, 32768, 6}};
  std::vector<int> sm_list = {16, 48, 148};
  // BW_CFGS="mode:chunk:stages,..." and BW_SMS="32,148" override the sweep
  if (const char* e = getenv("BW_CFGS")) {
    cfgs.clear();
    for (const char* q = e; *q;) {
      Cfg c;
      int n = 0;
      if (sscanf(q, "%d:%d:%d%n", &c.mode, &c.chunk, &c.stages, &n) != 3) break;
      cfgs.push_back(c);
      q += n;
      if (*q == ',') ++q;
    }
  }
  if (const char* e = getenv("BW_SMS")) {
    sm_list.clear();
    for (const char* q = e; *q;) {
      int v = 0, n = 0;
      if (sscanf(q, "%d%n", &v, &n) != 1) break;
      sm_list.push_back(v);
      q += n;
      if (*q == ',') ++q;
    }
  }
  const long long total_bytes = 2ll << 30;
  for (auto c : cfgs) {
    for (int sms : sm_list) {
      long long chunks = total_bytes / c.chunk;
      if (sms <= 16) chunks /= 8;
      int smem = c.stages * c.chunk + 1024;
      stream_kernel<<<sms, 32, smem, gstream>>>(map, buf, c.mode, c.stages, c.chunk, chunks, rows);
      CK(cudaEventRecord(e0, gstream));
      for (int i = 0; i < 3; ++i) stream_kernel<<<sms, 32, smem, gstream>>>(map, buf, c.mode, c.stages, c.chunk, chunks, rows);
      CK(cudaEventRecord(e1, gstream)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
      double gbs = 3.0 * chunks * c.chunk / (ms * 1e-3) / 1e9;
      printf("{\"mode\": \"%s\", \"green\": \"%s\", \"chunk\": %d, \"stages\": %d, \"sms\": %d, \"GBps\": %.0f, \"per_sm\": %.1f}\n",
             c.mode == 2 ? "bulk4k_strided" : c.mode ? "bulk1d" : "tma2d", gmode ? gmode : "none", c.chunk, c.stages, sms, gbs,
             gbs / sms);
    }
  }
  return 0;
}
