// tcgen05.mma issue-rate probe: cycles per M128 x N x K16 bf16 SS MMA as a
// function of N, the number of independent accumulator chains, and the
// issue order (chain-major: all K of chain 0, then chain 1; interleaved:
// chains alternate every MMA). Operands are fixed shared-memory tiles (no
// TMA), so this isolates the tensor pipe + operand fetch. One CTA per SM.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

#include "../paper_2507_06608_b200/csrc/device/ptx.cuh"

using namespace nxd;

constexpr int kStages = 2;
constexpr int kChainsMax = 4;
constexpr int kA = 128 * 64 * 2;  // 16 KB: 128 rows x 64 K
constexpr int kB = 256 * 64 * 2;  // 32 KB: up to 256 rows x 64 K

__global__ void __launch_bounds__(128, 1) probe(int m, int n, int chains, int interleave, int rounds,
                                                 unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;                                  // [stage][chain] A tiles
  uint8_t* sb = smem + kStages * kChainsMax * kA;      // [stage] B tiles
  uint64_t* bar = reinterpret_cast<uint64_t*>(sb + kStages * kB);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < (kStages * (kChainsMax * kA + kB)) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < 32) tmem_alloc<512>(slot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  const uint32_t idesc = umma_idesc_bf16(m, n);
  unsigned long long t0 = 0, t1 = 0;
  if (threadIdx.x == 0) {
    t0 = clock64();
    for (int r = 0; r < rounds; ++r) {
      const int st = r % kStages;
      const uint32_t a0 = smem_u32(sa + st * kChainsMax * kA);
      const uint32_t b0 = smem_u32(sb + st * kB);
      if (interleave) {
        for (int kk = 0; kk < 4; ++kk)
          for (int c = 0; c < chains; ++c)
            umma_bf16(tmem + c * n, umma_desc_sw128(a0 + c * kA + kk * 32), umma_desc_sw128(b0 + kk * 32), idesc,
                      (r > 0 || kk > 0) ? 1u : 0u);
      } else {
        for (int c = 0; c < chains; ++c)
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16(tmem + c * n, umma_desc_sw128(a0 + c * kA + kk * 32), umma_desc_sw128(b0 + kk * 32), idesc,
                      (r > 0 || kk > 0) ? 1u : 0u);
      }
    }
    umma_commit(bar);
    mbar_wait(bar, 0);
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

int main(int argc, char** argv) {
  const int sms = argc > 1 ? atoi(argv[1]) : 1;
  const size_t smem = kStages * (kChainsMax * kA + kB) + 2048;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  unsigned long long* d;
  cudaMalloc(&d, 1024 * 8);
  unsigned long long h[1024];
  const int rounds = 256;
  for (int m : {128, 64})
  for (int n : {32, 64, 128, 160, 192, 208, 224, 240, 256})
    for (int chains : {1, 2, 4})
      for (int il : {0, 1}) {
        if (chains * n > 512 || (chains == 1 && il) || (m == 64 && (chains > 1 || n % 64))) continue;
        probe<<<sms, 128, smem>>>(m, n, chains, il, rounds, d);
        probe<<<sms, 128, smem>>>(m, n, chains, il, rounds, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("error %s\n", cudaGetErrorString(e));
          return 1;
        }
        cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
        unsigned long long mx = 0;
        for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
        const double per = static_cast<double>(mx) / (rounds * 4.0 * chains);
        const double floor = 128.0 * n / 256.0;
        printf("{\"M\": %d, \"sms\": %d, \"N\": %d, \"chains\": %d, \"interleave\": %d, \"cyc_per_mma\": %.1f, \"floor\": %.0f, "
               "\"weight_B_per_cyc\": %.1f}\n",
               m, sms, n, chains, il, per, floor, 4096.0 / per);
      }
  return 0;
}
