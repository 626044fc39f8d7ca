// Probe: can weights-as-A in TMEM (TS-mode tcgen05.mma) beat the SS-mode
// decode ceiling? Times, per K16 step of a 128-row A tile, (a) tcgen05.cp
// smem -> TMEM of the A slice (128 x 256b = 4 KB), (b) a TS-mode M128 x N x K16
// MMA with A already in TMEM, (c) both back to back (the streaming pattern).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

#include "../paper_2507_06608_b200/csrc/device/ptx.cuh"

using namespace nxd;

__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc));
}
__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(acc));
}

__global__ void __launch_bounds__(128, 1) probe(int mode, int n, int steps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 96 * 1024);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x)
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
  const uint32_t idesc = umma_idesc_bf16(128, n);
  const uint32_t a_base = smem_u32(smem);             // 64 KB of A tiles (4 x 16 KB, SW128)
  const uint32_t b_base = smem_u32(smem + 64 * 1024); // B tile (n rows x 64 K)
  if (threadIdx.x == 0) {
    const unsigned long long t0 = clock64();
    for (int s = 0; s < steps; ++s) {
      const int kk = s & 3, tile = (s >> 2) & 3;
      const uint32_t a_cols = tmem + 256 + (s & 31) * 8;  // A ring: 32 K16 slices x 8 columns
      const uint64_t a_desc = umma_desc_sw128(a_base + tile * 16384 + kk * 32);
      if (mode != 1) tmem_cp_128x256b(a_cols, a_desc);
      if (mode != 0) umma_ts(tmem, mode == 1 ? tmem + 256 : a_cols, umma_desc_sw128(b_base + kk * 32), idesc, s > 0);
    }
    umma_commit(bar);
    mbar_wait(bar, 0);
    out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

int main() {
  const size_t smem = 97 * 1024 + 2048;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  unsigned long long* d;
  cudaMalloc(&d, 8 * 148);
  unsigned long long h[148];
  const int steps = 1024;
  const char* names[3] = {"cp_only", "mma_ts_only", "cp_then_mma_ts"};
  for (int mode = 0; mode < 3; ++mode)
    for (int n : {32, 64, 128, 256}) {
      if (mode == 0 && n != 64) continue;
      probe<<<1, 128, smem>>>(mode, n, steps, d);
      probe<<<1, 128, smem>>>(mode, n, steps, d);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("{\"mode\": \"%s\", \"N\": %d, \"error\": \"%s\"}\n", names[mode], n, cudaGetErrorString(e));
        return 1;
      }
      cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
      const double per = static_cast<double>(h[0]) / steps;
      printf("{\"mode\": \"%s\", \"N\": %d, \"cyc_per_k16_step\": %.1f, \"weight_B_per_cyc\": %.1f}\n", names[mode], n,
             per, 4096.0 / per);
    }
  return 0;
}
