// Decode-shaped projection GEMM (tokens <= 128) on tcgen05, weights as the
// wide operand.
//
//   D[t, f] = sum_k X[t, k] * W[f, k]      (A = X: M = 128 token rows,
//                                           B = W: N = 256 weight rows)
//
// Why not the prefill kernel's swap-AB tiling (weights as M = 128, tokens
// as N = 32..64)? On sm_100a an SS-mode M128 x N x K16 MMA costs ~100
// cycles for every N <= 128 and only reaches the tensor floor
// (max(M,128) * N / 256 cycles) at N = 256 (tools/mma_probe.cu,
// profiles/r01s2_mma_probe.md). With 128 weight rows per MMA that caps the
// weight stream at ~40 B/cycle/SM; with 256 weight rows per MMA at the
// floor it is 8 KB / 128 cycles = 64 B/cycle/SM (~126 GB/s per SM at
// 1.965 GHz) -- the per-SM ceiling of a bf16 tcgen05 decode GEMM, since the
// token side cannot go below M = 128.
//
// Work unit = one 256-row weight block (an aligned pair of packed 128 x 64
// tiles: one contiguous 32 KB cp.async.bulk per k-block) x all tokens.
// Stream-K over (block, k-block) iterations keeps every CTA streaming the
// same number of weight bytes; the cross-CTA fold is deferred to the
// consumer kernel (GemmFold planes, see device.cuh), so no CTA ever waits
// for another. Warp roles as in gemm_tc.cu: producer, MMA issuer, 4
// epilogue warps (TMEM lane quarter = token rows 32q..32q+31; a thread
// writes 32 consecutive features of its token straight from registers).
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "device.cuh"
#include "ptx.cuh"

namespace nxd {

namespace {

constexpr int kRowsBlk = 256;                    // weight rows per MMA (N)
constexpr int kKB = 64;                          // K per stage (one 128B swizzle row)
constexpr int kWBytes = kRowsBlk * kKB * 2;      // 32 KB
constexpr int kXBytes = 128 * kKB * 2;           // 16 KB (A tile, M = 128 rows)
constexpr int kStagesMax = 6;
constexpr int kThreads = 192;
constexpr int kEpiThreads = 128;
// Ring of `stages` stages of [W 32 KB | X box_rows x 128 B]. The MMA's A
// operand is always a 128-row tile (16 KB); rows past the box overhang into
// the next stage (or the slack after the ring) -- those TMEM lanes are never
// read, so a small X box buys ring depth (weight bytes in flight per SM,
// the bound of a partition-sized grid) instead of idle smem.
constexpr int kSmemBudget = 227 * 1024 - 1024 - 256;

struct DecParams {
  int rows, tokens, num_kb, n_tiles;  // n_tiles = 256-row blocks
  int streamk;
  long long total;                    // n_tiles * num_kb
  int mode;                           // kEpiF32 (direct) or kEpiPartial (fold planes)
  float* out;                         // kEpiF32: [tokens][ldo]; fold: planes [piece][tokens][rows]
  int ldo;
  uint32_t x_bytes;                   // bytes of one X box (box rows x 128 B)
  int stages;
  uint32_t stage_bytes;               // 32 KB + x_bytes rounded up to 1 KB
  int prefetch;                       // L2 prefetch distance in k-blocks past the ring (stream-K)
};

struct DecWork {
  int tile, kb0, kb1, piece;
};

struct DecIter {
  const DecParams& p;
  long long it = 0, end = 0;
  int u = 0;
  __device__ explicit DecIter(const DecParams& pp) : p(pp) {
    if (p.streamk) {
      it = p.total * blockIdx.x / gridDim.x;
      end = p.total * (blockIdx.x + 1) / gridDim.x;
    } else {
      u = blockIdx.x;
    }
  }
  __device__ bool next(DecWork& w) {
    if (p.streamk) {
      if (it >= end) return false;
      w.tile = static_cast<int>(it / p.num_kb);
      w.kb0 = static_cast<int>(it % p.num_kb);
      w.kb1 = static_cast<int>(min(static_cast<long long>(p.num_kb), w.kb0 + (end - it)));
      const long long it0 = static_cast<long long>(w.tile) * p.num_kb;
      w.piece = static_cast<int>(blockIdx.x) - static_cast<int>(((it0 + 1) * gridDim.x - 1) / p.total);
      it += w.kb1 - w.kb0;
      return true;
    }
    if (u >= p.n_tiles) return false;
    w.tile = u;
    w.kb0 = 0;
    w.kb1 = p.num_kb;
    w.piece = 0;
    u += gridDim.x;
    return true;
  }
};

__global__ void __launch_bounds__(kThreads, 1)
    gemm_decode_kernel(const __nv_bfloat16* __restrict__ wpack, const __grid_constant__ CUtensorMap tx,
                       DecParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int kStages = p.stages;
  const uint32_t kStage = p.stage_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStage + (kXBytes - p.x_bytes));
  uint64_t* empty = full + kStagesMax;
  uint64_t* tfull = empty + kStagesMax;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  if (warp == 0 && elect_one()) {
    tma_prefetch(&tx);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiThreads);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Dependents may launch only once every CTA of this grid holds its TMEM: a
  // dependent CTA co-resident on an SM could otherwise allocate first and
  // spin in griddepcontrol.wait while this CTA blocks in tcgen05.alloc.
  pdl_trigger();

  if (warp == 0) {
    // ---------------- producer ----------------
    if (elect_one()) {
      const uint64_t w_policy = policy_evict_first();  // weights stream once
      auto w_src = [&](int tile, int kb) {
        return wpack + (static_cast<size_t>(tile) * p.num_kb + kb) * (kRowsBlk * kKB);
      };
      // L2 prefetch ahead of the ring: a stream-K CTA's weight range is one
      // contiguous run ([lo, hi) iterations x 32 KB in the packed layout), so
      // the chunk kPrefetch iterations past the one being loaded is prefetched
      // into L2 and the ring's bulk copies see L2 instead of HBM latency (the
      // ring holds <= 5 x 32 KB per SM: at ~1.5 us loaded HBM latency that caps
      // a partition-sized grid near 100 GB/s/SM).
      const long long it_lo = p.streamk ? p.total * blockIdx.x / gridDim.x : 0;
      const long long it_hi = p.streamk ? p.total * (blockIdx.x + 1) / gridDim.x : 0;
      auto prefetch = [&](long long it) {
        if (p.prefetch > 0 && it < it_hi)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(wpack + it * (kRowsBlk * kKB)),
                       "r"(kWBytes)
                       : "memory");
      };
      for (long long it = it_lo + kStages; it < it_lo + kStages + p.prefetch; ++it) prefetch(it);
      // weights of the first kStages stages do not depend on the upstream
      // kernel: stream them before the grid dependency resolves (PDL)
      int pre = 0;
      {
        DecIter wp(p);
        DecWork w;
        while (pre < kStages && wp.next(w))
          for (int kb = w.kb0; kb < w.kb1 && pre < kStages; ++kb, ++pre) {
            mbar_expect_tx(&full[pre], kWBytes + p.x_bytes);
            bulk_load(smem + pre * kStage, w_src(w.tile, kb), kWBytes, &full[pre], w_policy);
          }
      }
      pdl_wait();  // activations are written by the previous kernel
      int stage = 0, fill = 0;
      uint32_t phase = 0;
      DecIter wi(p);
      DecWork w;
      while (wi.next(w)) {
        for (int kb = w.kb0; kb < w.kb1; ++kb, ++fill) {
          uint8_t* st = smem + stage * kStage;
          if (fill >= pre) {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_expect_tx(&full[stage], kWBytes + p.x_bytes);
            bulk_load(st, w_src(w.tile, kb), kWBytes, &full[stage], w_policy);
            prefetch(it_lo + fill + kStages + p.prefetch);
          }
          tma_load_2d(&tx, &full[stage], st + kWBytes, kb * kKB, 0);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t idesc = umma_idesc_bf16(128, kRowsBlk);
    int stage = 0;
    uint32_t phase = 0;
    int local = 0;
    DecIter wi(p);
    DecWork w;
    for (; wi.next(w); ++local) {
      const int acc = local & 1;
      mbar_wait(&tempty[acc], ((local >> 1) & 1) ^ 1);
      tc_fence_after();
      for (int kb = w.kb0; kb < w.kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t wb = smem_u32(smem + stage * kStage);
          const uint32_t xb = wb + kWBytes;
#pragma unroll
          for (int kk = 0; kk < kKB / 16; ++kk)
            umma_bf16(tmem + acc * kRowsBlk, umma_desc_sw128(xb + kk * 32), umma_desc_sw128(wb + kk * 32), idesc,
                      (kb > w.kb0 || kk > 0) ? 1u : 0u);
          umma_commit(&empty[stage]);
          if (kb == w.kb1 - 1) umma_commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else {
    // ---------------- epilogue ----------------
    pdl_wait();  // the fold planes / logits are read by the previous consumer
    const int q = warp & 3;
    const int t = q * 32 + lane_id();
    const bool live = q * 32 < p.tokens;  // warp-uniform: any valid token rows in this quarter
    int local = 0;
    DecIter wi(p);
    DecWork w;
    for (; wi.next(w); ++local) {
      const int acc = local & 1;
      mbar_wait(&tfull[acc], (local >> 1) & 1);
      tc_fence_after();
      if (live) {
        float* base = p.mode == kEpiF32
                          ? p.out + static_cast<size_t>(t) * p.ldo
                          : p.out + (static_cast<size_t>(w.piece) * p.tokens + t) * p.rows;
        for (int c0 = 0; c0 < kRowsBlk; c0 += 32) {
          const int f0 = w.tile * kRowsBlk + c0;
          if (f0 >= p.rows) break;
          uint32_t r[32];
          tmem_ld32(tmem + acc * kRowsBlk + c0 + (static_cast<uint32_t>(q * 32) << 16), r);
          tmem_ld_wait();
          if (t < p.tokens) {
            float4* dst = reinterpret_cast<float4*>(base + f0);
#pragma unroll
            for (int i = 0; i < 8; ++i)
              dst[i] = make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                                   __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace

cudaError_t gemm_decode(const __nv_bfloat16* w_packed, const CUtensorMap& x_map, int box_rows, int rows, int tokens,
                        int K, float* out, int ldo, float* ws, size_t ws_bytes, int sm_count, cudaStream_t stream,
                        GemmFold* fold) {
  if (tokens <= 0) return cudaSuccess;
  if (tokens > 128 || box_rows > 128 || rows % 128 || K % kKB) return cudaErrorInvalidValue;
  DecParams p{};
  p.rows = rows;
  p.tokens = tokens;
  p.num_kb = K / kKB;
  p.n_tiles = (rows / 128 + 1) / 2;
  p.total = static_cast<long long>(p.n_tiles) * p.num_kb;
  p.x_bytes = static_cast<uint32_t>(box_rows) * kKB * 2;
  p.stage_bytes = kWBytes + ((p.x_bytes + 1023u) & ~1023u);
  static const int prefetch_kb = [] {
    const char* e = std::getenv("NX_DEC_PREFETCH");
    return e ? std::max(0, std::atoi(e)) : 0;
  }();
  p.prefetch = prefetch_kb;
  p.stages = std::min<int>(kStagesMax, (kSmemBudget - 512 - (kXBytes - static_cast<int>(p.x_bytes))) /
                                          static_cast<int>(p.stage_bytes));
  const size_t smem = 1024 + static_cast<size_t>(p.stages) * p.stage_bytes + (kXBytes - p.x_bytes) + 512;
  p.ldo = ldo;
  int grid = std::max(1, std::min(p.n_tiles, sm_count));
  if (fold) {
    // planes live after the (unused here) gemm counter block, as for gemm()
    float* planes = ws ? reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + gemm_counter_bytes()) : nullptr;
    const size_t avail = ws_bytes > gemm_counter_bytes() ? ws_bytes - gemm_counter_bytes() : 0;
    const size_t plane_bytes = static_cast<size_t>(tokens) * rows * 4;
    if (planes == nullptr || plane_bytes > avail) return cudaErrorInvalidValue;
    p.mode = kEpiPartial;
    p.out = planes;
    GemmFold f;
    f.planes = planes;
    f.rows = rows;
    f.tokens = tokens;
    f.rows_per_blk = kRowsBlk;
    f.bn = 128;
    f.n_nblk = 1;
    f.num_kb = p.num_kb;
    if (p.n_tiles % sm_count != 0 && p.n_tiles < 8 * sm_count) {
      // Each CTA streams >= kMinIters k-blocks (512 KB): more CTAs would not
      // add bandwidth on a small GEMM, only more pieces -- each piece writes a
      // tokens x 256 fp32 plane slice that the consumer fold reads back.
      static const long long kMinIters = [] {
        const char* e = std::getenv("NX_DEC_MINKB");
        return e ? std::max(1, std::atoi(e)) : 16;
      }();
      const long long g_cap = std::max<long long>(1, (p.total + kMinIters - 1) / kMinIters);
      const int G = static_cast<int>(std::min<long long>(std::min<long long>(sm_count, p.total), g_cap));
      const long long per_min = p.total / G;
      const size_t max_pieces = static_cast<size_t>((p.num_kb + per_min - 1) / per_min) + 1;
      if (max_pieces * plane_bytes <= avail) {
        p.streamk = 1;
        grid = G;
        f.kind = 2;
        f.grid = G;
        f.total = p.total;
      }
    }
    *fold = f;
  } else {
    p.mode = kEpiF32;
    p.out = out;
  }
  ensure_kernels_prepared();
  ++g_kernel_launches;
  return launch_pdl(gemm_decode_kernel, dim3(grid), dim3(kThreads), smem, stream, w_packed, x_map, p);
}

void prepare_gemm_decode_kernel() {
  cudaFuncSetAttribute(gemm_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget + 1024);
}

}  // namespace nxd
