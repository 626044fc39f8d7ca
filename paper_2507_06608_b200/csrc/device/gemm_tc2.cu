// Prefill GEMM on CTA pairs (tcgen05 cta_group::2): one MMA instruction
// computes a 256 x 256 tile across two SMs of a cluster.
//
//   out[t, f] = epilogue( sum_k X[t, k] * W[f, k] )
//
// A = W (M = 256: weight block 2p in CTA 0's smem, block 2p + 1 in CTA 1's),
// B = X (N = 256 tokens: rows [0, 128) of the token block in CTA 0's smem,
// [128, 256) in CTA 1's). Each SM keeps the tensor rate of the single-CTA
// kernel (M128 x N256 per 128 cycles per SM), but every CTA stages only half
// of the activation tile: per k-block 16 KB of W + 16 KB of X instead of
// 16 + 32 KB, i.e. a third less shared-memory fill and L2 -> SM traffic (the
// single-CTA prefill GEMM drove L2 at ~53% of peak, ncu, which the decode
// lane's weight stream competes for when the lanes are co-located).
//
// Protocol (PTX forms as in CuTe's SM100 2SM atoms):
//  * both CTAs TMA their halves; the completion bytes of both land on CTA 0's
//    full barrier (mbarrier address with the peer bit cleared); CTA 0's
//    producer posts expect_tx for the pair;
//  * CTA 0's MMA warp issues tcgen05.mma.cta_group::2 and commits with
//    multicast to both CTAs' empty / accumulator-full barriers;
//  * each CTA's epilogue drains its own TMEM (its 128 weight rows x 256 tokens)
//    and arrives on CTA 0's accumulator-empty barrier (count 2 x 128).
// Weights are fetched by a 2D TMA over the packed, pre-swizzled tile layout
// (box 64 x 128 = one 16 KB tile image, no swizzle mode): the 2SM completion
// form exists only for tensor copies.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "device.cuh"
#include "ptx.cuh"

namespace nxd {

namespace {

constexpr int kBM = 128, kBK = 64, kBN = 256;
constexpr int kHalfN = kBN / 2;
constexpr int kWBytes = kBM * kBK * 2;      // 16 KB
constexpr int kXBytes = kHalfN * kBK * 2;   // 16 KB
constexpr int kStage = kWBytes + kXBytes;   // 32 KB
constexpr int kStages = 6;
constexpr int kThreads = 192;
constexpr int kEpiThreads = 128;
constexpr int kEpiBytes = 32 * kBM * 4;
constexpr int kSmem = 1024 + kStages * kStage + kEpiBytes + 256;
constexpr uint32_t kPeerMask = 0xFEFFFFFFu;  // clears the cluster-rank bit of a shared::cluster address

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_2d_pair(const CUtensorMap* m, uint64_t* bar, void* dst, int c0, int c1,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar) & kPeerMask), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}
// arrive on the same barrier in CTA 0 of the cluster
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, 0;\n\t"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ float silu2(float g) { return g / (1.0f + __expf(-g)); }

__host__ __device__ __forceinline__ size_t packed_row(int m_blk, int kb, int num_kb) {
  // row (of 64 elements) of packed tile (m_blk, kb): see packed_tile_offset in gemm_tc.cu
  return ((static_cast<size_t>(m_blk >> 1) * num_kb + kb) * 2 + (m_blk & 1)) * kBM;
}

struct Pair2Params {
  int rows, tokens, num_kb, n_pairs, n_nblk;  // n_pairs = 256-row weight pairs
  int bn;                                     // token tile width N (<= 256, multiple of 16; N / 2 per CTA)
  int mode;
  void* out;
  int ldo;
  const __nv_bfloat16* bias;
  const __nv_bfloat16* residual;
  int ldr;
  RopeKV rope;
  int wpol;  // weight-stream L2 policy: 0 evict_first, 1 evict_normal (default; NX_PAIR_WPOL)
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tw, const __grid_constant__ CUtensorMap tx, Pair2Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* s_epi = reinterpret_cast<float*>(smem + kStages * kStage);
  uint64_t* full = reinterpret_cast<uint64_t*>(s_epi + 32 * kBM);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair_id = blockIdx.x >> 1, n_pair_ctas = gridDim.x >> 1;
  // No early griddepcontrol.launch_dependents: with it (and the kernel launched
  // with PDL) the monolithic bench hung in ~1 of 3 runs, never with NX_PDL=0.
  // Launched with PDL but without the trigger (NX_PAIR_PDL=1) it ran 6 of 6
  // and saves <1% per prefill step, so the default launch is stream-ordered
  // and the griddepcontrol.wait calls below are no-ops.
  if (warp == 0 && elect_one()) {
    tma_prefetch(&tw);
    tma_prefetch(&tx);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * kEpiThreads);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();  // both CTAs' barriers exist before any cross-CTA signal
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int units = p.n_pairs * p.n_nblk;

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs) ----------------
    if (elect_one()) {
      uint64_t w_policy = policy_evict_first();
      if (p.wpol == 1) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(w_policy));
      const uint64_t x_policy = policy_evict_last();
      int stage = 0, fill = 0, pre = 0;
      uint32_t phase = 0;
      // weights of the first stages: before the grid dependency resolves (PDL)
      for (int u = pair_id; u < units && pre < kStages; u += n_pair_ctas) {
        const int m_blk = (u / p.n_nblk) * 2 + static_cast<int>(rank);
        for (int kb = 0; kb < p.num_kb && pre < kStages; ++kb, ++pre) {
          if (leader) mbar_expect_tx(&full[pre], 2 * kStage);
          tma_2d_pair(&tw, &full[pre], smem + pre * kStage, 0, static_cast<int>(packed_row(m_blk, kb, p.num_kb)),
                      w_policy);
        }
      }
      pdl_wait();
      for (int u = pair_id; u < units; u += n_pair_ctas) {
        const int m_blk = (u / p.n_nblk) * 2 + static_cast<int>(rank);
        const int n_blk = u % p.n_nblk;
        for (int kb = 0; kb < p.num_kb; ++kb, ++fill) {
          uint8_t* st = smem + stage * kStage;
          if (fill >= pre) {
            mbar_wait(&empty[stage], phase ^ 1);
            if (leader) mbar_expect_tx(&full[stage], 2 * kStage);
            tma_2d_pair(&tw, &full[stage], st, 0, static_cast<int>(packed_row(m_blk, kb, p.num_kb)), w_policy);
          }
          tma_2d_pair(&tx, &full[stage], st + kWBytes, kb * kBK, n_blk * p.bn + static_cast<int>(rank) * (p.bn >> 1),
                      x_policy);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (CTA 0 of the pair) ----------------
    if (leader) {
      const uint32_t idesc = umma_idesc_bf16(2 * kBM, p.bn);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int u = pair_id; u < units; u += n_pair_ctas, ++local) {
        const int acc = local & 1;
        mbar_wait(&tempty[acc], ((local >> 1) & 1) ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < p.num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t a_addr = smem_u32(smem + stage * kStage);
            const uint32_t b_addr = a_addr + kWBytes;
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk)
              umma_bf16_pair(tmem + acc * kBN, umma_desc_sw128(a_addr + kk * 32), umma_desc_sw128(b_addr + kk * 32),
                             idesc, (kb > 0 || kk > 0) ? 1u : 0u);
            umma_commit_pair(&empty[stage]);
            if (kb == p.num_kb - 1) umma_commit_pair(&tfull[acc]);
          }
          __syncwarp();
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else {
    // ---------------- epilogue (both CTAs: own 128 weight rows) ----------------
    pdl_wait();
    const int q = warp & 3;
    const int et = threadIdx.x - 64;
    const int lane = lane_id();
    int local = 0;
    for (int u = pair_id; u < units; u += n_pair_ctas, ++local) {
      const int acc = local & 1;
      mbar_wait(&tfull[acc], (local >> 1) & 1);
      tc_fence_after();
      const int m128 = (u / p.n_nblk) * 2 + static_cast<int>(rank);
      const int n_blk = u % p.n_nblk;
      const int f0 = m128 * kBM;
      const bool valid_rows = f0 < p.rows;
      const int tlim = min(p.tokens, (n_blk + 1) * p.bn);  // this tile's token rows
      for (int c0 = 0; c0 < p.bn && valid_rows; c0 += 32) {
        const int tok0 = n_blk * p.bn + c0;
        if (tok0 >= tlim) break;
        const bool has_res = p.mode == kEpiResidual || p.mode == kEpiBiasResidual;
        uint4 res[4];
        if (has_res) {
          const int g = et & 15;
#pragma unroll
          for (int pass = 0; pass < 4; ++pass) {
            const int t = tok0 + pass * 8 + (et >> 4);
            res[pass] = t < tlim ? *reinterpret_cast<const uint4*>(p.residual + static_cast<size_t>(t) * p.ldr +
                                                                      f0 + g * 8)
                                     : make_uint4(0, 0, 0, 0);
          }
        }
        uint32_t r[32];
        tmem_ld32(tmem + acc * kBN + c0 + (static_cast<uint32_t>(q * 32) << 16), r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) s_epi[j * kBM + q * 32 + lane] = __uint_as_float(r[j]);
        named_bar_sync(1, kEpiThreads);
        if (p.mode == kEpiRopeKV) {
          // tile rows = one head: q heads rotate into the qkv output, k heads rotate
          // into the paged cache, v heads are copied into it (as rope_kv_token)
          const RopeKV& rk = p.rope;
          const int head = m128, nq = rk.n_heads, nkv = rk.n_kv_heads;
          const bool is_v = head >= nq + nkv;
          auto rnd = [&](int j, int f) {  // bf16(acc + bias) as the unfused GEMM stored it
            float v = s_epi[j * kBM + f];
            if (p.bias) v += bf2f(p.bias[f0 + f]);
            return bf2f(__float2bfloat16(v));
          };
          if (!is_v) {
#pragma unroll
            for (int pass = 0; pass < 2; ++pass) {
              const int item = pass * kEpiThreads + et;  // 32 tokens x 8 groups of 8 pairs
              const int j = item >> 3, grp = item & 7;
              const int t = tok0 + j;
              if (t < tlim) {
                const float2* cs = rk.table + static_cast<size_t>(t) * 64 + grp * 8;
                __align__(16) __nv_bfloat16 ra[8], rb[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  const float x = rnd(j, grp * 8 + i), y = rnd(j, 64 + grp * 8 + i);
                  const float2 c = cs[i];
                  ra[i] = __float2bfloat16(x * c.x - y * c.y);
                  rb[i] = __float2bfloat16(y * c.x + x * c.y);
                }
                if (head < nq) {
                  __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.out) + static_cast<size_t>(t) * p.ldo + f0;
                  *reinterpret_cast<uint4*>(dst + grp * 8) = *reinterpret_cast<uint4*>(ra);
                  *reinterpret_cast<uint4*>(dst + 64 + grp * 8) = *reinterpret_cast<uint4*>(rb);
                } else {
                  const int sl = rk.slot[t], page = sl / rk.page_tokens, off = sl % rk.page_tokens;
                  __nv_bfloat16* dst =
                      rk.kplane + (static_cast<size_t>(page) * nkv + (head - nq)) * 2 * rk.page_tokens * kBM;
                  *reinterpret_cast<uint4*>(dst + kv_chunk_elem(off, grp)) = *reinterpret_cast<uint4*>(ra);
                  *reinterpret_cast<uint4*>(dst + kv_chunk_elem(off, grp + 8)) = *reinterpret_cast<uint4*>(rb);
                }
              }
            }
          } else {
#pragma unroll
            for (int pass = 0; pass < 4; ++pass) {
              const int item = pass * kEpiThreads + et;  // 32 tokens x 16 chunks of 8
              const int j = item >> 4, c = item & 15;
              const int t = tok0 + j;
              if (t < tlim) {
                __align__(16) __nv_bfloat16 o[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) o[i] = __float2bfloat16(rnd(j, c * 8 + i));
                const int sl = rk.slot[t], page = sl / rk.page_tokens, off = sl % rk.page_tokens;
                __nv_bfloat16* dst =
                    rk.vplane + (static_cast<size_t>(page) * nkv + (head - nq - nkv)) * 2 * rk.page_tokens * kBM;
                *reinterpret_cast<uint4*>(dst + kv_chunk_elem(off, c)) = *reinterpret_cast<uint4*>(o);
              }
            }
          }
        } else if (p.mode == kEpiSwiGLU) {
          const int g = et & 7;
#pragma unroll
          for (int pass = 0; pass < 2; ++pass) {
            const int j = pass * 16 + (et >> 3);
            const int t = tok0 + j;
            if (t < tlim) {
              __align__(16) __nv_bfloat16 o[8];
#pragma unroll
              for (int i = 0; i < 8; ++i)
                o[i] = __float2bfloat16(silu2(s_epi[j * kBM + g * 8 + i]) * s_epi[j * kBM + 64 + g * 8 + i]);
              *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.out) + static_cast<size_t>(t) * p.ldo +
                                        m128 * 64 + g * 8) = *reinterpret_cast<uint4*>(o);
            }
          }
        } else if (p.mode == kEpiF32) {
          const int g = et & 31;
#pragma unroll
          for (int pass = 0; pass < 8; ++pass) {
            const int j = pass * 4 + (et >> 5);
            const int t = tok0 + j;
            if (t < tlim)
              *reinterpret_cast<float4*>(static_cast<float*>(p.out) + static_cast<size_t>(t) * p.ldo + f0 + g * 4) =
                  *reinterpret_cast<const float4*>(&s_epi[j * kBM + g * 4]);
          }
        } else {
          const int g = et & 15;
#pragma unroll
          for (int pass = 0; pass < 4; ++pass) {
            const int j = pass * 8 + (et >> 4);
            const int t = tok0 + j;
            if (t < tlim) {
              float v[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) v[i] = s_epi[j * kBM + g * 8 + i];
              const int f = f0 + g * 8;
              if (p.mode == kEpiBias || p.mode == kEpiBiasResidual) {
                const uint4 b = *reinterpret_cast<const uint4*>(p.bias + f);
                const __nv_bfloat16* bb = reinterpret_cast<const __nv_bfloat16*>(&b);
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] += bf2f(bb[i]);
              }
              if (has_res) {
                const __nv_bfloat16* rb = reinterpret_cast<const __nv_bfloat16*>(&res[pass]);
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] += bf2f(rb[i]);
              }
              __align__(16) __nv_bfloat16 o[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) o[i] = __float2bfloat16(v[i]);
              *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.out) + static_cast<size_t>(t) * p.ldo + f) =
                  *reinterpret_cast<uint4*>(o);
            }
          }
        }
        named_bar_sync(1, kEpiThreads);
      }
      tc_fence_before();
      mbar_arrive_leader(&tempty[acc]);
    }
  }
  tc_fence_before();
  cluster_sync_all();  // no CTA leaves while its peer may still signal it
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
  }
}

bool encode_packed_w(CUtensorMap* map, const void* wpack, size_t rows64) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return false;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[2] = {64, rows64};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {64, kBM};
  const cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(wpack), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool gemm_pair_enabled() {  // NX_GEMM_2CTA=0 falls back to the single-CTA kernel
  static const bool on = [] {
    const char* e = std::getenv("NX_GEMM_2CTA");
    return !(e && e[0] == '0');
  }();
  return on;
}

cudaError_t gemm_pair(const __nv_bfloat16* w_packed, const CUtensorMap& x_map128, int rows, int tokens, int K,
                      int mode, void* out, int ldo, const __nv_bfloat16* bias, const __nv_bfloat16* residual, int ldr,
                      int sm_count, cudaStream_t stream, const RopeKV* rope) {
  if (rows % kBM || K % kBK || sm_count < 2) return cudaErrorInvalidValue;
  if (mode == kEpiRopeKV && (rope == nullptr || rows != (rope->n_heads + 2 * rope->n_kv_heads) * kBM))
    return cudaErrorInvalidValue;
  Pair2Params p{};
  p.rows = rows;
  p.tokens = tokens;
  p.num_kb = K / kBK;
  p.n_pairs = (rows / kBM + 1) / 2;
  // token tile width fitted to the pair waves of the partition (as gemm() does
  // for the single-CTA kernel); N / 2 rows per CTA stay a multiple of 8
  p.bn = kBN;
  const int n_pair_slots = std::max(1, sm_count / 2);
  if (gemm_bn_fit_enabled()) {
    long long best = -1;
    for (int n = kBN; n >= 192; n -= 16) {
      const long long t = static_cast<long long>(p.n_pairs) * ((tokens + n - 1) / n);
      const long long cost = (t + n_pair_slots - 1) / n_pair_slots * (std::max(n, 208) + 256);
      if (best < 0 || cost < best) best = cost, p.bn = n;
    }
  }
  p.n_nblk = (tokens + p.bn - 1) / p.bn;
  p.mode = mode;
  p.out = out;
  p.ldo = ldo;
  p.bias = bias;
  p.residual = residual;
  p.ldr = ldr;
  if (rope) p.rope = *rope;
  // evict_normal for the weight stream: with evict_first the 8 token blocks of a
  // prefill GEMM re-read each weight tile from DRAM (gate_up T = 2048: 390 MB vs
  // 262 MB with evict_normal, same time; ncu), DRAM the co-located decode lane needs
  static const int wpol = [] {
    const char* e = std::getenv("NX_PAIR_WPOL");
    return e ? std::atoi(e) : 1;
  }();
  p.wpol = wpol;
  CUtensorMap tw;
  const size_t rows64 = packed_weight_elems(rows, K) / 64;
  if (!encode_packed_w(&tw, w_packed, rows64)) return cudaErrorInvalidValue;
  const int units = p.n_pairs * p.n_nblk;
  const int pairs = std::max(1, std::min(units, sm_count / 2));
  ensure_kernels_prepared();
  ++g_kernel_launches;
  // NX_PAIR_PDL=1 (experiment): launch with programmatic serialization so the
  // prologue and weight prefetch overlap the previous kernel, still without an
  // early trigger for the kernels after it
  static const bool pdl = [] {
    const char* e = std::getenv("NX_PAIR_PDL");
    return e && e[0] == '1';
  }();
  if (pdl) return launch_pdl(gemm_tc2_kernel, dim3(2 * pairs), dim3(kThreads), kSmem, stream, tw, x_map128, p);
  gemm_tc2_kernel<<<dim3(2 * pairs), dim3(kThreads), kSmem, stream>>>(tw, x_map128, p);
  return cudaGetLastError();
}

void prepare_gemm_pair_kernel() {
  cudaFuncSetAttribute(gemm_tc2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
}

}  // namespace nxd
