// Causal prefill attention over the paged KV cache on tcgen05 / TMEM
// (replaces the reference's AttnPrefill operator, opcost.cpp:113-123).
//
// Work item = (sequence, 128 query rows, kv head). A query row is a (token,
// head-in-GQA-group) pair, row R = token * G + g, so the G heads that share a
// kv head share every staged K/V tile; a tile holds tq = 128 / G tokens.
// The CTA is persistent over items (host-sorted longest first) and runs ten
// warps:
//   warp 0   producer: Q tile by one 4D TMA per 64-dim half (straight from the
//            qkv activations, RoPE already applied by the QKV epilogue), K / V
//            tiles of 128 keys as 8 + 8 cp.async.bulk copies of 4 KB (one per
//            page) into separate 3-stage K and V rings (a K stage frees as soon
//            as S = Q K^T lands). The cache's atom layout (kv_chunk_elem) makes
//            8 consecutive K (V) page halves one uniform UMMA operand.
//   warp 1   MMA issuer: S_j = Q K_j^T (SS, K-major, M 128 x N 128 x K 128)
//            into one of two TMEM score buffers, then O += P_{j-1} V_{j-1}
//            (TS: P read from TMEM where softmax left it, V MN-major from
//            shared memory), so the scores of tile j are computed while the
//            softmax warps work on tile j - 1.
//   warps 2-9 softmax + epilogue, two threads per query row (TMEM lane): warps
//            2-5 own columns 0-63, warps 6-9 columns 64-127 of their lane
//            quarter; the row max and the final sum are swapped through spare
//            TMEM columns around a named barrier of the warp pair. tcgen05.ld
//            the scores, causal mask, running max in the exp2 domain,
//            P = 2^(s - m) written back over the scores as bf16 pairs
//            (tcgen05.st). The O accumulator is rescaled only when a row's
//            max grows by more than 2^8 (the final division by l uses the
//            same stale max, so the result is exact); the epilogue divides
//            by l and stores bf16 rows.
// TMEM: S0 [0, 128), S1 [128, 256), O [256, 384), exchange [384, 390) (512 allocated).
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "device.cuh"
#include "ptx.cuh"

namespace nxd {

namespace {

constexpr int kHD = 128;
constexpr int kRows = 128;                     // query rows per item (TMEM lanes)
constexpr int kKeys = 128;                     // keys per K / V tile
constexpr int kPagesT = kKeys / 16;            // pages per tile
constexpr int kKStages = 3;                     // K ring (freed as soon as S = Q K^T lands)
constexpr int kVStages = 3;                     // V ring (freed after O += P V)
constexpr int kThreads = 320;  // producer, MMA, 8 softmax warps (two per query row)
constexpr uint32_t kQHalf = kRows * 128;       // 16 KB: 128 rows x 64 dims
constexpr uint32_t kKVBytes = kKeys * kHD * 2; // 32 KB: K (or V) of one tile
constexpr uint32_t kSmemMain = 2 * kQHalf + (kKStages + kVStages) * kKVBytes;
constexpr size_t kSmemTotal = kSmemMain + 1024 + 256;
constexpr int kBlockElems = 2 * 16 * kHD;      // one (page, kv head) K | V block
constexpr uint32_t kIdescQK = umma_idesc_bf16(128, 128);
constexpr uint32_t kIdescPV = umma_idesc_bf16(128, 128) | (1u << 16);  // B (V) MN-major
constexpr uint32_t kTmemS = 0, kTmemO = 256;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

struct Item {
  int seq, kvh, tok0, start, q_len, q_start, kv_end, n_tiles, page_off;
};

__device__ __forceinline__ Item get_item(int it, const int2* __restrict__ work, const AttnSeq* __restrict__ seqs,
                                         int hkv, int tq) {
  Item x;
  const int2 w = work[it / hkv];
  x.kvh = it % hkv;
  x.seq = w.x;
  x.tok0 = w.y;
  const AttnSeq m = seqs[w.x];
  x.q_len = m.q_len;
  x.q_start = m.q_start;
  x.start = m.kv_len - m.q_len;
  x.page_off = m.page_off;
  const int last = min(m.q_len, x.tok0 + tq) - 1;
  x.kv_end = x.start + last + 1;
  x.n_tiles = (x.kv_end + kKeys - 1) / kKeys;
  return x;
}

// Two softmax threads share each query row (TMEM lane): warps 2-5 own score
// / output columns 0-63 of their lane quarter, warps 6-9 columns 64-127.
// Partial values are swapped through spare TMEM columns (384 + ...) of the
// row's lane around a named barrier of the two warps.
constexpr uint32_t kTmemXchg = 384;

__device__ __forceinline__ float pair_exchange(uint32_t trow, uint32_t col_mine, uint32_t col_other, float v,
                                               int bar_id) {
  tmem_st1(trow + col_mine, __float_as_uint(v));
  tmem_st_wait();
  tc_fence_before();
  named_bar_sync(bar_id, 64);
  tc_fence_after();
  const uint32_t o = tmem_ld1(trow + col_other);
  tmem_ld_wait();
  return __uint_as_float(o);
}

// One half-row's online-softmax step over a 128-key score tile in TMEM:
// causal mask (keys > limit), the row max from both halves (running, exp2
// domain), P = 2^(s * scale - m) written back as bf16 pairs over the tile's
// first 64 columns (keys 64h.. -> columns 32h..; the partner read its scores
// before the exchange barrier). O (this half's 64 columns) is rescaled after
// PV of the previous tile landed (o_done of global tile gt - 1) only when the
// max grows by more than 2^8; the final 1 / l uses the same stale max, so the
// result is exact. l is this half's partial sum.
__device__ __forceinline__ void softmax_half(uint32_t trow, uint32_t ts, uint32_t to, int h, int j, int limit,
                                             float scale_log2, uint64_t* o_done, uint32_t gt, int bar_id,
                                             float& m, float& l) {
  uint32_t v[2][32];
  tmem_ld32(ts + 64 * h, v[0]);
  tmem_ld32(ts + 64 * h + 32, v[1]);
  tmem_ld_wait();
  const int k0 = j * kKeys + 64 * h;
  float mx2[2] = {-INFINITY, -INFINITY};
  if (k0 + 63 > limit) {
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float sv = (k0 + 32 * c + i <= limit) ? __uint_as_float(v[c][i]) : -INFINITY;
        v[c][i] = __float_as_uint(sv);
        mx2[c] = fmaxf(mx2[c], sv);
      }
  } else {
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int i = 0; i < 32; ++i) mx2[c] = fmaxf(mx2[c], __uint_as_float(v[c][i]));
  }
  const uint32_t xc = kTmemXchg + 2 * (gt & 1);
  const float mine = fmaxf(mx2[0], mx2[1]);
  const float mnew = fmaxf(mine, pair_exchange(trow, xc + h, xc + (h ^ 1), mine, bar_id)) * scale_log2;
  const bool resc = mnew > m + 8.f;
  const bool rescale_o = __any_sync(0xffffffffu, resc && j > 0);
  if (rescale_o) {
    mbar_wait(o_done, (gt - 1) & 1);
    tc_fence_after();
    const float alpha = (resc && j > 0) ? ex2(m - mnew) : 1.f;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      uint32_t o[32];
      tmem_ld32(to + 64 * h + 32 * c, o);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
      tmem_st32(to + 64 * h + 32 * c, o);
    }
    tmem_st_wait();
  }
  if (resc) {
    l *= ex2(m - mnew);
    m = mnew;
  }
  const float mb = m == -INFINITY ? 0.f : m;
  float ls[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int e = 2 * i;
    const float p0 = ex2(fmaf(__uint_as_float(v[e >> 5][e & 31]), scale_log2, -mb));
    const float p1 = ex2(fmaf(__uint_as_float(v[(e + 1) >> 5][(e + 1) & 31]), scale_log2, -mb));
    ls[i & 7] += p0 + p1;
    v[0][i] = pack_bf16(p0, p1);
  }
  tmem_st32(ts + 32 * h, v[0]);
  l += ((ls[0] + ls[1]) + (ls[2] + ls[3])) + ((ls[4] + ls[5]) + (ls[6] + ls[7]));
  // every PV completion is observed exactly once (here, in the rescale above,
  // or in the epilogue for the item's last tile): by the end of this tile's
  // softmax PV_{j-1} has normally landed, so the wait costs nothing
  if (j > 0 && !rescale_o) mbar_wait(o_done, (gt - 1) & 1);
}

// Epilogue of one half-row: O (this half's 64 dims) / l -> bf16 (skipped for
// rows past the item's tokens).
__device__ __forceinline__ void store_half(uint32_t to, bool valid, float l, __nv_bfloat16* dst) {
  const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    uint32_t o[32];
    tmem_ld32(to + 32 * c, o);
    tmem_ld_wait();
    if (valid) {
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        uint4 w;
        w.x = pack_bf16(__uint_as_float(o[i]) * inv, __uint_as_float(o[i + 1]) * inv);
        w.y = pack_bf16(__uint_as_float(o[i + 2]) * inv, __uint_as_float(o[i + 3]) * inv);
        w.z = pack_bf16(__uint_as_float(o[i + 4]) * inv, __uint_as_float(o[i + 5]) * inv);
        w.w = pack_bf16(__uint_as_float(o[i + 6]) * inv, __uint_as_float(o[i + 7]) * inv);
        *reinterpret_cast<uint4*>(dst + 32 * c + i) = w;
      }
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    prefill_attn_tc_kernel(AttnGeom g, const __grid_constant__ CUtensorMap qmap,
                           const __nv_bfloat16* __restrict__ kvplane, const AttnSeq* __restrict__ seqs,
                           const int2* __restrict__ work, int n_items, int tq, const int32_t* __restrict__ pages,
                           __nv_bfloat16* __restrict__ out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sq = smem;                    // [2 halves][128 rows][128 B]
  uint8_t* sk = smem + 2 * kQHalf;                 // [kKStages][128 keys x 256 B]
  uint8_t* sv = sk + kKStages * kKVBytes;          // [kVStages][128 keys x 256 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSmemMain);
  uint64_t* q_full = bars;
  uint64_t* q_empty = bars + 1;
  uint64_t* s_full = bars + 2;           // [2]
  uint64_t* p_full = bars + 4;           // [2]
  uint64_t* o_done = bars + 6;
  uint64_t* o_free = bars + 7;
  uint64_t* k_full = bars + 8;           // [kKStages]
  uint64_t* k_empty = k_full + kKStages;
  uint64_t* v_full = k_empty + kKStages; // [kVStages]
  uint64_t* v_empty = v_full + kVStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(v_empty + kVStages);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hkv = g.n_kv_heads, G = g.group;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&qmap);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 256);
    }
    for (int i = 0; i < kKStages; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < kVStages; ++i) {
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    mbar_init(o_done, 1);
    mbar_init(o_free, 256);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  // Dependents may launch only once every CTA of this grid holds its TMEM: a
  // dependent CTA co-resident on an SM could otherwise allocate first and
  // spin in griddepcontrol.wait while this CTA blocks in tcgen05.alloc.
  pdl_trigger();
  pdl_wait();  // q / k / v of this chunk come from the QKV projection

  if (warp == 0) {
    // ---------------- producer ----------------
    // K / V stay L2-resident: every later query tile of the sequence re-reads them
    uint32_t kv_it = 0, item_it = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++item_it) {
      const Item x = get_item(it, work, seqs, hkv, tq);
      if (lane == 0) {
        mbar_wait(q_empty, (item_it & 1) ^ 1);
        mbar_expect_tx(q_full, 2u * G * tq * 128u);
        for (int h = 0; h < 2; ++h)
          tma_load_4d(&qmap, q_full, sq + h * kQHalf, 0, h, x.kvh * G, x.q_start + x.tok0);
      }
      const int32_t* pt = pages + x.page_off;
      const int last_page = pt[(x.kv_end - 1) >> 4];
      for (int j = 0; j < x.n_tiles; ++j, ++kv_it) {
        // lane p < 8 copies page p of the tile: keys past kv_end re-load the
        // last valid page (masked, finite), so P * V needs no zero fill
        const int key = j * kKeys + (lane & 7) * 16;
        const int page = key < x.kv_end ? pt[key >> 4] : last_page;
        const __nv_bfloat16* src = kvplane + (static_cast<size_t>(page) * hkv + x.kvh) * kBlockElems;
        const uint32_t ks = kv_it % kKStages, vs = kv_it % kVStages;
        if (lane == 0) {
          mbar_wait(&k_empty[ks], ((kv_it / kKStages) & 1) ^ 1);
          mbar_expect_tx(&k_full[ks], kKVBytes);
        }
        __syncwarp();
        if (lane < kPagesT) bulk_load(sk + ks * kKVBytes + lane * 4096, src, 4096, &k_full[ks]);
        if (lane == 0) {
          mbar_wait(&v_empty[vs], ((kv_it / kVStages) & 1) ^ 1);
          mbar_expect_tx(&v_full[vs], kKVBytes);
        }
        __syncwarp();
        if (lane < kPagesT) bulk_load(sv + vs * kKVBytes + lane * 4096, src + kBlockElems / 2, 4096, &v_full[vs]);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    uint32_t kv_it = 0, gt = 0, item_it = 0;
    const uint32_t sq_s = smem_u32(sq), sk_s = smem_u32(sk), sv_s = smem_u32(sv);
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++item_it) {
      const Item x = get_item(it, work, seqs, hkv, tq);
      if (lane == 0) {
        mbar_wait(q_full, item_it & 1);
        tc_fence_after();
        auto pv = [&](uint32_t gtp, uint32_t kvp, bool first) {
          const uint32_t b = gtp & 1, vst = kvp % kVStages;
          mbar_wait(&v_full[vst], (kvp / kVStages) & 1);
          mbar_wait(&p_full[b], (gtp >> 1) & 1);
          if (first && item_it > 0) mbar_wait(o_free, (item_it - 1) & 1);
          tc_fence_after();
          const uint32_t vb = sv_s + vst * kKVBytes;
#pragma unroll
          for (int s = 0; s < kPagesT; ++s)  // 16 keys (one page) per MMA: V atoms 2 KB (keys) / 1 KB (dims) apart
            umma_bf16_ts(tbase + kTmemO, tbase + kTmemS + b * 128 + 8 * s,
                         umma_desc_sw128(vb + s * 4096, 1024, 2048), kIdescPV, (!first || s > 0) ? 1u : 0u);
          umma_commit(&v_empty[vst]);
          umma_commit(o_done);
        };
        for (int j = 0; j < x.n_tiles; ++j, ++kv_it, ++gt) {
          const uint32_t kst = kv_it % kKStages;
          mbar_wait(&k_full[kst], (kv_it / kKStages) & 1);
          tc_fence_after();
          const uint32_t b = gt & 1;
          const uint32_t kb = sk_s + kst * kKVBytes;
#pragma unroll
          for (int s = 0; s < 8; ++s) {  // head dim in 8 steps of 16: dims 64..127 are the +1 KB / +16 KB atoms
            const uint32_t koff = (s >> 2) * 1024 + (s & 3) * 32, qoff = (s >> 2) * kQHalf + (s & 3) * 32;
            umma_bf16(tbase + kTmemS + b * 128, umma_desc_sw128(sq_s + qoff, 16, 1024),
                      umma_desc_sw128(kb + koff, 16, 2048), kIdescQK, s > 0 ? 1u : 0u);
          }
          umma_commit(&k_empty[kst]);
          umma_commit(&s_full[b]);
          if (j == x.n_tiles - 1) umma_commit(q_empty);
          if (j > 0) pv(gt - 1, kv_it - 1, j == 1);
        }
        pv(gt - 1, kv_it - 1, x.n_tiles == 1);
      }
      __syncwarp();
    }
  } else {
    // ---------------- softmax + epilogue: two threads per query row ----------------
    const int q = warp & 3;                 // TMEM lane quarter of this warp
    const int h = (warp - 2) >> 2;          // column half of the row
    const int bar_id = 1 + q;               // named barrier of the warp pair sharing these rows
    const int r = q * 32 + lane;            // query row within the item
    const uint32_t trow = tbase + (static_cast<uint32_t>(q * 32) << 16);
    uint32_t gt = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const Item x = get_item(it, work, seqs, hkv, tq);
      const int tk = x.tok0 + r / G;
      const bool valid = r < G * tq && tk < x.q_len;
      const int limit = valid ? x.start + tk : -1;  // keys <= limit are visible
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < x.n_tiles; ++j, ++gt) {
        const uint32_t b = gt & 1;
        mbar_wait(&s_full[b], (gt >> 1) & 1);
        tc_fence_after();
        softmax_half(trow, trow + kTmemS + b * 128, trow + kTmemO, h, j, limit, g.scale_log2, o_done, gt, bar_id,
                     m, l);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(&p_full[b]);
      }
      // epilogue: O / (l_0 + l_1) -> bf16, this half's 64 dims of [token][head * 128]
      mbar_wait(o_done, (gt - 1) & 1);
      tc_fence_after();
      const float lt = l + pair_exchange(trow, kTmemXchg + 4 + h, kTmemXchg + 4 + (h ^ 1), l, bar_id);
      store_half(trow + kTmemO + 64 * h, valid, lt,
                 out + static_cast<size_t>(x.q_start + tk) * g.out_stride + (x.kvh * G + r % G) * kHD + 64 * h);
      tc_fence_before();
      mbar_arrive(o_free);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}


}  // namespace

bool encode_q_heads_map(CUtensorMap* map, const void* qkv, int tokens, int n_heads, int group,
                        int row_stride_elems) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return false;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  // (64 dims, 2 halves, heads, tokens): box = one 64-dim half of G heads x tq
  // tokens -> smem rows token * G + g of 128 B, 128B-swizzled (UMMA K-major).
  const cuuint64_t dims[4] = {64, 2, static_cast<cuuint64_t>(n_heads), static_cast<cuuint64_t>(tokens)};
  const cuuint64_t strides[3] = {128, 256, static_cast<cuuint64_t>(row_stride_elems) * 2};
  const cuuint32_t box[4] = {64, 1, static_cast<cuuint32_t>(group), static_cast<cuuint32_t>(prefill_attn_tokens_per_item(group))};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(qkv), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int prefill_attn_tokens_per_item(int group) { return kRows / group; }

cudaError_t prefill_attention(const AttnGeom& g, const CUtensorMap& qmap, const __nv_bfloat16* kvplane,
                              const AttnSeq* seqs, const int2* work, int n_work, const int32_t* pages,
                              __nv_bfloat16* out, int sm_count, cudaStream_t s) {
  if (n_work == 0) return cudaSuccess;
  if (g.head_dim != kHD || g.group < 1 || g.group > kRows) return cudaErrorInvalidValue;
  if (const cudaError_t pe = ensure_kernels_prepared(); pe != cudaSuccess) return pe;
  const int n_items = n_work * g.n_kv_heads;
  const int grid = std::max(1, std::min(n_items, sm_count));
  ++g_kernel_launches;
  return launch_pdl(prefill_attn_tc_kernel, dim3(grid), dim3(kThreads), kSmemTotal, s, g, qmap, kvplane, seqs,
                    work, n_items, prefill_attn_tokens_per_item(g.group), pages, out);
}

cudaError_t prepare_prefill_attention_kernel() {
  return cudaFuncSetAttribute(prefill_attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(kSmemTotal));
}

}  // namespace nxd
