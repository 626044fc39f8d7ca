// Decode attention over the paged KV cache and the device-resident block
// table (prefill attention is attn_prefill.cu).
//
// KV cache layout per layer: [page][kv_head][K | V] blocks of 16 token rows x
// 128 dims, each half four 1 KB SWIZZLE_128B atoms (kv_chunk_elem,
// device.cuh). One (page, kv head) is a contiguous 8 KB run [K 4 KB | V 4 KB]
// that is already a conflict-free shared-memory image for ldmatrix (chunk
// (c & 7) ^ (r & 7) within each 128 B atom row): a decode tile is one
// cp.async.bulk per page. One 8 KB copy instead of two 4 KB ones: bulk copies
// pay a per-copy cost (tools/bw_probe.cu: 4 KB copies 27-55 GB/s/SM, 16-32 KB
// copies 107-190 GB/s/SM).
//
// Decode: the G query heads of a token form the rows of a kv head's item;
// items are split over warp pairs (stream-K) and partials merged by a
// log-sum-exp combine. Softmax runs in fp32 with exp2 and a running max.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cstdint>
#include <cstdlib>
#include <string>

#include "device.cuh"
#include "ptx.cuh"

namespace nxd {
namespace {

constexpr int kHD = 128;        // head dim (all supported models)

constexpr int kKVBlock = 2 * 16 * kHD;  // elements of one (page, kv head) K|V block

// Swizzled offset (elements) of (row, col) in a [rows][128] bf16 tile.
__device__ __forceinline__ int swz(int row, int col) {
  return row * kHD + ((((col >> 3) ^ (row & 7)) << 3) | (col & 7));
}

// Shared-window addresses (uint32): the generic-pointer forms below cost a
// cvta per ldmatrix, which was ~25% of the decode kernel's instructions (ncu).
__device__ __forceinline__ void ldsm_x4_s(uint32_t (&r)[4], uint32_t a) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
__device__ __forceinline__ void ldsm_x4_t_s(uint32_t (&r)[4], uint32_t a) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
// 2^x on the SFU (ftz; 2^-inf = 0): exp2f adds range fix-ups around MUFU.EX2.
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// 8x8 b16 transpose across the warp (fragment layout in and out).
__device__ __forceinline__ uint32_t movmatrix_trans(uint32_t v) {
  uint32_t r;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Decode ("stream-K flash decoding"): the work is the flattened list of
// 32-key tiles of every (sequence, kv head) item, ordered by sequence then
// head. Unit w (a warp pair) of the persistent grid owns the contiguous tile
// range [w T / W, (w + 1) T / W) (T tiles, W units), so every unit streams
// the same number of KV bytes regardless of the length mix: no wave
// quantization, no idle tails. Each pair runs its own cp.async.bulk ring of
// NX_DEC_STAGES stages (one lane issues 2 pages x one 8 KB K|V block per
// tile), continuing across item boundaries; warp h of the pair takes keys
// [16 h, 16 h + 16) of every tile. The kernel is issue-latency bound (ncu
// 4.4 cycles / instruction with one warp per SMSP), so warps beat ring
// depth: 8 pairs x 1 stage (4 warps per SMSP) streams ~21% more per SM
// than 4 pairs x 3 stages on a 32-SM lane
// (profiles/r01s2_attn_decode_bw.md). The pair merges its
// (m, l, O) at the end of each item segment. An item covered by one unit is
// finalized in place; an item split across units leaves (m, l, O) partials
// that the unit writing an item's last partial folds with a log-sum-exp
// rescale (an atomic count per item; no separate combine launch).
// The tile math is transposed (keys / head dims on the MMA's M side, the
// G <= 8 query heads of the kv head on its N = 8 side; see the kernel).
constexpr int kKTD = 32;      // keys per decode tile (two 16-token pages)
#ifndef NX_DEC_STAGES
#define NX_DEC_STAGES 1
#endif
#ifndef NX_DEC_PAIRS
#define NX_DEC_PAIRS 8
#endif
constexpr int kStD = NX_DEC_STAGES;   // ring stages per pair
constexpr int kPairsD = NX_DEC_PAIRS; // warp pairs per CTA (one CTA per SM)
constexpr int kTileD = kKTD * kHD;  // elements per K (or V) tile
// named barrier 1 + pair must stay below the 16 hardware barriers; the ring,
// the fp32 staging and the barriers must fit one SM's 227 KB opt-in
static_assert(kPairsD >= 1 && kPairsD <= 15, "NX_DEC_PAIRS must be in [1, 15]");
static_assert(kStD >= 1, "NX_DEC_STAGES must be >= 1");
static_assert(static_cast<size_t>(kPairsD) * (kStD * 2 * kTileD + 8 * kHD * 2) * 2 + 2 * kPairsD * kStD * 8 +
                      kPairsD * 32 * 4 + 64 <= 227u * 1024u,
              "NX_DEC_PAIRS x NX_DEC_STAGES exceeds 227 KB of shared memory");

// Head-pair items (HP = 2, even kv-head counts): one unit streams two kv heads
// of a sequence together, so every page refill is one 16 KB copy of two
// adjacent (page, kv head) blocks instead of two 8 KB copies; warp h of the
// pair owns kv head 2 hg + h over all 32 keys of a tile, so no pair merge.
// Bulk copies pay a per-copy cost: one issuing thread moves 55 / 109 / 182
// GB/s per SM with 8 / 16 / 32 KB copies on a 32-SM lane
// (profiles/r02_bw_probe_copy_size.jsonl).
#ifndef NX_DEC_PAIRS_HP2
#define NX_DEC_PAIRS_HP2 5
#endif
template <int HP>
struct DecCfg {
  static constexpr int kPairs = HP == 1 ? kPairsD : NX_DEC_PAIRS_HP2;
  static constexpr int kSt = HP == 1 ? kStD : 1;
  // ring stage (2 pages x HP blocks) and staging (HP = 1: Q / fp32 shared;
  // HP = 2: Q [16][128] bf16, then one [8][128] fp32 per warp), bf16 units
  static constexpr int kStageElems = 2 * HP * kKVBlock;
  static constexpr int kStagingElems = HP == 1 ? 8 * kHD * 2 : 3 * 8 * kHD * 2;
  static constexpr int kPairElems = kSt * kStageElems + kStagingElems;
  static constexpr size_t kSmem = static_cast<size_t>(kPairs) * kPairElems * 2 + 2 * kPairs * kSt * 8 +
                                  kPairs * 32 * 4 + 64;
};
static_assert(DecCfg<2>::kPairs >= 1 && DecCfg<2>::kPairs <= 15, "NX_DEC_PAIRS_HP2 must be in [1, 15]");
static_assert(DecCfg<2>::kSmem <= 227u * 1024u, "NX_DEC_PAIRS_HP2 exceeds 227 KB of shared memory");


// Item (sequence, kv head) holding flattened tile index gt: seq_prefix[s] is
// the first tile of sequence s (all heads), tiles(s) = ceil(kv_len / 32).
struct DecPos {
  int seq, kvh, tile, n_tiles;
  long long item_start;  // flattened index of the item's first tile
};
__device__ __forceinline__ DecPos dec_locate(const int* __restrict__ seq_prefix, int n_seq, int hkv,
                                             long long gt) {
  int lo = 0, hi = n_seq - 1;  // last s with seq_prefix[s] * hkv <= gt
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (static_cast<long long>(seq_prefix[mid]) * hkv <= gt) lo = mid;
    else hi = mid - 1;
  }
  DecPos d;
  d.seq = lo;
  d.n_tiles = seq_prefix[lo + 1] - seq_prefix[lo];
  const long long rel = gt - static_cast<long long>(seq_prefix[lo]) * hkv;
  d.kvh = static_cast<int>(rel / d.n_tiles);
  d.tile = static_cast<int>(rel % d.n_tiles);
  d.item_start = static_cast<long long>(seq_prefix[lo]) * hkv + static_cast<long long>(d.kvh) * d.n_tiles;
  return d;
}

__device__ __forceinline__ void dec_advance(DecPos& d, const int* __restrict__ seq_prefix, int n_seq,
                                            int hkv) {
  if (++d.tile < d.n_tiles) return;
  d.tile = 0;
  d.item_start += d.n_tiles;
  if (++d.kvh == hkv) {
    d.kvh = 0;
    if (++d.seq < n_seq) d.n_tiles = seq_prefix[d.seq + 1] - seq_prefix[d.seq];
  }
}

template <int HP>
__global__ void __launch_bounds__(2 * DecCfg<HP>::kPairs * 32, 1)
    decode_attn_kernel(AttnGeom g, const __nv_bfloat16* __restrict__ qkv,
                       const __nv_bfloat16* __restrict__ kplane,
                       const __nv_bfloat16* __restrict__ vplane, const AttnSeq* __restrict__ seqs,
                       const int* __restrict__ seq_prefix, int n_seq, long long total, long long W,
                       const int32_t* __restrict__ pages,
                       __nv_bfloat16* __restrict__ out, float* __restrict__ part_o,
                       float* __restrict__ part_ml, int* __restrict__ item_done) {
  extern __shared__ __align__(1024) uint8_t smem_attn[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp >> 1, half = warp & 1;
  // per pair: [kStD][K tile][V tile] + one [8][128] fp32 staging (warp 1
  // publishes its O there, warp 0 folds into it in place -- every element is
  // read and rewritten by the same lane -- and it doubles as the Q staging at
  // segment starts) + kStD barriers
  // (HP = 2: separate Q and per-warp output staging, see DecCfg)
  constexpr int kPairs = DecCfg<HP>::kPairs, kSt = DecCfg<HP>::kSt;
  constexpr int kPairElems = DecCfg<HP>::kPairElems;  // bf16 units
  __nv_bfloat16* pbase = reinterpret_cast<__nv_bfloat16*>(smem_attn) + pair * kPairElems;
  const uint32_t pbase_s = smem_u32(pbase);
  __nv_bfloat16* sq = pbase + kSt * DecCfg<HP>::kStageElems;  // Q staging [HP x 8][128] bf16
  float* stage_b = HP == 1 ? reinterpret_cast<float*>(sq)     // [8][128] fp32
                           : reinterpret_cast<float*>(sq + 8 * kHD * 2) + half * 8 * kHD;
  float* stage_a = stage_b;                                 // merged (m, l, O), in place
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<__nv_bfloat16*>(smem_attn) +
                                               kPairs * kPairElems) + pair * kSt;
  // empty[s]: both warps of the pair are done reading stage s (2 arrivals); only
  // the producer waits on it, so neither warp stalls on the other per tile
  uint64_t* empty = full + kPairs * kSt;
  float* ml_b = reinterpret_cast<float*>(full + 2 * kPairs * kSt - pair * kSt) + pair * 32;  // [8 heads][m, l]
  const uint32_t bar_id = 1 + pair;
  auto pair_sync = [&] { named_bar_sync(bar_id, 64); };
  pdl_trigger();
  // units are dealt to CTAs round-robin, so a short launch (W < SMs x pairs)
  // spreads over every SM of the lane instead of filling the first CTAs
  const long long gw = static_cast<long long>(pair) * gridDim.x + blockIdx.x;
  if (gw >= W) return;  // both warps of the pair leave together
  const long long lo = total * gw / W, hi = total * (gw + 1) / W;
  const int hkv = g.n_kv_heads;
  const int hkv_g = hkv / HP;  // items per sequence (kv heads or head pairs)
  const bool producer = half == 0 && lane == 0;
  if (producer) {
    for (int i = 0; i < kSt; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 2);
    }
    fence_barrier_init();
  }
  pair_sync();
  pdl_wait();  // the new token's K/V and Q come from the QKV / RoPE kernels
  const uint64_t pol = policy_evict_first();
  // producer cursor (one lane) runs kStD tiles ahead of the consumer cursor;
  // the page ids of the next tile to issue are looked up one refill ahead, so
  // the dependent global loads (sequence -> page table -> page) overlap a tile
  // of compute instead of stalling the producer's warp at every refill
  DecPos prod = dec_locate(seq_prefix, n_seq, hkv_g, lo);
  long long issued = lo;
  int nxt_pg0 = 0, nxt_pg1 = 0, nxt_kvh = 0;
  // the producer's sequence record is re-read only when its cursor enters a
  // new sequence, so a refill's lookup is one dependent load (the page ids),
  // not a chain (record -> page ids)
  int pm_seq = -1, pm_kv_len = 0;
  const int32_t* pm_pt = pages;
  auto lookup = [&]() {
    if (prod.seq != pm_seq) {
      const AttnSeq ms = seqs[prod.seq];
      pm_seq = prod.seq;
      pm_kv_len = ms.kv_len;
      pm_pt = pages + ms.page_off;
    }
    // a tile starts below kv_len; a second half past it re-loads the first
    // half's page (masked, finite)
    const int key = prod.tile * kKTD;
    nxt_pg0 = pm_pt[key >> 4];
    nxt_pg1 = key + 16 < pm_kv_len ? pm_pt[(key + 16) >> 4] : nxt_pg0;
    nxt_kvh = prod.kvh;
  };
  auto issue = [&](int st) {
    __nv_bfloat16* dst = pbase + st * DecCfg<HP>::kStageElems;
    mbar_expect_tx(&full[st], 2 * HP * 8192);
    bulk_load(dst, kplane + (static_cast<size_t>(nxt_pg0) * hkv + nxt_kvh * HP) * kKVBlock, HP * 8192, &full[st],
              pol);
    bulk_load(dst + HP * kKVBlock, kplane + (static_cast<size_t>(nxt_pg1) * hkv + nxt_kvh * HP) * kKVBlock,
              HP * 8192, &full[st], pol);
  };
  if (producer) {
    for (; issued < hi && issued < lo + kSt; ++issued) {
      lookup();
      issue(static_cast<int>(issued - lo));
      dec_advance(prod, seq_prefix, n_seq, hkv_g);
    }
    if (issued < hi) lookup();
  }
  DecPos cur = dec_locate(seq_prefix, n_seq, hkv_g, lo);
  // Transposed tile math: S^T = K Q^T and O^T += V^T P^T, so keys / head
  // dims are the MMA's 16-row M side and the <= 8 query heads of the GQA
  // group its N = 8 side (half the m16n8k16 count of Q-as-rows, where 16 MMA
  // rows carry G = 4 heads). Lane l owns heads h0 = 2 (l & 3), h0 + 1.
  uint32_t qb[8][2];   // B fragments of Q^T, 8 k-steps of 16 dims
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  float o[8][4];       // O^T block db: dims 16 db + l/4 (+8) x heads h0, h0 + 1
  AttnSeq meta = seqs[cur.seq];
  int seg_tile0 = cur.tile;
  const int h0 = 2 * (lane & 3);
  // ldmatrix lane addresses, hoisted: in a 1 KB atom (8 rows x 128 B), chunk
  // (2 k + b) & 7 of row r sits at r * 128 + ((2 k + b) ^ r) << 4 =
  // (b ^ (r & 1)) << 4 | ((k ^ g) << 5) with g = (r & 6) >> 1, so 4 per-lane
  // bases cover k = 0..3; dims 64..127 (k & 4) are the next atom, +1 KB, and
  // token rows 8..15 the atom pair 2 KB on (kv_chunk_elem). K: row (lane & 7) + 8 b3, chunk b = lane >> 4;
  // V (trans): row (lane & 7) + 8 (lane >> 4), chunk b = b3; relative to the
  // page block of the sub-tile (added at use).
  const int l7 = lane & 7, b3 = (lane >> 3) & 1, b4 = lane >> 4, gx = (l7 & 6) >> 1;
  uint32_t koff[4], voff[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    koff[j] = static_cast<uint32_t>(b3 * 2048 + l7 * 128 + (((b4 ^ l7) & 1) << 4) + ((j ^ gx) << 5));
    voff[j] = static_cast<uint32_t>(4096 + b4 * 2048 + l7 * 128 + (((b3 ^ l7) & 1) << 4) +
                                    ((j ^ gx) << 5));
  }
  for (long long gt = lo; gt < hi; ++gt) {
    const int i = static_cast<int>(gt - lo), buf = i % kSt;
    if (gt == lo || cur.tile == 0) {  // new segment: this item's queries
      meta = seqs[cur.seq];
      seg_tile0 = cur.tile;
      // rows 8 hh + q: query head q of the item's kv head hh (HP = 2: warp h
      // takes rows 8 h ..)
      for (int c = half * 32 + lane; c < HP * 8 * 16; c += 64) {
        const int r = c >> 4, chunk = c & 15, hh = r >> 3, qr = r & 7;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (qr < g.group)
          v = *reinterpret_cast<const uint4*>(qkv + static_cast<size_t>(meta.q_start) * g.qkv_stride +
                                              ((cur.kvh * HP + hh) * g.group + qr) * kHD + chunk * 8);
        *reinterpret_cast<uint4*>(sq + r * kHD + ((chunk ^ (r & 7)) << 3)) = v;
      }
      pair_sync();
      const __nv_bfloat16* sqw = sq + (HP == 2 ? half * 8 * kHD : 0);
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        uint32_t r[4];
        ldsm_x4(r, sqw + swz(lane & 7, k * 16 + ((lane >> 3) << 3)));
        qb[k][0] = r[0], qb[k][1] = r[1], qb[k + 1][0] = r[2], qb[k + 1][1] = r[3];
      }
      m0 = m1 = -INFINITY;
      l0 = l1 = 0.f;
#pragma unroll
      for (int d = 0; d < 8; ++d) o[d][0] = o[d][1] = o[d][2] = o[d][3] = 0.f;
    }
    mbar_wait(&full[buf], (i / kSt) & 1);
    // [2 pages][HP kv heads][K 16 | V 16][128]; shared-window byte address of the stage
    const uint32_t sbase0 = pbase_s + static_cast<uint32_t>(buf * DecCfg<HP>::kStageElems * 2);
    // HP = 1: warp h takes page h of the tile (keys 16 h ..); HP = 2: warp h
    // takes its kv head's block of both pages, one 16-key sub-tile after the other
#pragma unroll
    for (int j = 0; j < HP; ++j) {
    const int sub = HP == 1 ? half : j;
    const uint32_t sbase = sbase0 + static_cast<uint32_t>(sub * HP * 8192 + (HP == 2 ? half * 8192 : 0));
    // S^T = K Q^T over 16 keys: 8 k-steps
    // four independent accumulation chains of two MMAs (HMMA latency, not issue, bounds a chain)
    float sc[4][4];
#pragma unroll
    for (int c = 0; c < 4; ++c) sc[c][0] = sc[c][1] = sc[c][2] = sc[c][3] = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      uint32_t a[4];
      ldsm_x4_s(a, sbase + koff[k & 3] + ((k & 4) << 8));
      mma16816(sc[k & 3], a, qb[k][0], qb[k][1]);
    }
    float s[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) s[j] = (sc[0][j] + sc[1][j]) + (sc[2][j] + sc[3][j]);
    // mask keys past kv_len; online softmax down each head column
    const int key0 = cur.tile * kKTD + sub * 16 + (lane >> 2);
    float mx0 = m0, mx1 = m1;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const bool ok = key0 + j * 8 < meta.kv_len;
      s[2 * j] = ok ? s[2 * j] * g.scale_log2 : -INFINITY;
      s[2 * j + 1] = ok ? s[2 * j + 1] * g.scale_log2 : -INFINITY;
      mx0 = fmaxf(mx0, s[2 * j]);
      mx1 = fmaxf(mx1, s[2 * j + 1]);
    }
#pragma unroll
    for (int x = 4; x < 32; x <<= 1) {
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffff, mx0, x));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffff, mx1, x));
    }
    const float b0 = mx0 == -INFINITY ? 0.f : mx0, b1 = mx1 == -INFINITY ? 0.f : mx1;
    if (__any_sync(0xffffffff, mx0 != m0 || mx1 != m1)) {  // running max moved: rescale
      const float al0 = ex2(m0 - b0), al1 = ex2(m1 - b1);
      l0 *= al0, l1 *= al1;
#pragma unroll
      for (int d = 0; d < 8; ++d) o[d][0] *= al0, o[d][2] *= al0, o[d][1] *= al1, o[d][3] *= al1;
      m0 = mx0, m1 = mx1;
    }
    // P^T in C layout (keys x heads) -> B fragments (keys = k) by an 8x8 transpose
    const float p00 = ex2(s[0] - b0), p01 = ex2(s[1] - b1);
    const float p10 = ex2(s[2] - b0), p11 = ex2(s[3] - b1);
    l0 += p00 + p10;
    l1 += p01 + p11;
    const uint32_t pb0 = movmatrix_trans(pack_bf16(p00, p01));
    const uint32_t pb1 = movmatrix_trans(pack_bf16(p10, p11));
    // O^T += V^T P^T: 8 blocks of 16 dims, one k-step over this warp's keys
#pragma unroll
    for (int db = 0; db < 8; ++db) {
      uint32_t a[4];
      ldsm_x4_t_s(a, sbase + voff[db & 3] + ((db & 4) << 8));
      mma16816(o[db], a, pb0, pb1);
    }
    }  // sub-tiles
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[buf]);  // this warp is done with stage buf
    // refill this stage kSt tiles ahead, once both warps released it
    if (producer && issued < hi) {
      mbar_wait(&empty[buf], static_cast<uint32_t>((i / kSt) & 1));
      issue(buf);
      dec_advance(prod, seq_prefix, n_seq, hkv_g);
      if (++issued < hi) lookup();
    }
    // segment end: last tile of the item or of this unit's range
    const bool item_end = cur.tile == cur.n_tiles - 1;
    if (item_end || gt == hi - 1) {
      float lt0 = l0, lt1 = l1;
#pragma unroll
      for (int x = 4; x < 32; x <<= 1) {
        lt0 += __shfl_xor_sync(0xffffffff, lt0, x);
        lt1 += __shfl_xor_sync(0xffffffff, lt1, x);
      }
      // HP = 1: merge the pair (warp 1 publishes (m, l, O), warp 0 folds);
      // HP = 2: each warp finalizes its own kv head
      if (HP == 1 && half == 1) {
#pragma unroll
        for (int d = 0; d < 8; ++d) {
          const int dim = d * 16 + (lane >> 2);
          stage_b[h0 * kHD + dim] = o[d][0];
          stage_b[(h0 + 1) * kHD + dim] = o[d][1];
          stage_b[h0 * kHD + dim + 8] = o[d][2];
          stage_b[(h0 + 1) * kHD + dim + 8] = o[d][3];
        }
        if (lane < 4) {
          ml_b[h0 * 2] = m0, ml_b[h0 * 2 + 1] = lt0;
          ml_b[(h0 + 1) * 2] = m1, ml_b[(h0 + 1) * 2 + 1] = lt1;
        }
      }
      if (HP == 1) pair_sync();
      if (HP == 2 || half == 0) {
        const int kvh_w = cur.kvh * HP + (HP == 2 ? half : 0);  // this warp's kv head
        const float mb0 = HP == 1 ? ml_b[h0 * 2] : -INFINITY, lb0 = HP == 1 ? ml_b[h0 * 2 + 1] : 0.f;
        const float mb1 = HP == 1 ? ml_b[(h0 + 1) * 2] : -INFINITY, lb1 = HP == 1 ? ml_b[(h0 + 1) * 2 + 1] : 0.f;
        const float M0 = fmaxf(m0, mb0), M1 = fmaxf(m1, mb1);
        const float fa0 = m0 == -INFINITY ? 0.f : ex2(m0 - M0), fb0 = mb0 == -INFINITY ? 0.f : ex2(mb0 - M0);
        const float fa1 = m1 == -INFINITY ? 0.f : ex2(m1 - M1), fb1 = mb1 == -INFINITY ? 0.f : ex2(mb1 - M1);
        const float L0 = lt0 * fa0 + lb0 * fb0, L1 = lt1 * fa1 + lb1 * fb1;
        const bool whole = seg_tile0 == 0 && item_end;
        const float sa0 = fa0 * (whole ? (L0 > 0.f ? 1.f / L0 : 0.f) : 1.f);
        const float sb0 = fb0 * (whole ? (L0 > 0.f ? 1.f / L0 : 0.f) : 1.f);
        const float sa1 = fa1 * (whole ? (L1 > 0.f ? 1.f / L1 : 0.f) : 1.f);
        const float sb1 = fb1 * (whole ? (L1 > 0.f ? 1.f / L1 : 0.f) : 1.f);
#pragma unroll
        for (int d = 0; d < 8; ++d) {
          const int dim = d * 16 + (lane >> 2);
          if (HP == 1) {
            stage_a[h0 * kHD + dim] = o[d][0] * sa0 + stage_b[h0 * kHD + dim] * sb0;
            stage_a[(h0 + 1) * kHD + dim] = o[d][1] * sa1 + stage_b[(h0 + 1) * kHD + dim] * sb1;
            stage_a[h0 * kHD + dim + 8] = o[d][2] * sa0 + stage_b[h0 * kHD + dim + 8] * sb0;
            stage_a[(h0 + 1) * kHD + dim + 8] = o[d][3] * sa1 + stage_b[(h0 + 1) * kHD + dim + 8] * sb1;
          } else {
            stage_a[h0 * kHD + dim] = o[d][0] * sa0;
            stage_a[(h0 + 1) * kHD + dim] = o[d][1] * sa1;
            stage_a[h0 * kHD + dim + 8] = o[d][2] * sa0;
            stage_a[(h0 + 1) * kHD + dim + 8] = o[d][3] * sa1;
          }
        }
        __syncwarp();
        if (whole) {
          __nv_bfloat16* dst = out + static_cast<size_t>(meta.q_start) * g.out_stride + kvh_w * g.group * kHD;
          for (int c = lane; c < g.group * 16; c += 32) {
            const float4 u = *reinterpret_cast<const float4*>(stage_a + c * 8);
            const float4 v = *reinterpret_cast<const float4*>(stage_a + c * 8 + 4);
            uint4 w;
            w.x = pack_bf16(u.x, u.y), w.y = pack_bf16(u.z, u.w), w.z = pack_bf16(v.x, v.y), w.w = pack_bf16(v.z, v.w);
            *reinterpret_cast<uint4*>(dst + c * 8) = w;
          }
        } else {
          // compact partial slot: item + unit. The units of item k are
          // [first_k, last_k] with first_{k+1} >= last_k, so item + unit is unique
          // per (item, unit) and below n_items + W (the combine reads item + first + q);
          // HP heads per item slot
          const size_t slot =
              (static_cast<size_t>(cur.seq) * hkv_g + cur.kvh + static_cast<size_t>(gw)) * HP + (HP == 2 ? half : 0);
          float4* po = reinterpret_cast<float4*>(part_o + slot * g.group * kHD);
          for (int c = lane; c < g.group * 32; c += 32) po[c] = *reinterpret_cast<const float4*>(stage_a + c * 4);
          if (lane < 4) {
            if (h0 < g.group) {
              part_ml[(slot * g.group + h0) * 2] = M0;
              part_ml[(slot * g.group + h0) * 2 + 1] = L0;
            }
            if (h0 + 1 < g.group) {
              part_ml[(slot * g.group + h0 + 1) * 2] = M1;
              part_ml[(slot * g.group + h0 + 1) * 2 + 1] = L1;
            }
          }
          // The unit that writes an item's last partial folds them all (no
          // separate combine launch): each unit publishes its partial, fences,
          // and counts itself in; the last one in reads the others from L2.
          __syncwarp();
          const int item = cur.seq * hkv + kvh_w;  // completion count per kv head
          const long long first = ((cur.item_start + 1) * W - 1) / total;
          const long long lastu = ((cur.item_start + cur.n_tiles) * W - 1) / total;
          const int pieces = static_cast<int>(lastu - first + 1);
          int is_last = 0;
          if (lane == 0) {
            __threadfence();
            is_last = atomicAdd(&item_done[item], 1) == pieces - 1;
            if (is_last) item_done[item] = 0;  // ready for the next launch
          }
          if (__shfl_sync(0xffffffffu, is_last, 0)) {
            __threadfence();
            const size_t base = static_cast<size_t>(cur.seq) * hkv_g + cur.kvh + static_cast<size_t>(first);
            const size_t hw = HP == 2 ? half : 0;
            __nv_bfloat16* dst = out + static_cast<size_t>(meta.q_start) * g.out_stride + kvh_w * g.group * kHD;
            for (int r = 0; r < g.group; ++r) {
              // max and denominator across the lanes (pieces strided over
              // lanes), then every lane folds its 4 dims over all pieces with
              // the loads of 4 pieces in flight at once (L2 latency, not
              // bandwidth, bounds this loop)
              float M = -INFINITY;
              for (int q = lane; q < pieces; q += 32)
                M = fmaxf(M, __ldcg(part_ml + (((base + q) * HP + hw) * g.group + r) * 2));
#pragma unroll
              for (int x = 16; x > 0; x >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, x));
              float L = 0.f;
              for (int q = lane; q < pieces; q += 32) {
                const size_t sl = ((base + q) * HP + hw) * g.group + r;
                const float ms = __ldcg(part_ml + sl * 2);
                L += ms == -INFINITY ? 0.f : __ldcg(part_ml + sl * 2 + 1) * ex2(ms - M);
              }
#pragma unroll
              for (int x = 16; x > 0; x >>= 1) L += __shfl_xor_sync(0xffffffffu, L, x);
              float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
              for (int q = 0; q < pieces; ++q) {
                const size_t sl = ((base + q) * HP + hw) * g.group + r;
                const float ms = __ldcg(part_ml + sl * 2);
                const float4 o4 = __ldcg(reinterpret_cast<const float4*>(part_o + sl * kHD) + lane);
                const float w = ms == -INFINITY ? 0.f : ex2(ms - M);
                acc.x += o4.x * w, acc.y += o4.y * w, acc.z += o4.z * w, acc.w += o4.w * w;
              }
              const float inv = L > 0.f ? 1.f / L : 0.f;
              uint2 pk;
              pk.x = pack_bf16(acc.x * inv, acc.y * inv);
              pk.y = pack_bf16(acc.z * inv, acc.w * inv);
              *reinterpret_cast<uint2*>(dst + r * kHD + lane * 4) = pk;
            }
          }
        }
      }
      pair_sync();  // staging free again (Q of the next segment lands there)
    }
    dec_advance(cur, seq_prefix, n_seq, hkv_g);
  }
}

// Page-wide decode attention (small lanes): item = sequence, all kv heads
// of a page together. A dedicated producer warp streams each 16-token page
// of the unit's tile range as ONE bulk copy of every kv head's block
// ([page][kv head][K | V] is contiguous: Hkv x 8 KB, 64 KB at 8 kv heads)
// into a 3-stage ring; consumer warp h owns kv head h (16 keys per stage)
// and finalizes it alone. One issuing thread with 32-64 KB copies and
// ~192 KB in flight is what a 32-SM lane needs to stream ~180 GB/s per SM
// (profiles/r02_bw_probe_copy_size.jsonl, r02_bw_green.jsonl).
constexpr int kPgStages = 3;
template <int NH>
struct PgCfg {
  static constexpr int kStageBytes = NH * 8192;
  static constexpr int kWarpStaging = 8 * kHD * 4;  // Q (bf16) at a segment's start, O (fp32) at its end
  static constexpr size_t kSmem =
      static_cast<size_t>(kPgStages) * kStageBytes + NH * kWarpStaging + 2 * kPgStages * 8 + 64;
};
static_assert(PgCfg<8>::kSmem <= 227u * 1024u, "page-wide decode ring exceeds 227 KB");

template <int NH>
__global__ void __launch_bounds__((NH + 1) * 32, 1)
    decode_attn_page_kernel(AttnGeom g, const __nv_bfloat16* __restrict__ qkv,
                            const __nv_bfloat16* __restrict__ kplane, const AttnSeq* __restrict__ seqs,
                            const int* __restrict__ seq_prefix, int n_seq, long long total, long long W,
                            const int32_t* __restrict__ pages, __nv_bfloat16* __restrict__ out,
                            float* __restrict__ part_o, float* __restrict__ part_ml, int* __restrict__ item_done) {
  extern __shared__ __align__(1024) uint8_t smem_pg[];
  constexpr int kStage = PgCfg<NH>::kStageBytes;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = smem_pg;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_pg + kPgStages * kStage + NH * PgCfg<NH>::kWarpStaging);
  uint64_t* empty = full + kPgStages;
  pdl_trigger();
  const long long gw = blockIdx.x;
  if (gw >= W) return;  // the whole CTA leaves together
  const long long lo = total * gw / W, hi = total * (gw + 1) / W;
  if (warp == NH && lane == 0) {
    for (int i = 0; i < kPgStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NH);
    }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();  // the new token's K/V and Q come from the QKV / RoPE kernels
  if (warp == NH) {
    // ---------------- producer: one copy per page, all kv heads ----------------
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      DecPos prod = dec_locate(seq_prefix, n_seq, 1, lo);
      int pm_seq = -1, kv_len = 0;
      const int32_t* pt = pages;
      int stage = 0;
      uint32_t phase = 0;
      for (long long t = lo; t < hi; ++t) {
        if (prod.seq != pm_seq) {
          const AttnSeq ms = seqs[prod.seq];
          pm_seq = prod.seq;
          kv_len = ms.kv_len;
          pt = pages + ms.page_off;
        }
        const int key = prod.tile * kKTD;  // < kv_len; a second page past it re-loads the first (masked)
        const int pg0 = pt[key >> 4];
        const int pg1 = key + 16 < kv_len ? pt[(key + 16) >> 4] : pg0;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], kStage);
          bulk_load(ring + stage * kStage, kplane + static_cast<size_t>(j ? pg1 : pg0) * NH * kKVBlock, kStage,
                    &full[stage], pol);
          if (++stage == kPgStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        dec_advance(prod, seq_prefix, n_seq, 1);
      }
    }
    return;
  }
  // ---------------- consumer warp: kv head h ----------------
  const int h = warp;
  float* wstage = reinterpret_cast<float*>(smem_pg + kPgStages * kStage) + h * 8 * kHD;
  __nv_bfloat16* sq = reinterpret_cast<__nv_bfloat16*>(wstage);
  const uint32_t ring_s = smem_u32(ring) + static_cast<uint32_t>(h * 8192);
  DecPos cur = dec_locate(seq_prefix, n_seq, 1, lo);
  uint32_t qb[8][2];
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  float o[8][4];
  AttnSeq meta = seqs[cur.seq];
  int seg_tile0 = cur.tile;
  const int h0 = 2 * (lane & 3);
  const int l7 = lane & 7, b3 = (lane >> 3) & 1, b4 = lane >> 4, gx = (l7 & 6) >> 1;
  uint32_t koff[4], voff[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    koff[j] = static_cast<uint32_t>(b3 * 2048 + l7 * 128 + (((b4 ^ l7) & 1) << 4) + ((j ^ gx) << 5));
    voff[j] = static_cast<uint32_t>(4096 + b4 * 2048 + l7 * 128 + (((b3 ^ l7) & 1) << 4) + ((j ^ gx) << 5));
  }
  int stage = 0;
  uint32_t phase = 0;
  for (long long gt = lo; gt < hi; ++gt) {
    if (gt == lo || cur.tile == 0) {  // new segment: this head's queries
      meta = seqs[cur.seq];
      seg_tile0 = cur.tile;
      for (int c = lane; c < 8 * 16; c += 32) {
        const int r = c >> 4, chunk = c & 15;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (r < g.group)
          v = *reinterpret_cast<const uint4*>(qkv + static_cast<size_t>(meta.q_start) * g.qkv_stride +
                                              (h * g.group + r) * kHD + chunk * 8);
        *reinterpret_cast<uint4*>(sq + r * kHD + ((chunk ^ (r & 7)) << 3)) = v;
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        uint32_t r[4];
        ldsm_x4(r, sq + swz(lane & 7, k * 16 + ((lane >> 3) << 3)));
        qb[k][0] = r[0], qb[k][1] = r[1], qb[k + 1][0] = r[2], qb[k + 1][1] = r[3];
      }
      __syncwarp();  // the staging is the O staging at the segment's end
      m0 = m1 = -INFINITY;
      l0 = l1 = 0.f;
#pragma unroll
      for (int d = 0; d < 8; ++d) o[d][0] = o[d][1] = o[d][2] = o[d][3] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      mbar_wait(&full[stage], phase);
      const uint32_t sbase = ring_s + static_cast<uint32_t>(stage * kStage);
      float sc[4][4];
#pragma unroll
      for (int c = 0; c < 4; ++c) sc[c][0] = sc[c][1] = sc[c][2] = sc[c][3] = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        uint32_t a[4];
        ldsm_x4_s(a, sbase + koff[k & 3] + ((k & 4) << 8));
        mma16816(sc[k & 3], a, qb[k][0], qb[k][1]);
      }
      float sv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) sv[q] = (sc[0][q] + sc[1][q]) + (sc[2][q] + sc[3][q]);
      const int key0 = cur.tile * kKTD + j * 16 + (lane >> 2);
      float mx0 = m0, mx1 = m1;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const bool ok = key0 + q * 8 < meta.kv_len;
        sv[2 * q] = ok ? sv[2 * q] * g.scale_log2 : -INFINITY;
        sv[2 * q + 1] = ok ? sv[2 * q + 1] * g.scale_log2 : -INFINITY;
        mx0 = fmaxf(mx0, sv[2 * q]);
        mx1 = fmaxf(mx1, sv[2 * q + 1]);
      }
#pragma unroll
      for (int x = 4; x < 32; x <<= 1) {
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffff, mx0, x));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffff, mx1, x));
      }
      const float bb0 = mx0 == -INFINITY ? 0.f : mx0, bb1 = mx1 == -INFINITY ? 0.f : mx1;
      if (__any_sync(0xffffffff, mx0 != m0 || mx1 != m1)) {
        const float al0 = ex2(m0 - bb0), al1 = ex2(m1 - bb1);
        l0 *= al0, l1 *= al1;
#pragma unroll
        for (int d = 0; d < 8; ++d) o[d][0] *= al0, o[d][2] *= al0, o[d][1] *= al1, o[d][3] *= al1;
        m0 = mx0, m1 = mx1;
      }
      const float p00 = ex2(sv[0] - bb0), p01 = ex2(sv[1] - bb1);
      const float p10 = ex2(sv[2] - bb0), p11 = ex2(sv[3] - bb1);
      l0 += p00 + p10;
      l1 += p01 + p11;
      const uint32_t pb0 = movmatrix_trans(pack_bf16(p00, p01));
      const uint32_t pb1 = movmatrix_trans(pack_bf16(p10, p11));
#pragma unroll
      for (int db = 0; db < 8; ++db) {
        uint32_t a[4];
        ldsm_x4_t_s(a, sbase + voff[db & 3] + ((db & 4) << 8));
        mma16816(o[db], a, pb0, pb1);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == kPgStages) {
        stage = 0;
        phase ^= 1;
      }
    }
    const bool item_end = cur.tile == cur.n_tiles - 1;
    if (item_end || gt == hi - 1) {
      float lt0 = l0, lt1 = l1;
#pragma unroll
      for (int x = 4; x < 32; x <<= 1) {
        lt0 += __shfl_xor_sync(0xffffffff, lt0, x);
        lt1 += __shfl_xor_sync(0xffffffff, lt1, x);
      }
      const bool whole = seg_tile0 == 0 && item_end;
      const float sa0 = whole ? (lt0 > 0.f ? 1.f / lt0 : 0.f) : 1.f;
      const float sa1 = whole ? (lt1 > 0.f ? 1.f / lt1 : 0.f) : 1.f;
#pragma unroll
      for (int d = 0; d < 8; ++d) {
        const int dim = d * 16 + (lane >> 2);
        wstage[h0 * kHD + dim] = o[d][0] * sa0;
        wstage[(h0 + 1) * kHD + dim] = o[d][1] * sa1;
        wstage[h0 * kHD + dim + 8] = o[d][2] * sa0;
        wstage[(h0 + 1) * kHD + dim + 8] = o[d][3] * sa1;
      }
      __syncwarp();
      __nv_bfloat16* dst = out + static_cast<size_t>(meta.q_start) * g.out_stride + h * g.group * kHD;
      if (whole) {
        for (int c = lane; c < g.group * 16; c += 32) {
          const float4 u = *reinterpret_cast<const float4*>(wstage + c * 8);
          const float4 v = *reinterpret_cast<const float4*>(wstage + c * 8 + 4);
          uint4 w;
          w.x = pack_bf16(u.x, u.y), w.y = pack_bf16(u.z, u.w), w.z = pack_bf16(v.x, v.y), w.w = pack_bf16(v.z, v.w);
          *reinterpret_cast<uint4*>(dst + c * 8) = w;
        }
      } else {
        // partial slot (sequence + unit) x NH + head; the unit writing a
        // head's last partial folds them (atomic count per (sequence, head))
        const size_t slot = (static_cast<size_t>(cur.seq) + static_cast<size_t>(gw)) * NH + h;
        float4* po = reinterpret_cast<float4*>(part_o + slot * g.group * kHD);
        for (int c = lane; c < g.group * 32; c += 32) po[c] = *reinterpret_cast<const float4*>(wstage + c * 4);
        if (lane < 4) {
          if (h0 < g.group) {
            part_ml[(slot * g.group + h0) * 2] = m0;
            part_ml[(slot * g.group + h0) * 2 + 1] = lt0;
          }
          if (h0 + 1 < g.group) {
            part_ml[(slot * g.group + h0 + 1) * 2] = m1;
            part_ml[(slot * g.group + h0 + 1) * 2 + 1] = lt1;
          }
        }
        __syncwarp();
        const int item = cur.seq * NH + h;
        const long long first = ((cur.item_start + 1) * W - 1) / total;
        const long long lastu = ((cur.item_start + cur.n_tiles) * W - 1) / total;
        const int pieces = static_cast<int>(lastu - first + 1);
        int is_last = 0;
        if (lane == 0) {
          __threadfence();
          is_last = atomicAdd(&item_done[item], 1) == pieces - 1;
          if (is_last) item_done[item] = 0;
        }
        if (__shfl_sync(0xffffffffu, is_last, 0)) {
          __threadfence();
          const size_t base = static_cast<size_t>(cur.seq) + static_cast<size_t>(first);
          for (int r = 0; r < g.group; ++r) {
            float M = -INFINITY;
            for (int q = lane; q < pieces; q += 32)
              M = fmaxf(M, __ldcg(part_ml + (((base + q) * NH + h) * g.group + r) * 2));
#pragma unroll
            for (int x = 16; x > 0; x >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, x));
            float L = 0.f;
            for (int q = lane; q < pieces; q += 32) {
              const size_t sl = ((base + q) * NH + h) * g.group + r;
              const float ms = __ldcg(part_ml + sl * 2);
              L += ms == -INFINITY ? 0.f : __ldcg(part_ml + sl * 2 + 1) * ex2(ms - M);
            }
#pragma unroll
            for (int x = 16; x > 0; x >>= 1) L += __shfl_xor_sync(0xffffffffu, L, x);
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
            for (int q = 0; q < pieces; ++q) {
              const size_t sl = ((base + q) * NH + h) * g.group + r;
              const float ms = __ldcg(part_ml + sl * 2);
              const float4 o4 = __ldcg(reinterpret_cast<const float4*>(part_o + sl * kHD) + lane);
              const float w = ms == -INFINITY ? 0.f : ex2(ms - M);
              acc.x += o4.x * w, acc.y += o4.y * w, acc.z += o4.z * w, acc.w += o4.w * w;
            }
            const float inv = L > 0.f ? 1.f / L : 0.f;
            uint2 pk;
            pk.x = pack_bf16(acc.x * inv, acc.y * inv);
            pk.y = pack_bf16(acc.z * inv, acc.w * inv);
            *reinterpret_cast<uint2*>(dst + r * kHD + lane * 4) = pk;
          }
        }
      }
      __syncwarp();  // staging free for the next segment's Q
    }
    dec_advance(cur, seq_prefix, n_seq, 1);
  }
}

// Items of HP kv heads: head pairs on lanes of >= 96 SMs when the kv-head
// count is even (NX_DEC_HP=1 / 2 forces one form where it applies). Measured
// (profiles/r02_attn_decode_variants_ab.jsonl, 8B): on the whole GPU head
// pairs stream short launches 15% and B = 128 x ctx 600 4% faster; on a
// 32-SM lane both forms run at ~90 GB/s per SM (every unit waits on its
// one-stage refill) and single heads are up to 5% ahead.
int decode_heads_per_item(int n_kv_heads, int sm_count) {
  static const int force = [] {
    const char* e = std::getenv("NX_DEC_HP");
    return e ? std::atoi(e) : 0;
  }();
  if (n_kv_heads % 2 != 0 || force == 1) return 1;
  return force == 2 || sm_count >= 96 ? 2 : 1;
}
}  // namespace

size_t attn_smem_bytes_dec() { return DecCfg<1>::kSmem; }

cudaError_t decode_attention(const AttnGeom& g, const __nv_bfloat16* qkv,
                             const __nv_bfloat16* kplane, const __nv_bfloat16* vplane,
                             const AttnSeq* seqs, int n_seq, const int* seq_prefix,
                             long long total_tiles, int max_seq_tiles, const int32_t* pages,
                             __nv_bfloat16* out, float* part_o, float* part_ml, size_t part_cap,
                             int* item_done, int sm_count, cudaStream_t s) {
  if (n_seq == 0 || total_tiles == 0) return cudaSuccess;
  if (g.group > 8) return cudaErrorInvalidValue;
  if (const cudaError_t pe = ensure_kernels_prepared(); pe != cudaSuccess) return pe;
  // page-wide items (one copy of all kv heads per page) whenever the kv-head
  // count is 2, 4 or 8: ahead of the pair kernels on every lane measured
  // (profiles/r02_attn_decode_variants_ab.jsonl); NX_DEC_PAGE=0 turns it off
  static const bool page_on = [] {
    const char* e = std::getenv("NX_DEC_PAGE");
    return !(e && e[0] == '0');
  }();
  const int nh = g.n_kv_heads;
  if (page_on && (nh == 2 || nh == 4 || nh == 8)) {
    static const long long kMinPg = [] {
      const char* e = std::getenv("NX_DEC_MIN_TILES");
      return e ? std::max(1, std::atoi(e)) : 4;
    }();
    const long long total_seq = total_tiles / nh;  // tiles per sequence (all heads in one item)
    const long long Wp = std::min<long long>(sm_count, std::max<long long>(1, (total_seq + kMinPg - 1) / kMinPg));
    if ((static_cast<size_t>(n_seq) + static_cast<size_t>(Wp)) * nh * g.group * kHD > part_cap)
      return cudaErrorInvalidValue;
    ++g_kernel_launches;
    const dim3 grid_p(static_cast<int>(Wp)), block_p((nh + 1) * 32);
    if (nh == 8)
      return launch_pdl(decode_attn_page_kernel<8>, grid_p, block_p, PgCfg<8>::kSmem, s, g, qkv, kplane, seqs,
                        seq_prefix, n_seq, total_seq, Wp, pages, out, part_o, part_ml, item_done);
    if (nh == 4)
      return launch_pdl(decode_attn_page_kernel<4>, grid_p, block_p, PgCfg<4>::kSmem, s, g, qkv, kplane, seqs,
                        seq_prefix, n_seq, total_seq, Wp, pages, out, part_o, part_ml, item_done);
    return launch_pdl(decode_attn_page_kernel<2>, grid_p, block_p, PgCfg<2>::kSmem, s, g, qkv, kplane, seqs,
                      seq_prefix, n_seq, total_seq, Wp, pages, out, part_o, part_ml, item_done);
  }
  const int HP = decode_heads_per_item(g.n_kv_heads, sm_count);
  const int pairs = HP == 2 ? DecCfg<2>::kPairs : DecCfg<1>::kPairs;
  const size_t smem = HP == 2 ? DecCfg<2>::kSmem : DecCfg<1>::kSmem;
  total_tiles /= HP;  // the caller counts tiles per kv head; items hold HP heads
  // >= kMinTiles tiles per unit: a launch with fewer tiles than units would
  // otherwise split every item into one-tile pieces whose in-kernel merge
  // (one warp, L2 round trips per piece) costs more than the streaming
  static const long long kMinTiles = [] {
    const char* e = std::getenv("NX_DEC_MIN_TILES");
    return e ? std::max(1, std::atoi(e)) : 4;
  }();
  const long long W = std::min<long long>(static_cast<long long>(sm_count) * pairs,
                                          std::max<long long>(1, (total_tiles + kMinTiles - 1) / kMinTiles));
  const int grid = static_cast<int>(std::min<long long>(sm_count, W));
  // compact partial slots: (item + unit) x HP heads < (n_seq * Hkv / HP + W) x
  // HP, independent of how many pieces the longest item splits into
  if ((static_cast<size_t>(n_seq) * (g.n_kv_heads / HP) + static_cast<size_t>(W)) * HP * g.group * kHD > part_cap)
    return cudaErrorInvalidValue;
  ++g_kernel_launches;
  const dim3 block(2 * pairs * 32);
  return HP == 2 ? launch_pdl(decode_attn_kernel<2>, dim3(grid), block, smem, s, g, qkv, kplane, vplane, seqs,
                              seq_prefix, n_seq, total_tiles, W, pages, out, part_o, part_ml, item_done)
                 : launch_pdl(decode_attn_kernel<1>, dim3(grid), block, smem, s, g, qkv, kplane, vplane, seqs,
                              seq_prefix, n_seq, total_tiles, W, pages, out, part_o, part_ml, item_done);
}

cudaError_t prepare_attention_kernels() {
  cudaError_t e = cudaFuncSetAttribute(decode_attn_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(DecCfg<1>::kSmem));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(decode_attn_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(DecCfg<2>::kSmem));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(decode_attn_page_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(PgCfg<8>::kSmem));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(decode_attn_page_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(PgCfg<4>::kSmem));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(decode_attn_page_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(PgCfg<2>::kSmem));
  if (e == cudaSuccess) e = prepare_prefill_attention_kernel();
  return e;
}

}  // namespace nxd
