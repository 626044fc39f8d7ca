// Paged attention over the device-resident block table.
//
// KV cache layout per layer: [page][kv_head][K | V][16][hd] bf16, written
// pre-swizzled (16 B chunk c of token row r stored at c ^ (r & 7)), so one
// (page, kv head) is a contiguous 8 KB run [K 16 x 128 | V 16 x 128] that is
// *already* the conflict-free shared-memory image: a 64-key tile is 4
// cp.async.bulk copies issued by one thread on an mbarrier. In smem, key r of
// a tile sits at row kv_row(r) = 32 (r / 16) + r % 16 of the K view and the
// same row of the V view (16 rows further). One 8 KB copy instead of two 4 KB
// ones: bulk copies pay a per-copy cost (tools/bw_probe.cu: 4 KB copies 27-55
// GB/s/SM, 16-32 KB copies 107-190 GB/s/SM).
//
//  * prefill: CTA = (sequence, kv head, 64 query rows); a query row is a
//    (token, head-in-GQA-group) pair so all G heads sharing a KV head reuse
//    each staged tile. Causal: token i sees keys [0, start + i].
//  * decode: CTA = (sequence, kv head, KV split); the G query heads of the
//    single token form the rows; 4 warps take 16-key slices of every staged
//    tile and are merged in shared memory; splits > 1 write (O, m, l)
//    partials that decode_combine() merges with a log-sum-exp rescale.
// Softmax runs in fp32 with exp2 and a per-row running max (online
// softmax); reductions are 4-lane quad shuffles.
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
constexpr int kKT = 64;         // keys per staged tile
constexpr int kRowsPF = 64;     // query rows per prefill CTA
constexpr int kThreadsAttn = 128;
constexpr int kStagesPF = 2;   // prefill: 2 x 32 KB KV stages (+16 KB Q staging)

constexpr int kKVBlock = 2 * 16 * kHD;  // elements of one (page, kv head) K|V block
// Key r of a tile of interleaved (page, kv head) blocks sits at smem row
// kv_row(r) = 32 (r / 16) + r % 16 of the K view (the V view is 16 rows on).

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

// One thread: bulk-copies the pages covering keys [key0, key0 + 64) of one
// kv head (K and V) into a tile; completion on `bar`. Pages wholly past
// kv_end are skipped (their smem keeps finite stale/zero data; masked).
__device__ __forceinline__ void issue_kv_tile(__nv_bfloat16* sk, __nv_bfloat16* sv, uint64_t* bar,
                                              const __nv_bfloat16* kplane,
                                              const __nv_bfloat16* vplane, const int32_t* pages,
                                              int kv_end, int key0, int kvh, const AttnGeom& g,
                                              uint64_t policy) {
  // Slots past kv_end re-load the last valid page: their keys are masked and
  // the data is finite, so P * V stays exact without zero-filling smem.
  const int last_page = pages[(kv_end - 1) >> 4];
  mbar_expect_tx(bar, 4 * 2 * 4096);
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int key = key0 + p * 16;
    const int page = key < kv_end ? pages[key >> 4] : last_page;
    const size_t off = (static_cast<size_t>(page) * g.n_kv_heads + kvh) * kKVBlock;
    bulk_load(sk + p * kKVBlock, kplane + off, 8192, bar, policy);  // sv = sk + 16 rows
  }
}

// One warp: 16 query rows against a 64-key tile already staged in smem.
// Updates the running max / sum and the 16 x 128 output accumulator.
template <bool kMask>
__device__ __forceinline__ void attend_tile(const uint32_t (&qf)[8][4], uint32_t sk, uint32_t sv,
                                            int key_lo, int key_hi,
                                            const int (&row_limit)[2], float (&m)[2],
                                            float (&l)[2], float (&o)[16][4], float scale_log2,
                                            int key0) {
  const int lane = threadIdx.x & 31;
  // hoisted ldmatrix lane offsets (see decode_attn_kernel): K rows 2 kb + (lane & 7) + 8 b4,
  // chunk 2 k + b3; V rows 2 ks 16 + (lane & 7) + 8 b3, chunk 2 d2 + b4
  const int l7 = lane & 7, b3 = (lane >> 3) & 1, b4 = lane >> 4, gx = (l7 & 6) >> 1;
  uint32_t koff[4], voff[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    koff[j] = static_cast<uint32_t>((l7 + 8 * b4) * kHD * 2 + (((b3 ^ l7) & 1) << 4) + ((j ^ gx) << 5));
    voff[j] = static_cast<uint32_t>((l7 + 8 * b3) * kHD * 2 + (((b4 ^ l7) & 1) << 4) + ((j ^ gx) << 5));
  }
  float s[8][4];
#pragma unroll
  for (int n = 0; n < 8; ++n)
#pragma unroll
    for (int i = 0; i < 4; ++i) s[n][i] = 0.f;
  // S = Q K^T over the warp's key slice [key_lo, key_hi) (multiple of 16).
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) {
    const int kb = n2 * 16;
    if (kb < key_lo || kb >= key_hi) continue;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      uint32_t b[4];
      ldsm_x4_s(b, sk + kb * 2 * kHD * 2 + koff[k & 3] + ((k & 4) << 5));  // kv_row(kb + y) = 2 kb + y
      mma16816(s[2 * n2], qf[k], b[0], b[1]);
      mma16816(s[2 * n2 + 1], qf[k], b[2], b[3]);
    }
  }
  // mask + running max
  float mx[2] = {m[0], m[1]};
#pragma unroll
  for (int n = 0; n < 8; ++n) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int key = key0 + n * 8 + (lane & 3) * 2 + (i & 1);
      const int r = i >> 1;
      const bool in_slice = (n * 8 >= key_lo) && (n * 8 < key_hi);
      if (!in_slice || (kMask && key > row_limit[r])) s[n][i] = -INFINITY;
      else s[n][i] *= scale_log2;
      mx[r] = fmaxf(mx[r], s[n][i]);
    }
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffff, mx[r], 1));
    mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffff, mx[r], 2));
  }
  float base[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) base[r] = mx[r] == -INFINITY ? 0.f : mx[r];
  if (__any_sync(0xffffffff, mx[0] != m[0] || mx[1] != m[1])) {  // a running max moved: rescale
    float alpha[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      alpha[r] = ex2(m[r] - base[r]);
      m[r] = mx[r];
      l[r] *= alpha[r];
    }
#pragma unroll
    for (int d = 0; d < 16; ++d) {
      o[d][0] *= alpha[0];
      o[d][1] *= alpha[0];
      o[d][2] *= alpha[1];
      o[d][3] *= alpha[1];
    }
  }
  uint32_t pf[4][4];  // P as A fragments, one per 16-key step
#pragma unroll
  for (int n = 0; n < 8; ++n) {
    float p[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      p[i] = ex2(s[n][i] - base[i >> 1]);
      l[i >> 1] += p[i];
    }
    const int ks = n >> 1;
    if ((n & 1) == 0) {
      pf[ks][0] = pack_bf16(p[0], p[1]);
      pf[ks][1] = pack_bf16(p[2], p[3]);
    } else {
      pf[ks][2] = pack_bf16(p[0], p[1]);
      pf[ks][3] = pack_bf16(p[2], p[3]);
    }
  }
  // O += P V
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    if (ks * 16 < key_lo || ks * 16 >= key_hi) continue;
#pragma unroll
    for (int d2 = 0; d2 < 8; ++d2) {
      uint32_t b[4];
      ldsm_x4_t_s(b, sv + ks * 32 * kHD * 2 + voff[d2 & 3] + ((d2 & 4) << 5));
      mma16816(o[2 * d2], pf[ks], b[0], b[1]);
      mma16816(o[2 * d2 + 1], pf[ks], b[2], b[3]);
    }
  }
}

// Loads a warp's 16 query rows (row r -> token r / G, head r % G) as A
// fragments straight from global memory; padded rows are zero.
__device__ __forceinline__ void load_q_frag(uint32_t (&qf)[8][4], const __nv_bfloat16* qkv,
                                            const AttnGeom& g, int tok_base, int n_tok,
                                            int row0, int kvh, __nv_bfloat16* stage) {
  const int lane = threadIdx.x & 31;
  // stage 16 x 128 into (swizzled) smem via 16 B loads, then ldmatrix. Lane l
  // covers chunk l & 15 of rows (l >> 4) + 2 i; all 8 loads are issued before
  // the first store, and (token, head) of row r advance incrementally (a
  // per-element division by the group size was 8% of the kernel's instructions).
  const int chunk = lane & 15;
  int gr = row0 + (lane >> 4);
  int t = gr / g.group, hd = gr - t * g.group;
  uint4 v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    v[i] = t < n_tok ? *reinterpret_cast<const uint4*>(qkv + static_cast<size_t>(tok_base + t) * g.qkv_stride +
                                                        (kvh * g.group + hd) * kHD + chunk * 8)
                     : make_uint4(0, 0, 0, 0);
    hd += 2;
    while (hd >= g.group) hd -= g.group, ++t;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = (lane >> 4) + 2 * i;
    *reinterpret_cast<uint4*>(stage + r * kHD + ((chunk ^ (r & 7)) << 3)) = v[i];
  }
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int row = (lane & 7) + (((lane >> 3) & 1) << 3);
    const int col = k * 16 + ((lane >> 4) << 3);
    ldsm_x4(qf[k], stage + swz(row, col));
  }
}

__global__ void __launch_bounds__(kThreadsAttn)
    prefill_attn_kernel(AttnGeom g, const __nv_bfloat16* __restrict__ qkv,
                        const __nv_bfloat16* __restrict__ kplane,
                        const __nv_bfloat16* __restrict__ vplane, const AttnSeq* __restrict__ seqs,
                        const int2* __restrict__ work, const int32_t* __restrict__ pages,
                        __nv_bfloat16* __restrict__ out) {
  extern __shared__ __align__(1024) uint8_t smem_attn[];
  constexpr int S = kStagesPF;
  // [S][4 blocks][K 16 | V 16][128]: K view at the stage base, V view 16 rows on
  __nv_bfloat16* sk = reinterpret_cast<__nv_bfloat16*>(smem_attn);
  __nv_bfloat16* sv = sk + 16 * kHD;
  const uint32_t sk_s = smem_u32(sk), sv_s = smem_u32(sv);
  __nv_bfloat16* sq = sk + S * 2 * kKT * kHD;                        // [4 warps][16][128]
  uint64_t* full = reinterpret_cast<uint64_t*>(sq + 4 * 16 * kHD);
  pdl_trigger();
  const int2 wi = work[blockIdx.x];
  const AttnSeq sq_meta = seqs[wi.x];
  const int kvh = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row0 = wi.y + warp * 16;  // first query row of this warp
  const int start = sq_meta.kv_len - sq_meta.q_len;
  const int32_t* pt = pages + sq_meta.page_off;
  const int last_tok = min(sq_meta.q_len - 1, (wi.y + kRowsPF - 1) / g.group);
  const int kv_end = start + last_tok + 1;  // keys needed by this CTA
  const int n_tiles = (kv_end + kKT - 1) / kKT;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();  // K/V of this chunk and Q come from the QKV / RoPE kernels
  const uint64_t pol = policy_evict_first();
  if (threadIdx.x == 0)
    for (int t = 0; t < S && t < n_tiles; ++t)
      issue_kv_tile(sk + t * 2 * kKT * kHD, sv + t * 2 * kKT * kHD, &full[t], kplane, vplane, pt, kv_end,
                    t * kKT, kvh, g, pol);

  uint32_t qf[8][4];
  load_q_frag(qf, qkv, g, sq_meta.q_start, sq_meta.q_len, row0, kvh, sq + warp * 16 * kHD);
  int row_limit[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int gr = row0 + (lane >> 2) + r * 8;
    row_limit[r] = start + gr / g.group;  // causal: keys <= own position
  }
  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
  float o[16][4];
#pragma unroll
  for (int d = 0; d < 16; ++d)
#pragma unroll
    for (int i = 0; i < 4; ++i) o[d][i] = 0.f;

  for (int t = 0; t < n_tiles; ++t) {
    const int buf = t % S;
    mbar_wait(&full[buf], (t / S) & 1);
    // tiles wholly below the CTA's first causal limit skip the mask math
    if (t * kKT + kKT - 1 <= start + wi.y / g.group)
      attend_tile<false>(qf, sk_s + buf * 2 * kKT * kHD * 2, sv_s + buf * 2 * kKT * kHD * 2, 0, kKT, row_limit, m,
                         l, o, g.scale_log2, t * kKT);
    else
      attend_tile<true>(qf, sk_s + buf * 2 * kKT * kHD * 2, sv_s + buf * 2 * kKT * kHD * 2, 0, kKT, row_limit, m, l,
                        o, g.scale_log2, t * kKT);
    __syncthreads();  // every warp is done with buf
    if (threadIdx.x == 0 && t + S < n_tiles)
      issue_kv_tile(sk + buf * 2 * kKT * kHD, sv + buf * 2 * kKT * kHD, &full[buf], kplane, vplane, pt,
                    kv_end, (t + S) * kKT, kvh, g, pol);
  }
  // normalize + store
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l[r] += __shfl_xor_sync(0xffffffff, l[r], 1);
    l[r] += __shfl_xor_sync(0xffffffff, l[r], 2);
  }
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int gr = row0 + (lane >> 2) + r * 8;
    const int tk = gr / g.group;
    if (tk >= sq_meta.q_len) continue;
    const int head = kvh * g.group + gr % g.group;
    const float inv = l[r] > 0.f ? 1.f / l[r] : 0.f;
    __nv_bfloat16* dst =
        out + static_cast<size_t>(sq_meta.q_start + tk) * g.out_stride + head * kHD;
#pragma unroll
    for (int d = 0; d < 16; ++d) {
      const int col = d * 8 + (lane & 3) * 2;
      *reinterpret_cast<uint32_t*>(dst + col) = pack_bf16(o[d][2 * r] * inv, o[d][2 * r + 1] * inv);
    }
  }
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
// that decode_combine_kernel folds with a log-sum-exp rescale.
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
constexpr int kWarpsD = 2 * kPairsD;
constexpr int kTileD = kKTD * kHD;  // elements per K (or V) tile
// named barrier 1 + pair must stay below the 16 hardware barriers; the ring,
// the fp32 staging and the barriers must fit one SM's 227 KB opt-in
static_assert(kPairsD >= 1 && kPairsD <= 15, "NX_DEC_PAIRS must be in [1, 15]");
static_assert(kStD >= 1, "NX_DEC_STAGES must be >= 1");
static_assert(static_cast<size_t>(kPairsD) * (kStD * 2 * kTileD + 2 * 8 * kHD * 2) * 2 + 2 * kPairsD * kStD * 8 +
                      kPairsD * 32 * 4 + 64 <= 227u * 1024u,
              "NX_DEC_PAIRS x NX_DEC_STAGES exceeds 227 KB of shared memory");


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

__global__ void __launch_bounds__(kWarpsD * 32, 1)
    decode_attn_kernel(AttnGeom g, const __nv_bfloat16* __restrict__ qkv,
                       const __nv_bfloat16* __restrict__ kplane,
                       const __nv_bfloat16* __restrict__ vplane, const AttnSeq* __restrict__ seqs,
                       const int* __restrict__ seq_prefix, int n_seq, long long total, long long W,
                       const int32_t* __restrict__ pages,
                       __nv_bfloat16* __restrict__ out, float* __restrict__ part_o,
                       float* __restrict__ part_ml) {
  extern __shared__ __align__(1024) uint8_t smem_attn[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pair = warp >> 1, half = warp & 1;
  // per pair: [kStD][K tile][V tile] + 2 x [8][128] fp32 staging (warp 0's
  // doubles as the Q staging) + kStD barriers
  constexpr int kPairElems = kStD * 2 * kTileD + 2 * 8 * kHD * 2;  // bf16 units
  __nv_bfloat16* pbase = reinterpret_cast<__nv_bfloat16*>(smem_attn) + pair * kPairElems;
  const uint32_t pbase_s = smem_u32(pbase);
  __nv_bfloat16* sq = pbase + kStD * 2 * kTileD;           // Q staging [8][128] bf16 (= stage_a)
  float* stage_a = reinterpret_cast<float*>(sq);            // [8][128] fp32, warp 0
  float* stage_b = stage_a + 8 * kHD;                       // [8][128] fp32, warp 1
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<__nv_bfloat16*>(smem_attn) +
                                               kPairsD * kPairElems) + pair * kStD;
  // empty[s]: both warps of the pair are done reading stage s (2 arrivals); only
  // the producer waits on it, so neither warp stalls on the other per tile
  uint64_t* empty = full + kPairsD * kStD;
  float* ml_b = reinterpret_cast<float*>(full + 2 * kPairsD * kStD - pair * kStD) + pair * 32;  // [8 heads][m, l]
  const uint32_t bar_id = 1 + pair;
  auto pair_sync = [&] { named_bar_sync(bar_id, 64); };
  pdl_trigger();
  const long long gw = static_cast<long long>(blockIdx.x) * kPairsD + pair;
  if (gw >= W) return;  // both warps of the pair leave together
  const long long lo = total * gw / W, hi = total * (gw + 1) / W;
  const int hkv = g.n_kv_heads;
  const bool producer = half == 0 && lane == 0;
  if (producer) {
    for (int i = 0; i < kStD; ++i) {
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
  DecPos prod = dec_locate(seq_prefix, n_seq, hkv, lo);
  long long issued = lo;
  int nxt_pg0 = 0, nxt_pg1 = 0, nxt_kvh = 0;
  auto lookup = [&]() {
    const AttnSeq ms = seqs[prod.seq];
    const int32_t* pt = pages + ms.page_off;
    const int last = pt[(ms.kv_len - 1) >> 4];  // keys past kv_len re-load it (masked, finite)
    const int key = prod.tile * kKTD;
    nxt_pg0 = key < ms.kv_len ? pt[key >> 4] : last;
    nxt_pg1 = key + 16 < ms.kv_len ? pt[(key + 16) >> 4] : last;
    nxt_kvh = prod.kvh;
  };
  auto issue = [&](int st) {
    __nv_bfloat16* dst = pbase + st * 2 * kTileD;
    mbar_expect_tx(&full[st], 2 * 2 * 4096);
    bulk_load(dst, kplane + (static_cast<size_t>(nxt_pg0) * hkv + nxt_kvh) * kKVBlock, 8192, &full[st], pol);
    bulk_load(dst + kKVBlock, kplane + (static_cast<size_t>(nxt_pg1) * hkv + nxt_kvh) * kKVBlock, 8192, &full[st],
              pol);
  };
  if (producer) {
    for (; issued < hi && issued < lo + kStD; ++issued) {
      lookup();
      issue(static_cast<int>(issued - lo));
      dec_advance(prod, seq_prefix, n_seq, hkv);
    }
    if (issued < hi) lookup();
  }
  DecPos cur = dec_locate(seq_prefix, n_seq, hkv, lo);
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
  const int krow = half * 16;  // this warp's 16 keys of every tile
  // ldmatrix lane addresses, hoisted: in the 128B-swizzled rows, chunk (2 k + b)
  // of a row r sits at ((2 k + b) ^ (r & 7)) << 4 = (b ^ (r & 1)) << 4 | ((k ^ g) << 5)
  // with g = (r & 6) >> 1, so 4 per-lane bases cover k = 0..7 (k & 4 is an
  // immediate +128 B). K: row 2 krow + (lane & 7) + 8 b3, chunk b = lane >> 4;
  // V (trans): row 2 krow + (lane & 7) + 8 (lane >> 4), chunk b = b3.
  const int l7 = lane & 7, b3 = (lane >> 3) & 1, b4 = lane >> 4, gx = (l7 & 6) >> 1;
  uint32_t koff[4], voff[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    koff[j] = static_cast<uint32_t>((2 * krow + l7 + 8 * b3) * kHD * 2 + (((b4 ^ l7) & 1) << 4) + ((j ^ gx) << 5));
    voff[j] = static_cast<uint32_t>((2 * krow + l7 + 8 * b4) * kHD * 2 + 16 * kHD * 2 + (((b3 ^ l7) & 1) << 4) +
                                    ((j ^ gx) << 5));
  }
  for (long long gt = lo; gt < hi; ++gt) {
    const int i = static_cast<int>(gt - lo), buf = i % kStD;
    if (gt == lo || cur.tile == 0) {  // new segment: this item's queries
      meta = seqs[cur.seq];
      seg_tile0 = cur.tile;
      for (int c = half * 32 + lane; c < 8 * 16; c += 64) {
        const int r = c >> 4, chunk = c & 15;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (r < g.group)
          v = *reinterpret_cast<const uint4*>(qkv + static_cast<size_t>(meta.q_start) * g.qkv_stride +
                                              (cur.kvh * g.group + r) * kHD + chunk * 8);
        *reinterpret_cast<uint4*>(sq + r * kHD + ((chunk ^ (r & 7)) << 3)) = v;
      }
      pair_sync();
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        uint32_t r[4];
        ldsm_x4(r, sq + swz(lane & 7, k * 16 + ((lane >> 3) << 3)));
        qb[k][0] = r[0], qb[k][1] = r[1], qb[k + 1][0] = r[2], qb[k + 1][1] = r[3];
      }
      m0 = m1 = -INFINITY;
      l0 = l1 = 0.f;
#pragma unroll
      for (int d = 0; d < 8; ++d) o[d][0] = o[d][1] = o[d][2] = o[d][3] = 0.f;
    }
    mbar_wait(&full[buf], (i / kStD) & 1);
    // [2 blocks][K 16 | V 16][128]; shared-window byte address of the stage
    const uint32_t sbase = pbase_s + static_cast<uint32_t>(buf * 2 * kTileD * 2);
    // S^T = K Q^T over this warp's 16 keys: 8 k-steps in two chains
    // four independent accumulation chains of two MMAs (HMMA latency, not issue, bounds a chain)
    float sc[4][4];
#pragma unroll
    for (int c = 0; c < 4; ++c) sc[c][0] = sc[c][1] = sc[c][2] = sc[c][3] = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      uint32_t a[4];
      ldsm_x4_s(a, sbase + koff[k & 3] + ((k & 4) << 5));
      mma16816(sc[k & 3], a, qb[k][0], qb[k][1]);
    }
    float s[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) s[j] = (sc[0][j] + sc[1][j]) + (sc[2][j] + sc[3][j]);
    // mask keys past kv_len; online softmax down each head column
    const int key0 = cur.tile * kKTD + krow + (lane >> 2);
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
      ldsm_x4_t_s(a, sbase + voff[db & 3] + ((db & 4) << 5));
      mma16816(o[db], a, pb0, pb1);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[buf]);  // this warp is done with stage buf
    // refill this stage kStD tiles ahead, once both warps released it
    if (producer && issued < hi) {
      mbar_wait(&empty[buf], static_cast<uint32_t>((i / kStD) & 1));
      issue(buf);
      dec_advance(prod, seq_prefix, n_seq, hkv);
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
      // merge the pair: warp 1 publishes (m, l, O), warp 0 folds
      if (half == 1) {
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
      pair_sync();
      if (half == 0) {
        const float mb0 = ml_b[h0 * 2], lb0 = ml_b[h0 * 2 + 1];
        const float mb1 = ml_b[(h0 + 1) * 2], lb1 = ml_b[(h0 + 1) * 2 + 1];
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
          stage_a[h0 * kHD + dim] = o[d][0] * sa0 + stage_b[h0 * kHD + dim] * sb0;
          stage_a[(h0 + 1) * kHD + dim] = o[d][1] * sa1 + stage_b[(h0 + 1) * kHD + dim] * sb1;
          stage_a[h0 * kHD + dim + 8] = o[d][2] * sa0 + stage_b[h0 * kHD + dim + 8] * sb0;
          stage_a[(h0 + 1) * kHD + dim + 8] = o[d][3] * sa1 + stage_b[(h0 + 1) * kHD + dim + 8] * sb1;
        }
        __syncwarp();
        if (whole) {
          __nv_bfloat16* dst = out + static_cast<size_t>(meta.q_start) * g.out_stride + cur.kvh * g.group * kHD;
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
          // per (item, unit) and below n_items + W (the combine reads item + first + q)
          const size_t slot = static_cast<size_t>(cur.seq) * hkv + cur.kvh + static_cast<size_t>(gw);
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
        }
      }
      pair_sync();  // staging free again (Q of the next segment lands in stage_a)
    }
    dec_advance(cur, seq_prefix, n_seq, hkv);
  }
}

// Folds the pieces of items split across warps:
// out = sum_p 2^(m_p - M) O_p / sum_p 2^(m_p - M) l_p. CTA = (item, query
// head), thread = head dim; items covered by a single warp are skipped.
__global__ void decode_combine_kernel(AttnGeom g, const AttnSeq* __restrict__ seqs,
                                      const int* __restrict__ seq_prefix, long long total, long long W,
                                      const float* __restrict__ part_o,
                                      const float* __restrict__ part_ml, __nv_bfloat16* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int item = blockIdx.x, r = blockIdx.y, d = threadIdx.x;
  const int hkv = g.n_kv_heads;
  const int seq = item / hkv, kvh = item % hkv;
  const int n_tiles = seq_prefix[seq + 1] - seq_prefix[seq];
  const long long s0 = static_cast<long long>(seq_prefix[seq]) * hkv + static_cast<long long>(kvh) * n_tiles;
  const long long first = ((s0 + 1) * W - 1) / total;
  const long long last = ((s0 + n_tiles) * W - 1) / total;
  const int pieces = static_cast<int>(last - first + 1);
  if (pieces <= 1) return;
  const size_t slot0 = (static_cast<size_t>(item) + static_cast<size_t>(first)) * g.group + r;
  float M = -INFINITY;
  for (int q = 0; q < pieces; ++q) M = fmaxf(M, part_ml[(slot0 + static_cast<size_t>(q) * g.group) * 2]);
  float acc = 0.f, L = 0.f;
  for (int q = 0; q < pieces; ++q) {
    const size_t slot = slot0 + static_cast<size_t>(q) * g.group;
    const float ms = part_ml[slot * 2];
    const float w = ms == -INFINITY ? 0.f : ex2(ms - M);
    L += part_ml[slot * 2 + 1] * w;
    acc += part_o[slot * kHD + d] * w;
  }
  out[static_cast<size_t>(seqs[seq].q_start) * g.out_stride + (kvh * g.group + r) * kHD + d] =
      __float2bfloat16(L > 0.f ? acc / L : 0.f);
}


// Decode, page-major variant: a CTA of Hkv warps (warp w = kv head w) streams
// whole pages of one sequence -- [page][kv head][K | V] makes a page of all
// kv heads one contiguous Hkv x 8 KB block, so every stage is a single
// 64 KB cp.async.bulk (bulk copies pay a per-copy cost: 4-8 KB copies cap a
// warp-pair ring at ~55-60 GB/s/SM, tools/bw_probe.cu). Unit u of the
// persistent grid owns the 32-key tiles [u T / W, (u + 1) T / W) of the
// sequence-major tile list (T = seq_prefix[n_seq]); a tile is two page
// stages. Per warp and stage the math is the transposed 16-key step of the
// pair kernel (S^T = K Q^T, O^T += V^T P^T). A sequence covered by one unit
// is finalized in place; otherwise units write (m, l, O) partials per kv head
// and decode_combine_pages_kernel folds them.
constexpr int kStPg = 3;  // page stages per CTA ring

__global__ void __launch_bounds__(8 * 32, 1)
    decode_attn_pages_kernel(AttnGeom g, const __nv_bfloat16* __restrict__ qkv,
                             const __nv_bfloat16* __restrict__ kvbase, const AttnSeq* __restrict__ seqs,
                             const int* __restrict__ seq_prefix, int n_seq, long long total, long long W,
                             const int32_t* __restrict__ pages, __nv_bfloat16* __restrict__ out,
                             float* __restrict__ part_o, float* __restrict__ part_ml) {
  extern __shared__ __align__(1024) uint8_t smem_attn[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hkv = g.n_kv_heads;
  const int stage_elems = hkv * kKVBlock;
  __nv_bfloat16* ring = reinterpret_cast<__nv_bfloat16*>(smem_attn);
  const uint32_t ring_s = smem_u32(ring);
  float* wstage = reinterpret_cast<float*>(ring + kStPg * stage_elems) + warp * 8 * kHD;  // [8][128] fp32
  __nv_bfloat16* sq = reinterpret_cast<__nv_bfloat16*>(wstage);                           // Q staging [8][128]
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<float*>(ring + kStPg * stage_elems) + hkv * 8 * kHD);
  pdl_trigger();
  const long long u = blockIdx.x;
  if (u >= W) return;
  const long long lo = total * u / W, hi = total * (u + 1) / W;  // 32-key tiles
  const bool producer = threadIdx.x == 0;
  if (producer) {
    for (int i = 0; i < kStPg; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();  // the new token's K/V and Q come from the QKV / RoPE kernels
  const uint64_t pol = policy_evict_first();
  const uint32_t stage_bytes = static_cast<uint32_t>(stage_elems) * 2;
  // tile gt -> (sequence, tile within it): the unit's first tile by binary search
  auto locate = [&](long long gt, int& seq) {
    int a = 0, b = n_seq - 1;
    while (a < b) {
      const int mid = (a + b + 1) >> 1;
      if (seq_prefix[mid] <= gt) a = mid;
      else b = mid - 1;
    }
    seq = a;
  };
  // producer: stage j of the range = page (j & 1) of tile lo + j / 2
  int pseq = 0;
  locate(lo, pseq);
  const long long n_stages = 2 * (hi - lo);
  long long issued = 0;
  auto issue = [&](long long j) {
    const long long gt = lo + j / 2;
    while (pseq + 1 < n_seq && seq_prefix[pseq + 1] <= gt) ++pseq;
    const AttnSeq ms = seqs[pseq];
    const int key = static_cast<int>(gt - seq_prefix[pseq]) * kKTD + static_cast<int>(j & 1) * 16;
    const int32_t* pt = pages + ms.page_off;
    // keys past kv_len re-load the last valid page: masked, finite data
    const int page = key < ms.kv_len ? pt[key >> 4] : pt[(ms.kv_len - 1) >> 4];
    const int st = static_cast<int>(j % kStPg);
    mbar_expect_tx(&full[st], stage_bytes);
    bulk_load(ring + st * stage_elems, kvbase + static_cast<size_t>(page) * stage_elems, stage_bytes, &full[st],
              pol);
  };
  if (producer)
    for (; issued < n_stages && issued < kStPg; ++issued) issue(issued);

  const bool live = warp < hkv;
  uint32_t qb[8][2];
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  float o[8][4];
  const int h0 = 2 * (lane & 3);
  int seq = 0;
  locate(lo, seq);
  AttnSeq meta = seqs[seq];
  long long seg_tile0 = lo;
  for (long long j = 0; j < n_stages; ++j) {
    const long long gt = lo + j / 2;
    const int half = static_cast<int>(j & 1);
    if (j == 0 || (half == 0 && gt == seq_prefix[seq + 1])) {  // new segment (sequence)
      if (j > 0) ++seq;
      meta = seqs[seq];
      seg_tile0 = gt;
      if (live) {
        for (int c = lane; c < 8 * 16; c += 32) {
          const int r = c >> 4, chunk = c & 15;
          uint4 v = make_uint4(0, 0, 0, 0);
          if (r < g.group)
            v = *reinterpret_cast<const uint4*>(qkv + static_cast<size_t>(meta.q_start) * g.qkv_stride +
                                                (warp * g.group + r) * kHD + chunk * 8);
          *reinterpret_cast<uint4*>(sq + r * kHD + ((chunk ^ (r & 7)) << 3)) = v;
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
          uint32_t r[4];
          ldsm_x4(r, sq + swz(lane & 7, k * 16 + ((lane >> 3) << 3)));
          qb[k][0] = r[0], qb[k][1] = r[1], qb[k + 1][0] = r[2], qb[k + 1][1] = r[3];
        }
        m0 = m1 = -INFINITY;
        l0 = l1 = 0.f;
#pragma unroll
        for (int d = 0; d < 8; ++d) o[d][0] = o[d][1] = o[d][2] = o[d][3] = 0.f;
      }
    }
    const int st = static_cast<int>(j % kStPg);
    mbar_wait(&full[st], static_cast<uint32_t>((j / kStPg) & 1));
    const int key0 = static_cast<int>(gt - seq_prefix[seq]) * kKTD + half * 16;
    if (live && key0 < meta.kv_len) {
      const uint32_t sk = ring_s + static_cast<uint32_t>((st * stage_elems + warp * kKVBlock) * 2);  // [K 16 | V 16]
      const uint32_t sv = sk + 16 * kHD * 2;
      float s[4] = {0.f, 0.f, 0.f, 0.f}, s2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        uint32_t a[4];
        ldsm_x4_s(a, sk + 2 * swz((lane & 7) + (((lane >> 3) & 1) << 3), k * 16 + ((lane >> 4) << 3)));
        mma16816((k & 1) ? s2 : s, a, qb[k][0], qb[k][1]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) s[i] += s2[i];
      const int kq = key0 + (lane >> 2);
      float mx0 = m0, mx1 = m1;
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        const bool ok = kq + jj * 8 < meta.kv_len;
        s[2 * jj] = ok ? s[2 * jj] * g.scale_log2 : -INFINITY;
        s[2 * jj + 1] = ok ? s[2 * jj + 1] * g.scale_log2 : -INFINITY;
        mx0 = fmaxf(mx0, s[2 * jj]);
        mx1 = fmaxf(mx1, s[2 * jj + 1]);
      }
#pragma unroll
      for (int x = 4; x < 32; x <<= 1) {
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffff, mx0, x));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffff, mx1, x));
      }
      const float b0 = mx0 == -INFINITY ? 0.f : mx0, b1 = mx1 == -INFINITY ? 0.f : mx1;
      if (__any_sync(0xffffffff, mx0 != m0 || mx1 != m1)) {
        const float al0 = ex2(m0 - b0), al1 = ex2(m1 - b1);
        l0 *= al0, l1 *= al1;
#pragma unroll
        for (int d = 0; d < 8; ++d) o[d][0] *= al0, o[d][2] *= al0, o[d][1] *= al1, o[d][3] *= al1;
        m0 = mx0, m1 = mx1;
      }
      const float p00 = ex2(s[0] - b0), p01 = ex2(s[1] - b1);
      const float p10 = ex2(s[2] - b0), p11 = ex2(s[3] - b1);
      l0 += p00 + p10;
      l1 += p01 + p11;
      const uint32_t pb0 = movmatrix_trans(pack_bf16(p00, p01));
      const uint32_t pb1 = movmatrix_trans(pack_bf16(p10, p11));
#pragma unroll
      for (int db = 0; db < 8; ++db) {
        uint32_t a[4];
        ldsm_x4_t_s(a, sv + 2 * swz((lane & 7) + ((lane >> 4) << 3), db * 16 + (((lane >> 3) & 1) << 3)));
        mma16816(o[db], a, pb0, pb1);
      }
    }
    __syncthreads();  // every warp is done with stage st
    if (producer && issued < n_stages) issue(issued++);
    // segment end: last stage of the sequence or of the unit's range
    const bool seq_end = half == 1 && gt + 1 == seq_prefix[seq + 1];
    if (live && (seq_end || j == n_stages - 1)) {
      float lt0 = l0, lt1 = l1;
#pragma unroll
      for (int x = 4; x < 32; x <<= 1) {
        lt0 += __shfl_xor_sync(0xffffffff, lt0, x);
        lt1 += __shfl_xor_sync(0xffffffff, lt1, x);
      }
      const bool whole = seg_tile0 == seq_prefix[seq] && seq_end;
      const float sc0 = whole ? (lt0 > 0.f ? 1.f / lt0 : 0.f) : 1.f;
      const float sc1 = whole ? (lt1 > 0.f ? 1.f / lt1 : 0.f) : 1.f;
      __syncwarp();
#pragma unroll
      for (int d = 0; d < 8; ++d) {
        const int dim = d * 16 + (lane >> 2);
        wstage[h0 * kHD + dim] = o[d][0] * sc0;
        wstage[(h0 + 1) * kHD + dim] = o[d][1] * sc1;
        wstage[h0 * kHD + dim + 8] = o[d][2] * sc0;
        wstage[(h0 + 1) * kHD + dim + 8] = o[d][3] * sc1;
      }
      __syncwarp();
      if (whole) {
        __nv_bfloat16* dst = out + static_cast<size_t>(meta.q_start) * g.out_stride + warp * g.group * kHD;
        for (int c = lane; c < g.group * 16; c += 32) {
          const float4 a = *reinterpret_cast<const float4*>(wstage + c * 8);
          const float4 b = *reinterpret_cast<const float4*>(wstage + c * 8 + 4);
          uint4 w;
          w.x = pack_bf16(a.x, a.y), w.y = pack_bf16(a.z, a.w), w.z = pack_bf16(b.x, b.y), w.w = pack_bf16(b.z, b.w);
          *reinterpret_cast<uint4*>(dst + c * 8) = w;
        }
      } else {
        // compact slot (sequence + unit) x kv head, unique as in the pair kernel
        const size_t slot = (static_cast<size_t>(seq) + static_cast<size_t>(u)) * hkv + warp;
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
      }
      __syncwarp();  // the staging holds the next segment's Q next
    }
  }
}

// Folds the unit pieces of sequences split across units (page-major
// decode): CTA = (sequence, kv head, query head), thread = head dim.
__global__ void decode_combine_pages_kernel(AttnGeom g, const AttnSeq* __restrict__ seqs,
                                            const int* __restrict__ seq_prefix, long long total, long long W,
                                            const float* __restrict__ part_o,
                                            const float* __restrict__ part_ml, __nv_bfloat16* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int item = blockIdx.x, r = blockIdx.y, d = threadIdx.x;
  const int hkv = g.n_kv_heads;
  const int seq = item / hkv, kvh = item % hkv;
  const long long t0 = seq_prefix[seq], t1 = seq_prefix[seq + 1];
  const long long first = ((t0 + 1) * W - 1) / total;
  const long long last = (t1 * W - 1) / total;
  const int pieces = static_cast<int>(last - first + 1);
  if (pieces <= 1) return;
  const size_t slot0 = ((static_cast<size_t>(seq) + static_cast<size_t>(first)) * hkv + kvh) * g.group + r;
  float M = -INFINITY;
  for (int q = 0; q < pieces; ++q) M = fmaxf(M, part_ml[(slot0 + static_cast<size_t>(q) * hkv * g.group) * 2]);
  float acc = 0.f, L = 0.f;
  for (int q = 0; q < pieces; ++q) {
    const size_t slot = slot0 + static_cast<size_t>(q) * hkv * g.group;
    const float ms = part_ml[slot * 2];
    const float w = ms == -INFINITY ? 0.f : ex2(ms - M);
    L += part_ml[slot * 2 + 1] * w;
    acc += part_o[slot * kHD + d] * w;
  }
  out[static_cast<size_t>(seqs[seq].q_start) * g.out_stride + (kvh * g.group + r) * kHD + d] =
      __float2bfloat16(L > 0.f ? acc / L : 0.f);
}

}  // namespace

size_t attn_smem_bytes_pf() {
  return static_cast<size_t>(2 * kStagesPF * kKT * kHD + 4 * 16 * kHD) * 2 + 64;
}
size_t attn_smem_bytes_dec() {
  return static_cast<size_t>(kPairsD) * (kStD * 2 * kTileD + 2 * 8 * kHD * 2) * 2 + 2 * kPairsD * kStD * 8 +
         kPairsD * 32 * 4 + 64;
}
size_t attn_smem_bytes_dec_pages(int hkv) {
  return static_cast<size_t>(kStPg) * hkv * kKVBlock * 2 + static_cast<size_t>(hkv) * 8 * kHD * 4 + kStPg * 8 + 64;
}
size_t attn_smem_bytes() { return std::max(attn_smem_bytes_pf(), attn_smem_bytes_dec()); }

cudaError_t prefill_attention(const AttnGeom& g, const __nv_bfloat16* qkv,
                              const __nv_bfloat16* kplane, const __nv_bfloat16* vplane,
                              const AttnSeq* seqs, const int2* work, int n_work,
                              const int32_t* pages, __nv_bfloat16* out, cudaStream_t s) {
  if (n_work == 0) return cudaSuccess;
  if (const cudaError_t pe = ensure_kernels_prepared(); pe != cudaSuccess) return pe;
  const size_t smem = attn_smem_bytes_pf();
  ++g_kernel_launches;
  return launch_pdl(prefill_attn_kernel, dim3(n_work, g.n_kv_heads), dim3(kThreadsAttn), smem, s, g, qkv,
                    kplane, vplane, seqs, work, pages, out);
}

cudaError_t decode_attention(const AttnGeom& g, const __nv_bfloat16* qkv,
                             const __nv_bfloat16* kplane, const __nv_bfloat16* vplane,
                             const AttnSeq* seqs, int n_seq, const int* seq_prefix,
                             long long total_tiles, int max_seq_tiles, const int32_t* pages,
                             __nv_bfloat16* out, float* part_o, float* part_ml, size_t part_cap,
                             int sm_count, cudaStream_t s) {
  if (n_seq == 0 || total_tiles == 0) return cudaSuccess;
  if (g.group > 8) return cudaErrorInvalidValue;
  if (const cudaError_t pe = ensure_kernels_prepared(); pe != cudaSuccess) return pe;
  // NX_DEC_ATTN=pages: the page-major variant (64 KB copies; measured ~4%
  // slower than the warp-pair kernel on 48 SMs: both are issue-bound)
  static const bool pages_major = [] {
    const char* e = std::getenv("NX_DEC_ATTN");
    return e && std::string(e) == "pages";
  }();
  if (pages_major && g.n_kv_heads <= 8) {
    const long long T = total_tiles / g.n_kv_heads;  // 32-key tiles, sequence-major
    const long long W = std::min<long long>(sm_count, T);
    // compact slots: (sequence + unit) x kv head < (n_seq + W) x Hkv
    if (static_cast<size_t>(n_seq + W) * g.n_kv_heads * g.group * kHD > part_cap) return cudaErrorInvalidValue;
    const size_t smem = attn_smem_bytes_dec_pages(g.n_kv_heads);
    ++g_kernel_launches;
    cudaError_t e = launch_pdl(decode_attn_pages_kernel, dim3(static_cast<unsigned>(W)), dim3(g.n_kv_heads * 32),
                               smem, s, g, qkv, kplane, seqs, seq_prefix, n_seq, T, W, pages, out,
                               part_o, part_ml);
    if (e != cudaSuccess) return e;
    ++g_kernel_launches;
    return launch_pdl(decode_combine_pages_kernel, dim3(n_seq * g.n_kv_heads, g.group), dim3(kHD), 0, s, g, seqs,
                      seq_prefix, T, W, part_o, part_ml, out);
  }
  const size_t smem = attn_smem_bytes_dec();
  const long long W = std::min<long long>(static_cast<long long>(sm_count) * kPairsD, total_tiles);
  const int grid = static_cast<int>((W + kPairsD - 1) / kPairsD);
  // compact partial slots: item + unit < n_seq * Hkv + W, independent of how
  // many pieces the longest item splits into
  if ((static_cast<size_t>(n_seq) * g.n_kv_heads + static_cast<size_t>(W)) * g.group * kHD > part_cap)
    return cudaErrorInvalidValue;
  ++g_kernel_launches;
  cudaError_t e = launch_pdl(decode_attn_kernel, dim3(grid), dim3(kWarpsD * 32), smem, s, g, qkv, kplane,
                             vplane, seqs, seq_prefix, n_seq, total_tiles, W, pages, out,
                             part_o, part_ml);
  if (e != cudaSuccess) return e;
  ++g_kernel_launches;
  return launch_pdl(decode_combine_kernel, dim3(n_seq * g.n_kv_heads, g.group), dim3(kHD), 0, s, g, seqs,
                    seq_prefix, total_tiles, W, part_o, part_ml, out);
}

cudaError_t prepare_attention_kernels() {
  cudaError_t e = cudaFuncSetAttribute(prefill_attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(attn_smem_bytes_pf()));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(decode_attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(attn_smem_bytes_dec()));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(decode_attn_pages_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(attn_smem_bytes_dec_pages(8)));
  cudaFuncAttributes fa;
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, decode_combine_pages_kernel);
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, decode_combine_kernel);
  return e;
}

}  // namespace nxd
