// Paged attention over the device-resident block table.
//
// KV cache layout per layer: K and V planes of [page][kv_head][16][hd] bf16,
// written pre-swizzled (16 B chunk c of token row r stored at c ^ (r & 7)), so
// one (page, kv head) is a contiguous 4 KB run that is *already* the
// conflict-free shared-memory image: a 64-key tile is 4 + 4 cp.async.bulk
// copies issued by one thread on an mbarrier, with no per-thread address math
// (the 16 B-per-thread loader this replaced was instruction-bound at ~2 TB/s).
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

#include "device.cuh"
#include "ptx.cuh"

namespace nxd {
namespace {

constexpr int kHD = 128;        // head dim (all supported models)
constexpr int kKT = 64;         // keys per staged tile
constexpr int kRowsPF = 64;     // query rows per prefill CTA
constexpr int kThreadsAttn = 128;
constexpr int kStagesPF = 2;   // prefill: 2 x 32 KB KV stages (+16 KB Q staging)
constexpr int kStagesDec = 3;  // decode: 3 x 32 KB in flight per CTA, 2 CTAs / SM

// Swizzled offset (elements) of (row, col) in a [rows][128] bf16 tile.
__device__ __forceinline__ int swz(int row, int col) {
  return row * kHD + ((((col >> 3) ^ (row & 7)) << 3) | (col & 7));
}

__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
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
    const size_t off = (static_cast<size_t>(page) * g.n_kv_heads + kvh) * (16 * kHD);
    bulk_load(sk + p * 16 * kHD, kplane + off, 4096, bar, policy);
    bulk_load(sv + p * 16 * kHD, vplane + off, 4096, bar, policy);
  }
}

// One warp: 16 query rows against a 64-key tile already staged in smem.
// Updates the running max / sum and the 16 x 128 output accumulator.
template <bool kMask>
__device__ __forceinline__ void attend_tile(const uint32_t (&qf)[8][4], const __nv_bfloat16* sk,
                                            const __nv_bfloat16* sv, int key_lo, int key_hi,
                                            const int (&row_limit)[2], float (&m)[2],
                                            float (&l)[2], float (&o)[16][4], float scale_log2,
                                            int key0) {
  const int lane = threadIdx.x & 31;
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
      const int row = kb + (lane & 7) + ((lane >> 4) << 3);
      const int col = k * 16 + (((lane >> 3) & 1) << 3);
      ldsm_x4(b, sk + swz(row, col));
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
  float alpha[2], base[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    base[r] = mx[r] == -INFINITY ? 0.f : mx[r];
    alpha[r] = exp2f(m[r] - base[r]);
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
  uint32_t pf[4][4];  // P as A fragments, one per 16-key step
#pragma unroll
  for (int n = 0; n < 8; ++n) {
    float p[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      p[i] = exp2f(s[n][i] - base[i >> 1]);
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
      const int row = ks * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
      const int col = d2 * 16 + ((lane >> 4) << 3);
      ldsm_x4_t(b, sv + swz(row, col));
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
  // stage 16 x 128 into (swizzled) smem via 16 B loads, then ldmatrix
  for (int c = lane; c < 16 * 16; c += 32) {
    const int r = c >> 4, chunk = c & 15;
    const int gr = row0 + r;
    const int t = gr / g.group, head = kvh * g.group + gr % g.group;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (t < n_tok)
      v = *reinterpret_cast<const uint4*>(qkv + static_cast<size_t>(tok_base + t) * g.qkv_stride +
                                          head * kHD + chunk * 8);
    *reinterpret_cast<uint4*>(stage + r * kHD + ((chunk ^ (r & 7)) << 3)) = v;
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
  __nv_bfloat16* sk = reinterpret_cast<__nv_bfloat16*>(smem_attn);  // [S][64][128]
  __nv_bfloat16* sv = sk + S * kKT * kHD;                            // [S][64][128]
  __nv_bfloat16* sq = sv + S * kKT * kHD;                            // [4 warps][16][128]
  uint64_t* full = reinterpret_cast<uint64_t*>(sq + 4 * 16 * kHD);
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
  const uint64_t pol = policy_evict_first();
  if (threadIdx.x == 0)
    for (int t = 0; t < S && t < n_tiles; ++t)
      issue_kv_tile(sk + t * kKT * kHD, sv + t * kKT * kHD, &full[t], kplane, vplane, pt, kv_end,
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
    attend_tile<true>(qf, sk + buf * kKT * kHD, sv + buf * kKT * kHD, 0, kKT, row_limit, m, l, o,
                      g.scale_log2, t * kKT);
    __syncthreads();  // every warp is done with buf
    if (threadIdx.x == 0 && t + S < n_tiles)
      issue_kv_tile(sk + buf * kKT * kHD, sv + buf * kKT * kHD, &full[buf], kplane, vplane, pt,
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

// Decode: one token per sequence. 4 warps split every staged 64-key tile
// into 16-key slices; the warps' (m, l, O) are merged in shared memory.
__global__ void __launch_bounds__(kThreadsAttn)
    decode_attn_kernel(AttnGeom g, const __nv_bfloat16* __restrict__ qkv,
                       const __nv_bfloat16* __restrict__ kplane,
                       const __nv_bfloat16* __restrict__ vplane, const AttnSeq* __restrict__ seqs,
                       const int32_t* __restrict__ pages, int splits, int tiles_per_split,
                       __nv_bfloat16* __restrict__ out, float* __restrict__ part_o,
                       float* __restrict__ part_ml) {
  extern __shared__ __align__(1024) uint8_t smem_attn[];
  constexpr int S = kStagesDec;
  __nv_bfloat16* sk = reinterpret_cast<__nv_bfloat16*>(smem_attn);
  __nv_bfloat16* sv = sk + S * kKT * kHD;
  __nv_bfloat16* sq = sv + S * kKT * kHD;  // 16 x 128
  float* red = reinterpret_cast<float*>(sq + 16 * kHD);  // merge scratch
  uint64_t* full = reinterpret_cast<uint64_t*>(red + 128 + 16 * kHD);
  const int seq = blockIdx.x / splits, split = blockIdx.x % splits;
  const int kvh = blockIdx.y;
  const AttnSeq meta = seqs[seq];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t* pt = pages + meta.page_off;
  const int total_tiles = (meta.kv_len + kKT - 1) / kKT;
  const int t0 = split * tiles_per_split;
  const int t1 = min(total_tiles, t0 + tiles_per_split);
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const uint64_t pol = policy_evict_first();
  if (threadIdx.x == 0)
    for (int t = t0; t < t1 && t < t0 + S; ++t)
      issue_kv_tile(sk + (t - t0) * kKT * kHD, sv + (t - t0) * kKT * kHD, &full[t - t0], kplane,
                    vplane, pt, meta.kv_len, t * kKT, kvh, g, pol);

  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
  float o[16][4];
#pragma unroll
  for (int d = 0; d < 16; ++d)
#pragma unroll
    for (int i = 0; i < 4; ++i) o[d][i] = 0.f;
  uint32_t qf[8][4];
  // every warp loads the same 16-row Q fragment (rows >= G are zero)
  {
    for (int c = threadIdx.x; c < 16 * 16; c += kThreadsAttn) {
      const int r = c >> 4, chunk = c & 15;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (r < g.group)
        v = *reinterpret_cast<const uint4*>(qkv + static_cast<size_t>(meta.q_start) * g.qkv_stride +
                                            (kvh * g.group + r) * kHD + chunk * 8);
      *reinterpret_cast<uint4*>(sq + r * kHD + ((chunk ^ (r & 7)) << 3)) = v;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int row = (lane & 7) + (((lane >> 3) & 1) << 3);
      const int col = k * 16 + ((lane >> 4) << 3);
      ldsm_x4(qf[k], sq + swz(row, col));
    }
  }
  const int lim[2] = {meta.kv_len - 1, meta.kv_len - 1};
  for (int t = t0; t < t1; ++t) {
    const int i = t - t0, buf = i % S;
    mbar_wait(&full[buf], (i / S) & 1);
    // this warp's 16-key slice; keys past kv_len are masked via the limit
    attend_tile<true>(qf, sk + buf * kKT * kHD, sv + buf * kKT * kHD, warp * 16, warp * 16 + 16,
                      lim, m, l, o, g.scale_log2, t * kKT);
    __syncthreads();
    if (threadIdx.x == 0 && t + S < t1)
      issue_kv_tile(sk + buf * kKT * kHD, sv + buf * kKT * kHD, &full[buf], kplane, vplane, pt,
                    meta.kv_len, (t + S) * kKT, kvh, g, pol);
  }
  // merge the 4 warps: rows 0..G-1 live in lanes 0..(4*G-1) (row = lane/4).
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    l[r] += __shfl_xor_sync(0xffffffff, l[r], 1);
    l[r] += __shfl_xor_sync(0xffffffff, l[r], 2);
  }
  float* s_m = red;                  // [4 warps][16]
  float* s_l = red + 64;             // [4][16]
  float* s_o = red + 128;            // [16 rows][128] accumulated
  const int row = lane >> 2;
  if ((lane & 3) == 0) {
    s_m[warp * 16 + row] = m[0];
    s_l[warp * 16 + row] = l[0];
  }
  for (int i = threadIdx.x; i < 16 * kHD; i += kThreadsAttn) s_o[i] = 0.f;
  __syncthreads();
  float M = -INFINITY;
#pragma unroll
  for (int w = 0; w < 4; ++w) M = fmaxf(M, s_m[w * 16 + row]);
  const float scale_mine = (m[0] == -INFINITY) ? 0.f : exp2f(m[0] - M);
  if (row < g.group) {
#pragma unroll
    for (int d = 0; d < 16; ++d) {
      const int col = d * 8 + (lane & 3) * 2;
      atomicAdd(&s_o[row * kHD + col], o[d][0] * scale_mine);
      atomicAdd(&s_o[row * kHD + col + 1], o[d][1] * scale_mine);
    }
  }
  __syncthreads();
  // finalize: thread -> (row, 8 dims)
  for (int c = threadIdx.x; c < g.group * 16; c += kThreadsAttn) {
    const int r = c >> 4, d0 = (c & 15) * 8;
    float Mr = -INFINITY, L = 0.f;
    for (int w = 0; w < 4; ++w) Mr = fmaxf(Mr, s_m[w * 16 + r]);
    for (int w = 0; w < 4; ++w) {
      const float mw = s_m[w * 16 + r];
      if (mw != -INFINITY) L += s_l[w * 16 + r] * exp2f(mw - Mr);
    }
    const int head = kvh * g.group + r;
    if (splits == 1) {
      const float inv = L > 0.f ? 1.f / L : 0.f;
      __align__(16) __nv_bfloat16 v[8];
      for (int i = 0; i < 8; ++i) v[i] = __float2bfloat16(s_o[r * kHD + d0 + i] * inv);
      *reinterpret_cast<uint4*>(out + static_cast<size_t>(meta.q_start) * g.out_stride +
                                head * kHD + d0) = *reinterpret_cast<uint4*>(v);
    } else {
      const size_t base = (static_cast<size_t>(seq) * splits + split) * g.n_heads + head;
      for (int i = 0; i < 8; ++i) part_o[base * kHD + d0 + i] = s_o[r * kHD + d0 + i];
      if (d0 == 0) {
        part_ml[base * 2] = Mr;
        part_ml[base * 2 + 1] = L;
      }
    }
  }
}

// Merge KV-split partials: out = sum_s 2^(m_s - M) O_s / sum_s 2^(m_s - M) l_s.
__global__ void decode_combine_kernel(AttnGeom g, const AttnSeq* __restrict__ seqs, int splits,
                                      const float* __restrict__ part_o,
                                      const float* __restrict__ part_ml,
                                      __nv_bfloat16* __restrict__ out) {
  const int seq = blockIdx.x, head = blockIdx.y, d = threadIdx.x;  // 128 threads
  float M = -INFINITY;
  for (int s = 0; s < splits; ++s)
    M = fmaxf(M, part_ml[((static_cast<size_t>(seq) * splits + s) * g.n_heads + head) * 2]);
  float acc = 0.f, L = 0.f;
  for (int s = 0; s < splits; ++s) {
    const size_t base = (static_cast<size_t>(seq) * splits + s) * g.n_heads + head;
    const float ms = part_ml[base * 2];
    if (ms == -INFINITY) continue;
    const float w = exp2f(ms - M);
    L += part_ml[base * 2 + 1] * w;
    acc += part_o[base * kHD + d] * w;
  }
  out[static_cast<size_t>(seqs[seq].q_start) * g.out_stride + head * kHD + d] =
      __float2bfloat16(L > 0.f ? acc / L : 0.f);
}

}  // namespace

size_t attn_smem_bytes_pf() {
  return static_cast<size_t>(2 * kStagesPF * kKT * kHD + 4 * 16 * kHD) * 2 + 64;
}
size_t attn_smem_bytes_dec() {
  return static_cast<size_t>(2 * kStagesDec * kKT * kHD + 16 * kHD) * 2 + (128 + 16 * kHD) * 4 + 64;
}
size_t attn_smem_bytes() { return std::max(attn_smem_bytes_pf(), attn_smem_bytes_dec()); }

cudaError_t prefill_attention(const AttnGeom& g, const __nv_bfloat16* qkv,
                              const __nv_bfloat16* kplane, const __nv_bfloat16* vplane,
                              const AttnSeq* seqs, const int2* work, int n_work,
                              const int32_t* pages, __nv_bfloat16* out, cudaStream_t s) {
  if (n_work == 0) return cudaSuccess;
  ensure_kernels_prepared();
  const size_t smem = attn_smem_bytes_pf();
  ++g_kernel_launches;
  prefill_attn_kernel<<<dim3(n_work, g.n_kv_heads), kThreadsAttn, smem, s>>>(
      g, qkv, kplane, vplane, seqs, work, pages, out);
  return cudaGetLastError();
}

cudaError_t decode_attention(const AttnGeom& g, const __nv_bfloat16* qkv,
                             const __nv_bfloat16* kplane, const __nv_bfloat16* vplane,
                             const AttnSeq* seqs, int n_seq, int max_kv_len, const int32_t* pages,
                             __nv_bfloat16* out, float* part_o, float* part_ml, size_t part_cap,
                             int sm_count, cudaStream_t s) {
  if (n_seq == 0) return cudaSuccess;
  ensure_kernels_prepared();
  const size_t smem = attn_smem_bytes_dec();
  const int tiles = (max_kv_len + kKT - 1) / kKT;
  // Enough CTAs for ~2 waves over the partition, at least 2 tiles per split.
  const int base = n_seq * g.n_kv_heads;
  int splits = 1;
  if (part_o != nullptr && base < 2 * sm_count) {
    splits = (2 * sm_count + base - 1) / base;
    splits = std::min(splits, std::max(1, tiles / 2));
    splits = std::min(splits, 32);
    while (splits > 1 &&
           static_cast<size_t>(n_seq) * splits * g.n_heads * kHD > part_cap)
      --splits;
  }
  const int per = (tiles + splits - 1) / splits;
  splits = std::max(1, (tiles + per - 1) / per);
  ++g_kernel_launches;
  decode_attn_kernel<<<dim3(n_seq * splits, g.n_kv_heads), kThreadsAttn, smem, s>>>(
      g, qkv, kplane, vplane, seqs, pages, splits, per, out, part_o, part_ml);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || splits == 1) return e;
  ++g_kernel_launches;
  decode_combine_kernel<<<dim3(n_seq, g.n_heads), kHD, 0, s>>>(g, seqs, splits, part_o, part_ml,
                                                               out);
  return cudaGetLastError();
}

void prepare_attention_kernels() {
  cudaFuncSetAttribute(prefill_attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(attn_smem_bytes_pf()));
  cudaFuncSetAttribute(decode_attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(attn_smem_bytes_dec()));
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, decode_combine_kernel);
}

}  // namespace nxd
