// Dense projection GEMM on 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
//   out[t, f] = epilogue( sum_k X[t, k] * W[f, k] )      (y = x W^T)
//
// "Swap-AB" tiling: the weight tile is the MMA's A operand (M = 128 output
// features) and the token tile is B (N = BN tokens), so one kernel serves
// both the 2048-token prefill chunk (BN = 256, tensor-bound) and the
// <= 64-token decode batch (BN = 32/64, HBM-bound on the weight stream:
// every weight byte is read exactly once per launch).
//
// Structure (one CTA per SM, persistent over work units):
//   warp 0      TMA producer: W and X 128B-swizzled K-major tiles -> smem ring
//   warp 1      MMA issuer: one elected lane issues tcgen05.mma (M128 x N x K16)
//               into a double-buffered TMEM accumulator; owns TMEM alloc
//   warps 2-5   epilogue: tcgen05.ld -> smem stage -> fused op -> coalesced
//               16-byte global stores (bias / residual add / SwiGLU / fp32)
// A work tile is MT (1-2) 128-row weight blocks x BN tokens. Decode shapes
// use stream-K over (tile, k-block) iterations with an in-kernel fix-up;
// forced K splits (tests) use a separate reduce kernel.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "device.cuh"
#include "ptx.cuh"

namespace nxd {

namespace {

constexpr int kBM = 128;          // output features per tile (MMA M)
constexpr int kBK = 64;           // K per stage: 64 bf16 = one 128B swizzle row
constexpr int kThreads = 192;     // 6 warps
constexpr int kEpiThreads = 128;
constexpr int kABytes = kBM * kBK * 2;

// A work tile is MT consecutive 128-row weight blocks x BN tokens: the MT
// weight tiles of a stage share one activation tile, which cuts the shared-
// memory traffic per weight byte (TMA write + MMA read of W, plus X) from
// 3x to 2.5x at MT = 2 -- the per-SM bound of the decode (GEMV-like) shapes.
constexpr int pow2_cols(int c) { return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512; }

template <int BN, int MT>
struct Cfg {
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStage = MT * kABytes + kBBytes;
  static constexpr int kEpiBytes = 32 * kBM * 4;
  static constexpr int kBudget = 227 * 1024 - kEpiBytes - 1280;  // 227 KB opt-in smem per CTA
  static constexpr int kStages = kBudget / kStage > 9 ? 9 : kBudget / kStage;
  static constexpr int kTmemCols = pow2_cols(2 * MT * BN);
  static constexpr int kSmem = 1024 + kStages * kStage + kEpiBytes + 256;
  static_assert(kStages >= 2, "pipeline too shallow");
  static_assert(2 * MT * BN <= 512, "TMEM: 512 columns");
};

// Experiments only (NX_GEMM_DBG & 16): per-CTA %globaltimer stamps of the
// pipeline milestones, read back with nx_dbg_gemm_trace.
__device__ unsigned long long g_gemm_trace[1024][8];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define NX_STAMP(i) do { if (p.dbg & 16) g_gemm_trace[blockIdx.x & 1023][i] = gtimer(); } while (0)

__device__ __forceinline__ float silu(float g) { return g / (1.0f + __expf(-g)); }

struct Unit {
  int m_blk, n_blk, split;
};

// Packed weight layout: 128-row blocks in pairs, [pair][kb][2][128][64],
// each 128 x 64 tile stored as its 128B-swizzled shared-memory image (16 B
// chunk c of row r at chunk position c ^ (r & 7)), so a stage is one
// contiguous 16 KB cp.async.bulk and pairs of row blocks are adjacent.
__host__ __device__ __forceinline__ size_t packed_tile_offset(int m_blk, int kb, int num_kb) {
  return ((static_cast<size_t>(m_blk >> 1) * num_kb + kb) * 2 + (m_blk & 1)) * (kBM * kBK);
}

__global__ void pack_weights_kernel(const __nv_bfloat16* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                    int rows, int K, int pad_rows) {
  const int num_kb = K / kBK;
  const size_t n_chunks = static_cast<size_t>(pad_rows) * (K / 8);
  for (size_t c = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; c < n_chunks;
       c += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int row = static_cast<int>(c / (K / 8));
    const int kc = static_cast<int>(c % (K / 8));  // 16 B chunk along K
    const int kb = kc >> 3, ch = kc & 7;
    const int m_blk = row / kBM, r = row % kBM;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (row < rows) v = *reinterpret_cast<const uint4*>(src + static_cast<size_t>(row) * K + kc * 8);
    __nv_bfloat16* t = dst + packed_tile_offset(m_blk, kb, num_kb) + r * kBK + ((ch ^ (r & 7)) << 3);
    *reinterpret_cast<uint4*>(t) = v;
  }
}

__global__ void unpack_weights_kernel(const __nv_bfloat16* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                      int rows, int K) {
  const int num_kb = K / kBK;
  const size_t n_chunks = static_cast<size_t>(rows) * (K / 8);
  for (size_t c = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; c < n_chunks;
       c += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int row = static_cast<int>(c / (K / 8));
    const int kc = static_cast<int>(c % (K / 8));
    const int kb = kc >> 3, ch = kc & 7;
    const int m_blk = row / kBM, r = row % kBM;
    *reinterpret_cast<uint4*>(dst + static_cast<size_t>(row) * K + kc * 8) =
        *reinterpret_cast<const uint4*>(src + packed_tile_offset(m_blk, kb, num_kb) + r * kBK +
                                        ((ch ^ (r & 7)) << 3));
  }
}

__device__ __forceinline__ Unit unit_of(int u, const GemmParams& p) {
  Unit r;
  r.split = u % p.splits;
  const int tile = u / p.splits;
  r.n_blk = tile % p.n_nblk;
  r.m_blk = tile / p.n_nblk;
  return r;
}

struct Work {
  int m_blk, n_blk, kb0, kb1;
  int slot;      // stream-K: partial slot (tile * max_pieces + piece); split-K: split index
  int piece;     // fold planes: stream-K piece within the tile / split index / 0
  bool partial;  // true: write fp32 partials for a fix-up pass
};

// Stream-K covers tiles [p.sk_tile0, tiles): the leading tiles (whole
// waves) run data-parallel first (hybrid schedule for prefill shapes). Counter,
// slot and piece arithmetic use the stream-K-local tile index.
__device__ __forceinline__ int sk_local(const GemmParams& p, int m_blk, int n_blk) {
  return m_blk * p.n_nblk + n_blk - p.sk_tile0;
}
__device__ __forceinline__ long long sk_total(const GemmParams& p) {
  return (static_cast<long long>(p.n_mblk) * p.n_nblk - p.sk_tile0) * p.num_kb;
}

// This CTA's work items, in the same order for every warp role.
//  * data-parallel / split-K: units blockIdx.x, +gridDim.x, ...
//  * stream-K: the contiguous iteration range [c*I/G, (c+1)*I/G) over the
//    flattened (tile, k-block) space, cut at tile boundaries into pieces.
struct WorkIter {
  const GemmParams& p;
  int u = 0;
  long long it = 0, end = 0, total = 0;
  __device__ explicit WorkIter(const GemmParams& pp) : p(pp) {
    u = blockIdx.x;
    if (p.streamk) {
      total = sk_total(p);
      it = total * blockIdx.x / gridDim.x;
      end = total * (blockIdx.x + 1) / gridDim.x;
    }
  }
  __device__ bool next(Work& w) {
    if (p.streamk && u < p.sk_tile0) {  // hybrid: whole-tile waves first
      w.n_blk = u % p.n_nblk;
      w.m_blk = u / p.n_nblk;
      w.kb0 = 0;
      w.kb1 = p.num_kb;
      w.partial = false;
      w.slot = -1;
      w.piece = 0;
      u += gridDim.x;
      return true;
    }
    if (p.streamk) {
      if (it >= end) return false;
      const int tile = static_cast<int>(it / p.num_kb);  // stream-K-local
      w.kb0 = static_cast<int>(it % p.num_kb);
      w.kb1 = static_cast<int>(min(static_cast<long long>(p.num_kb), w.kb0 + (end - it)));
      w.n_blk = (tile + p.sk_tile0) % p.n_nblk;
      w.m_blk = (tile + p.sk_tile0) / p.n_nblk;
      w.partial = !(w.kb0 == 0 && w.kb1 == p.num_kb);
      w.slot = -1;
      w.piece = 0;
      if (w.partial) {
        const long long it0 = static_cast<long long>(tile) * p.num_kb;
        const int first = static_cast<int>(((it0 + 1) * gridDim.x - 1) / total);
        w.piece = static_cast<int>(blockIdx.x) - first;
        w.slot = tile * p.max_pieces + w.piece;
      }
      it += w.kb1 - w.kb0;
      return true;
    }
    if (u >= p.n_mblk * p.n_nblk * p.splits) return false;
    const Unit x = unit_of(u, p);
    w.m_blk = x.m_blk;
    w.n_blk = x.n_blk;
    w.kb0 = x.split * p.kb_per_split;
    w.kb1 = min(p.num_kb, w.kb0 + p.kb_per_split);
    w.partial = p.splits > 1;
    w.slot = x.split;
    w.piece = x.split;
    u += gridDim.x;
    return true;
  }
};

// Stream-K fix-up by the last arriving piece of a split tile: the 128
// epilogue threads publish their fp32 partial, count the tile's arrivals
// with one atomic, and the last CTA folds every piece of the tile and
// applies the epilogue (classic threadfence reduction; no extra launch).
template <int BN, int MT>
__device__ __forceinline__ void streamk_arrive(const GemmParams& p, const Work& w, int et, int* s_flag) {
  const int tile = sk_local(p, w.m_blk, w.n_blk);
  const long long total = sk_total(p);
  const long long it0 = static_cast<long long>(tile) * p.num_kb;
  const int first = static_cast<int>(((it0 + 1) * gridDim.x - 1) / total);
  const int last = static_cast<int>(((it0 + p.num_kb) * gridDim.x - 1) / total);
  const int pieces = last - first + 1;
  __threadfence();
  named_bar_sync(1, kEpiThreads);
  if (et == 0) {
    const int prev = atomicAdd(&p.tile_count[tile], 1);
    *s_flag = prev == pieces - 1;
    if (prev == pieces - 1) p.tile_count[tile] = 0;  // ready for the next launch
  }
  named_bar_sync(1, kEpiThreads);
  if (!*s_flag) return;
  __threadfence();
  const int tok_base = w.n_blk * p.bn_rt;
  const int n_tok = min(p.bn_rt, p.tokens - tok_base);
  const float4* base = reinterpret_cast<const float4*>(
      p.ws + static_cast<size_t>(tile) * p.max_pieces * MT * BN * kBM);
  constexpr int kSlot4 = BN * kBM / 4;  // float4 per (piece, sub-tile) slot
  const int valid = min(MT, p.n_tiles128 - w.m_blk * MT);
  // Each thread owns kPer float4 positions (coalesced: position = et + 128 i);
  // pieces are the outer loop so every pass issues kPer independent loads.
  constexpr int kPer = 8;
  const int n4 = n_tok * (kBM / 4);
  for (int sub = 0; sub < valid; ++sub)
  for (int chunk = 0; chunk < n4; chunk += kEpiThreads * kPer) {
    const int m128 = w.m_blk * MT + sub;
    float4 acc[kPer];
#pragma unroll
    for (int i = 0; i < kPer; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int q = 0; q < pieces; ++q) {
      float4 v[kPer];
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        const int pos = chunk + et + i * kEpiThreads;
        v[i] = pos < n4 ? __ldcg(base + (q * MT + sub) * kSlot4 + pos) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        acc[i].x += v[i].x;
        acc[i].y += v[i].y;
        acc[i].z += v[i].z;
        acc[i].w += v[i].w;
      }
    }
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int pos = chunk + et + i * kEpiThreads;
      if (pos >= n4) continue;
      const int j = pos / (kBM / 4), c = (pos % (kBM / 4)) * 4;  // token, feature in tile
      const int t = tok_base + j;
      if (p.mode == kEpiSwiGLU) {
        if (c >= 64) continue;  // gate half drives the output; up half read below
        float4 u = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int q = 0; q < pieces; ++q) {
          const float4 b = __ldcg(base + (q * MT + sub) * kSlot4 + pos + 16);
          u.x += b.x, u.y += b.y, u.z += b.z, u.w += b.w;
        }
        __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.out) + static_cast<size_t>(t) * p.ldo +
                             m128 * 64 + c;
        *reinterpret_cast<__nv_bfloat162*>(dst) =
            __floats2bfloat162_rn(silu(acc[i].x) * u.x, silu(acc[i].y) * u.y);
        *reinterpret_cast<__nv_bfloat162*>(dst + 2) =
            __floats2bfloat162_rn(silu(acc[i].z) * u.z, silu(acc[i].w) * u.w);
        continue;
      }
      const int f = m128 * kBM + c;
      if (p.mode == kEpiF32) {
        *reinterpret_cast<float4*>(static_cast<float*>(p.out) + static_cast<size_t>(t) * p.ldo + f) =
            acc[i];
        continue;
      }
      float o0 = acc[i].x, o1 = acc[i].y, o2 = acc[i].z, o3 = acc[i].w;
      if (p.mode == kEpiBias || p.mode == kEpiBiasResidual) {
        const __nv_bfloat162 b01 = *reinterpret_cast<const __nv_bfloat162*>(p.bias + f);
        const __nv_bfloat162 b23 = *reinterpret_cast<const __nv_bfloat162*>(p.bias + f + 2);
        o0 += __low2float(b01), o1 += __high2float(b01), o2 += __low2float(b23), o3 += __high2float(b23);
      }
      if (p.mode == kEpiResidual || p.mode == kEpiBiasResidual) {
        const __nv_bfloat16* rp = p.residual + static_cast<size_t>(t) * p.ldr + f;
        const __nv_bfloat162 r01 = *reinterpret_cast<const __nv_bfloat162*>(rp);
        const __nv_bfloat162 r23 = *reinterpret_cast<const __nv_bfloat162*>(rp + 2);
        o0 += __low2float(r01), o1 += __high2float(r01), o2 += __low2float(r23), o3 += __high2float(r23);
      }
      __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.out) + static_cast<size_t>(t) * p.ldo + f;
      *reinterpret_cast<__nv_bfloat162*>(dst) = __floats2bfloat162_rn(o0, o1);
      *reinterpret_cast<__nv_bfloat162*>(dst + 2) = __floats2bfloat162_rn(o2, o3);
    }
  }
}

// Stream-K fix-up when all CTAs are co-resident (p.coresident): every piece
// publishes its fp32 partial and counts itself in; once a tile's pieces are
// all in, piece i folds rows [i R/P, (i+1) R/P) of the tile (R = tokens x
// sub-tiles) across all P partials and applies the epilogue. The fold is
// spread over the P CTAs instead of serialized on the last arriver, and its
// loads are issued P-deep. The last piece to leave resets the counters.
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void streamk_tile_pieces(const GemmParams& p, int tile, int* first, int* pieces) {
  const long long total = sk_total(p);
  const long long it0 = static_cast<long long>(tile) * p.num_kb;
  *first = static_cast<int>(((it0 + 1) * gridDim.x - 1) / total);
  const int last = static_cast<int>(((it0 + p.num_kb) * gridDim.x - 1) / total);
  *pieces = last - *first + 1;
}

__device__ __forceinline__ void store_out4(const GemmParams& p, int t, int f, float4 a) {
  if (p.mode == kEpiF32) {
    *reinterpret_cast<float4*>(static_cast<float*>(p.out) + static_cast<size_t>(t) * p.ldo + f) = a;
    return;
  }
  if (p.mode == kEpiBias || p.mode == kEpiBiasResidual) {
    const __nv_bfloat162 b01 = *reinterpret_cast<const __nv_bfloat162*>(p.bias + f);
    const __nv_bfloat162 b23 = *reinterpret_cast<const __nv_bfloat162*>(p.bias + f + 2);
    a.x += __low2float(b01), a.y += __high2float(b01), a.z += __low2float(b23), a.w += __high2float(b23);
  }
  if (p.mode == kEpiResidual || p.mode == kEpiBiasResidual) {
    const __nv_bfloat16* rp = p.residual + static_cast<size_t>(t) * p.ldr + f;
    const __nv_bfloat162 r01 = *reinterpret_cast<const __nv_bfloat162*>(rp);
    const __nv_bfloat162 r23 = *reinterpret_cast<const __nv_bfloat162*>(rp + 2);
    a.x += __low2float(r01), a.y += __high2float(r01), a.z += __low2float(r23), a.w += __high2float(r23);
  }
  __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.out) + static_cast<size_t>(t) * p.ldo + f;
  __nv_bfloat162 lo = __floats2bfloat162_rn(a.x, a.y), hi = __floats2bfloat162_rn(a.z, a.w);
  uint2 v;
  v.x = *reinterpret_cast<uint32_t*>(&lo);
  v.y = *reinterpret_cast<uint32_t*>(&hi);
  *reinterpret_cast<uint2*>(dst) = v;
}

template <int BN, int MT>
__device__ void streamk_publish(const GemmParams& p, const Work& w, int et) {
  __threadfence();
  named_bar_sync(1, kEpiThreads);
  if (et == 0) atomicAdd(&p.tile_count[sk_local(p, w.m_blk, w.n_blk)], 1);
}

template <int BN, int MT>
__device__ void streamk_reduce_slice(const GemmParams& p, int m_blk, int n_blk, int et, uint8_t* scratch,
                                     uint64_t* bar, uint32_t& phase) {
  const int tile = sk_local(p, m_blk, n_blk);
  int first, pieces;
  streamk_tile_pieces(p, tile, &first, &pieces);
  const int piece = static_cast<int>(blockIdx.x) - first;
  int* arrive = p.tile_count + tile;
  int* depart = p.tile_count + kGemmMaxCounterTiles + tile;
  const int tok_base = n_blk * p.bn_rt;
  const int n_tok = min(p.bn_rt, p.tokens - tok_base);
  const int valid = min(MT, p.n_tiles128 - m_blk * MT);
  const int R = valid * n_tok;
  const int r0 = R * piece / pieces, r1 = R * (piece + 1) / pieces;
  const int nrows = r1 - r0;
  constexpr int kRowBytes = kBM * 4;
  if (et == 0) {
    while (ld_acquire_gpu(arrive) < pieces) __nanosleep(32);
    // one bulk copy per (piece, sub-tile run of rows): the whole slice of
    // every partial lands in shared memory after a single round trip
    if (nrows > 0) {
      mbar_expect_tx(bar, static_cast<uint32_t>(pieces * nrows * kRowBytes));
      const float* base = p.ws + static_cast<size_t>(tile) * p.max_pieces * MT * BN * kBM;
      for (int q = 0; q < pieces; ++q) {
        int r = r0;
        while (r < r1) {
          const int sub = r / n_tok, j = r % n_tok;
          const int run = min(r1 - r, n_tok - j);
          const float* src = base + ((static_cast<size_t>(q) * MT + sub) * BN + j) * kBM;
          bulk_load(scratch + (static_cast<size_t>(q) * nrows + (r - r0)) * kRowBytes, src,
                    static_cast<uint32_t>(run * kRowBytes), bar);
          r += run;
        }
      }
    }
  }
  named_bar_sync(1, kEpiThreads);
  if (nrows > 0) {
    mbar_wait(bar, phase);
    phase ^= 1;
  }
  const bool swiglu = p.mode == kEpiSwiGLU;
  const int per_row = swiglu ? 16 : 32;  // float4 units per (sub, token) row
  const int units = nrows * per_row;
  const float4* sc = reinterpret_cast<const float4*>(scratch);
  const int slice4 = nrows * (kBM / 4);
  for (int u = et; u < units; u += kEpiThreads) {
    const int lr = u / per_row, c4 = u % per_row;
    const int pos = lr * (kBM / 4) + c4;
    float4 g = make_float4(0.f, 0.f, 0.f, 0.f), up = g;
    for (int q = 0; q < pieces; ++q) {
      const float4 v = sc[q * slice4 + pos];
      g.x += v.x, g.y += v.y, g.z += v.z, g.w += v.w;
      if (swiglu) {
        const float4 b = sc[q * slice4 + pos + 16];
        up.x += b.x, up.y += b.y, up.z += b.z, up.w += b.w;
      }
    }
    const int row = r0 + lr;
    const int sub = row / n_tok, j = row % n_tok, c = c4 * 4;
    const int t = tok_base + j;
    const int m128 = m_blk * MT + sub;
    if (swiglu) {
      __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.out) + static_cast<size_t>(t) * p.ldo + m128 * 64 + c;
      __nv_bfloat162 lo = __floats2bfloat162_rn(silu(g.x) * up.x, silu(g.y) * up.y);
      __nv_bfloat162 hi = __floats2bfloat162_rn(silu(g.z) * up.z, silu(g.w) * up.w);
      uint2 o;
      o.x = *reinterpret_cast<uint32_t*>(&lo);
      o.y = *reinterpret_cast<uint32_t*>(&hi);
      *reinterpret_cast<uint2*>(dst) = o;
    } else {
      store_out4(p, t, m128 * kBM + c, g);
    }
  }
  named_bar_sync(1, kEpiThreads);
  if (et == 0 && atomicAdd(depart, 1) == pieces - 1) {
    *arrive = 0;  // every piece is past its wait: ready for the next launch
    *depart = 0;
  }
}

template <int BN, int MT>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __nv_bfloat16* __restrict__ wpack, const __grid_constant__ CUtensorMap tx,
                   GemmParams p) {
  using C = Cfg<BN, MT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  float* s_epi = reinterpret_cast<float*>(smem + C::kStages * C::kStage);
  uint64_t* full = reinterpret_cast<uint64_t*>(s_epi + 32 * kBM);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + 2;
  uint64_t* fix_bar = tempty + 2;  // parallel stream-K fix-up loads
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 3);
  int* s_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) NX_STAMP(0);
  if (warp == 0 && elect_one()) {
    tma_prefetch(&tx);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiThreads);
    }
    mbar_init(fix_bar, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Dependents may launch only once every CTA of this grid holds its TMEM: a
  // dependent CTA co-resident on an SM could otherwise allocate first and
  // spin in griddepcontrol.wait while this CTA blocks in tcgen05.alloc.
  pdl_trigger();
  if (threadIdx.x == 0) NX_STAMP(1);

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (elect_one()) {
      const uint64_t w_policy = policy_evict_first();  // weights stream once
      const uint32_t stage_bytes_x = (p.dbg & 1) ? 0 : C::kBBytes;
      // weight tiles = contiguous pre-swizzled 16 KB chunks (pack_weights); an
      // aligned pair of row blocks is one 32 KB copy
      auto load_w = [&](const Work& w, int kb, int valid, uint8_t* sa, uint64_t* bar) {
        if (MT == 2 && valid == 2) {
          bulk_load(sa, wpack + packed_tile_offset(w.m_blk * 2, kb, p.num_kb), 2 * kABytes, bar, w_policy);
        } else {
          for (int t = 0; t < valid; ++t)
            bulk_load(sa + t * kABytes, wpack + packed_tile_offset(w.m_blk * MT + t, kb, p.num_kb), kABytes,
                      bar, w_policy);
        }
      };
      // 1) The weights of the first kStages fills depend on nothing upstream:
      //    stream them before the grid dependency resolves (programmatic
      //    dependent launch), hiding the pipeline fill behind the previous kernel.
      int pre = 0;
      {
        WorkIter wp(p);
        Work w;
        while (pre < C::kStages && wp.next(w)) {
          const int valid = min(MT, p.n_tiles128 - w.m_blk * MT);
          for (int kb = w.kb0; kb < w.kb1 && pre < C::kStages; ++kb, ++pre) {
            mbar_expect_tx(&full[pre], valid * kABytes + stage_bytes_x);
            load_w(w, kb, valid, smem + pre * C::kStage, &full[pre]);
          }
        }
      }
      pdl_wait();  // activations below are written by the previous kernel
      int stage = 0, fill = 0;
      uint32_t phase = 0;
      WorkIter wi(p);
      Work w;
      while (wi.next(w)) {
        const int valid = min(MT, p.n_tiles128 - w.m_blk * MT);
        for (int kb = w.kb0; kb < w.kb1; ++kb, ++fill) {
          uint8_t* sa = smem + stage * C::kStage;
          if (fill >= pre) {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_expect_tx(&full[stage], valid * kABytes + stage_bytes_x);
            load_w(w, kb, valid, sa, &full[stage]);
          }
          if (!(p.dbg & 1)) tma_load_2d(&tx, &full[stage], sa + MT * kABytes, kb * kBK, w.n_blk * p.bn_rt);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = umma_idesc_bf16(kBM, p.bn_rt);  // runtime N <= BN (prefill wave fit)
    int stage = 0;
    uint32_t phase = 0;
    int local = 0;
    WorkIter wi(p);
    Work w;
    for (; wi.next(w); ++local) {
      const int kb0 = w.kb0, kb1 = w.kb1;
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const int valid = min(MT, p.n_tiles128 - w.m_blk * MT);
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&full[stage], phase);
        if (local == 0 && kb == kb0 && lane_id() == 0) NX_STAMP(2);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t base = smem_u32(smem + stage * C::kStage);
          const uint32_t b_addr = base + MT * kABytes;
          for (int t = 0; t < ((p.dbg & 2) ? 0 : valid); ++t) {
            const uint32_t d = tmem + (acc * MT + t) * BN;
            const uint32_t a_addr = base + t * kABytes;
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk)
              umma_bf16(d, umma_desc_sw128(a_addr + kk * 32), umma_desc_sw128(b_addr + kk * 32),
                        idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
          }
          umma_commit(&empty[stage]);
          if (kb == kb1 - 1) umma_commit(&tfull[acc]);
          NX_STAMP(3);
        }
        __syncwarp();
        if (++stage == C::kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else {
    // ---------------- epilogue ----------------
    pdl_wait();  // residual / stream-K workspace come from upstream kernels
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int et = threadIdx.x - 64;
    const int lane = lane_id();
    int local = 0;
    int pend_m[2], pend_n[2], n_pend = 0;  // partial items awaiting the parallel fix-up
    WorkIter wi(p);
    Work w;
    for (; wi.next(w); ++local) {
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      mbar_wait(&tfull[acc], acc_phase);
      if (et == 0) NX_STAMP(4);
      tc_fence_after();
      const int valid = min(MT, p.n_tiles128 - w.m_blk * MT);
      for (int sub = 0; sub < valid; ++sub)
      for (int c0 = 0; c0 < p.bn_rt; c0 += 32) {
        const int m128 = w.m_blk * MT + sub;
        const int f0 = m128 * kBM;
        const int tok0 = w.n_blk * p.bn_rt + c0;
        const int tlim = min(p.tokens, (w.n_blk + 1) * p.bn_rt);  // this tile's token rows
        if (tok0 >= tlim) break;
        // residual rows of this 32-token chunk: issued before the TMEM load
        // so their global latency overlaps the accumulator staging
        const bool has_res = !w.partial && !p.fold && (p.mode == kEpiResidual || p.mode == kEpiBiasResidual);
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
        tmem_ld32(tmem + (acc * MT + sub) * BN + c0 + (static_cast<uint32_t>(q * 32) << 16), r);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) s_epi[j * kBM + q * 32 + lane] = __uint_as_float(r[j]);
        named_bar_sync(1, kEpiThreads);
        if (w.partial || p.fold) {
          // fp32 partials: fold plane [piece][token][rows], stream-K slot
          // [BN tokens][128] or split-K plane
          const int g = et & 31;
#pragma unroll
          for (int pass = 0; pass < 8; ++pass) {
            const int j = pass * 4 + (et >> 5);
            const int t = tok0 + j;
            if (t < tlim) {
              const float4 v = *reinterpret_cast<const float4*>(&s_epi[j * kBM + g * 4]);
              float* dst =
                  p.fold      ? p.ws + (static_cast<size_t>(w.piece) * p.tokens + t) * p.rows + f0 + g * 4
                  : p.streamk ? p.ws + ((static_cast<size_t>(w.slot) * MT + sub) * BN + c0 + j) * kBM + g * 4
                              : p.ws + (static_cast<size_t>(w.slot) * p.tokens + t) * p.rows + f0 + g * 4;
              *reinterpret_cast<float4*>(dst) = v;
            }
          }
        } else if (p.mode == kEpiSwiGLU) {
          // rows 0-63 of the tile are gate features, 64-127 the matching up features
          const int g = et & 7;
#pragma unroll
          for (int pass = 0; pass < 2; ++pass) {
            const int j = pass * 16 + (et >> 3);
            const int t = tok0 + j;
            if (t < tlim) {
              __align__(16) __nv_bfloat16 o[8];
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const float gt = s_epi[j * kBM + g * 8 + i];
                const float up = s_epi[j * kBM + 64 + g * 8 + i];
                o[i] = __float2bfloat16(silu(gt) * up);
              }
              __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(p.out) +
                                   static_cast<size_t>(t) * p.ldo + m128 * 64 + g * 8;
              *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<uint4*>(o);
            }
          }
        } else if (p.mode == kEpiF32) {
          const int g = et & 31;
#pragma unroll
          for (int pass = 0; pass < 8; ++pass) {
            const int j = pass * 4 + (et >> 5);
            const int t = tok0 + j;
            if (t < tlim) {
              const float4 v = *reinterpret_cast<const float4*>(&s_epi[j * kBM + g * 4]);
              float* dst = static_cast<float*>(p.out) + static_cast<size_t>(t) * p.ldo + f0 + g * 4;
              *reinterpret_cast<float4*>(dst) = v;
            }
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
              __nv_bfloat16* dst =
                  static_cast<__nv_bfloat16*>(p.out) + static_cast<size_t>(t) * p.ldo + f;
              *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<uint4*>(o);
            }
          }
        }
        named_bar_sync(1, kEpiThreads);
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (et == 0) NX_STAMP(5);
      if (p.streamk && w.partial && !p.fold) {
        if (p.coresident && n_pend < 2) {
          // publish now, fold after the last item: publishing never waits,
          // so no chain of waits can form across CTAs
          streamk_publish<BN, MT>(p, w, et);
          pend_m[n_pend] = w.m_blk;
          pend_n[n_pend++] = w.n_blk;
        } else {
          streamk_arrive<BN, MT>(p, w, et, s_flag);
        }
      }
    }
    // the stage ring is idle now (every stage was consumed by the MMAs that
    // produced the accumulators above): it stages the fix-up slices
    uint32_t fix_phase = 0;
    for (int i = 0; i < n_pend; ++i)
      streamk_reduce_slice<BN, MT>(p, pend_m[i], pend_n[i], et, smem, fix_bar, fix_phase);
    if (et == 0) NX_STAMP(6);
  }
  __syncthreads();
  if (threadIdx.x == 0) NX_STAMP(7);
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem);
  }
}

// Folds K-split partials [split][token][rows] with the requested epilogue.
__global__ void splitk_reduce_kernel(GemmParams p, int final_mode) {
  pdl_trigger();
  pdl_wait();
  const int out_cols = final_mode == kEpiSwiGLU ? p.rows / 2 : p.rows;
  const int groups = out_cols / 8;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= p.tokens * groups) return;
  const int t = idx / groups;
  const int g = idx % groups;
  float v[8], u[8];
  const size_t plane = static_cast<size_t>(p.tokens) * p.rows;
  if (final_mode == kEpiSwiGLU) {
    // output features [64*b + i] come from tile rows i (gate) and 64+i (up)
    const int fo = g * 8;
    const int blk = fo / 64, off = fo % 64;
    const int fg = blk * kBM + off, fu = fg + 64;
    for (int i = 0; i < 8; ++i) v[i] = u[i] = 0.f;
    for (int s = 0; s < p.splits; ++s) {
      const float* src = p.ws + s * plane + static_cast<size_t>(t) * p.rows;
      for (int i = 0; i < 8; ++i) {
        v[i] += src[fg + i];
        u[i] += src[fu + i];
      }
    }
    __align__(16) __nv_bfloat16 o[8];
    for (int i = 0; i < 8; ++i) o[i] = __float2bfloat16(silu(v[i]) * u[i]);
    *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.out) + static_cast<size_t>(t) * p.ldo +
                              fo) = *reinterpret_cast<uint4*>(o);
    return;
  }
  const int f = g * 8;
  for (int i = 0; i < 8; ++i) v[i] = 0.f;
  for (int s = 0; s < p.splits; ++s) {
    const float4* src =
        reinterpret_cast<const float4*>(p.ws + s * plane + static_cast<size_t>(t) * p.rows + f);
    const float4 a = src[0], b = src[1];
    v[0] += a.x, v[1] += a.y, v[2] += a.z, v[3] += a.w;
    v[4] += b.x, v[5] += b.y, v[6] += b.z, v[7] += b.w;
  }
  if (final_mode == kEpiF32) {
    float* dst = static_cast<float*>(p.out) + static_cast<size_t>(t) * p.ldo + f;
    for (int i = 0; i < 8; ++i) dst[i] = v[i];
    return;
  }
  if (final_mode == kEpiBias || final_mode == kEpiBiasResidual)
    for (int i = 0; i < 8; ++i) v[i] += bf2f(p.bias[f + i]);
  if (final_mode == kEpiResidual || final_mode == kEpiBiasResidual)
    for (int i = 0; i < 8; ++i) v[i] += bf2f(p.residual[static_cast<size_t>(t) * p.ldr + f + i]);
  __align__(16) __nv_bfloat16 o[8];
  for (int i = 0; i < 8; ++i) o[i] = __float2bfloat16(v[i]);
  *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.out) + static_cast<size_t>(t) * p.ldo + f) =
      *reinterpret_cast<uint4*>(o);
}

template <int BN, int MT>
cudaError_t launch_bn(const __nv_bfloat16* tw, const CUtensorMap& tx, const GemmParams& p, int grid,
                      cudaStream_t s) {
  using C = Cfg<BN, MT>;
  ensure_kernels_prepared();
  ++g_kernel_launches;
  return launch_pdl(gemm_tc_kernel<BN, MT>, dim3(grid), dim3(kThreads), C::kSmem, s, tw, tx, p);
}

}  // namespace

// NX_BN_FIT=0 keeps N = 256 for every prefill tile.
bool gemm_bn_fit_enabled();
static bool bn_fit_enabled() { return gemm_bn_fit_enabled(); }
bool gemm_bn_fit_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("NX_BN_FIT");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Prefill hybrid stream-K applies when the last wave is at most this full
// (NX_HYBRID_FRAC; 0 disables).
static double hybrid_max_frac() {
  static const double f = [] {
    const char* e = std::getenv("NX_HYBRID_FRAC");
    return e ? std::atof(e) : 0.0;
  }();
  return f;
}

size_t packed_weight_elems(int rows, int K) {
  const int blocks = (rows + kBM - 1) / kBM;
  return static_cast<size_t>((blocks + 1) & ~1) * kBM * K;
}

cudaError_t pack_weights(const __nv_bfloat16* src, __nv_bfloat16* dst, int rows, int K,
                         cudaStream_t s) {
  if (K % kBK) return cudaErrorInvalidValue;
  const int blocks = (rows + kBM - 1) / kBM;
  const int pad_rows = ((blocks + 1) & ~1) * kBM;
  ++g_kernel_launches;
  pack_weights_kernel<<<1184, 256, 0, s>>>(src, dst, rows, K, pad_rows);
  return cudaGetLastError();
}

cudaError_t unpack_weights(const __nv_bfloat16* src, __nv_bfloat16* dst, int rows, int K,
                           cudaStream_t s) {
  ++g_kernel_launches;
  unpack_weights_kernel<<<1184, 256, 0, s>>>(src, dst, rows, K);
  return cudaGetLastError();
}

int gemm_pick_bn(int tokens) {
  return tokens <= 32 ? 32 : tokens <= 64 ? 64 : tokens <= 128 ? 128 : 256;
}

cudaError_t gemm(const __nv_bfloat16* w_map, const CUtensorMap& x_map_for_bn, int bn, int rows,
                 int tokens, int K, int mode, void* out, int ldo, const __nv_bfloat16* bias,
                 const __nv_bfloat16* residual, int ldr, float* ws, size_t ws_bytes, int sm_count,
                 cudaStream_t stream, int force_splits, bool coresident, GemmFold* fold) {
  if (tokens <= 0) return cudaSuccess;
  if (rows % kBM || K % kBK) return cudaErrorInvalidValue;
  GemmParams p{};
  p.rows = rows;
  p.tokens = tokens;
  p.K = K;
  // Two weight blocks per work tile only pay off on small partitions, where
  // per-SM shared-memory traffic is the bound (gate_up on 16 SMs: +39%); at
  // full occupancy the stream-K fix-up of 2-block tiles serializes (ncu:
  // per-SM active cycles 70K..184K), so larger partitions keep MT = 1.
  const int mt = (bn <= 64 && sm_count <= 24) ? 2 : 1;
  p.n_tiles128 = rows / kBM;
  p.n_mblk = (p.n_tiles128 + mt - 1) / mt;
  // Prefill (BN = 256): the token tile width N is a runtime choice in
  // [192, 256] (multiples of 16) that fits the tile count to whole waves of
  // the partition -- e.g. T = 1450 on 112 SMs: o / down have 32 x 6 = 192
  // tiles (1.7 waves) at N = 256, 32 x 7 = 224 (2.0 waves) at N = 208. MMAs
  // with N >= ~200 stay near the tensor floor (N <= 128 costs ~100 cycles
  // regardless, tools/mma_probe.cu), so narrower tiles are not an option.
  p.bn_rt = bn;
  if (bn == 256 && force_splits == 0 && !fold && bn_fit_enabled()) {
    long long best = -1;
    for (int n = 256; n >= 192; n -= 16) {
      const long long tiles_n = static_cast<long long>(p.n_mblk) * ((tokens + n - 1) / n);
      const long long waves = (tiles_n + sm_count - 1) / sm_count;
      // tile time ~ half fixed (weight / activation staging, epilogue per tile),
      // half MMA (cycles ~ max(N, 208) per K16 step, tools/mma_probe.cu); measured:
      // gate_up at 12 vs 14 waves of N = 256 vs 208 was 10% faster at 256
      const long long cost = waves * (std::max(n, 208) + 256);
      if (best < 0 || cost < best) best = cost, p.bn_rt = n;
    }
  }
  p.n_nblk = (tokens + p.bn_rt - 1) / p.bn_rt;
  p.num_kb = K / kBK;
  p.mode = mode;
  p.out = out;
  p.ldo = ldo;
  p.bias = bias;
  p.residual = residual;
  p.ldr = ldr;
  p.bn = bn;
  static const int dbg = [] {
    const char* e = std::getenv("NX_GEMM_DBG");
    return e ? std::atoi(e) : 0;
  }();
  p.dbg = dbg;
  p.coresident = coresident ? 1 : 0;
  p.fold = fold ? 1 : 0;
  // ws layout: [int tile counters | fp32 partials]
  p.tile_count = reinterpret_cast<int*>(ws);
  p.ws = ws ? reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + gemm_counter_bytes()) : nullptr;
  ws_bytes = ws_bytes > gemm_counter_bytes() ? ws_bytes - gemm_counter_bytes() : 0;
  const int tiles = p.n_mblk * p.n_nblk;
  const long long iters = static_cast<long long>(tiles) * p.num_kb;
  int grid;
  p.splits = 1;
  p.kb_per_split = p.num_kb;
  p.streamk = 0;
  const size_t plane_bytes = static_cast<size_t>(tokens) * rows * 4;
  if (fold) {
    // Deferred fold: planes only, no counters, no fix-up, no reduce kernel.
    GemmFold f;
    f.planes = p.ws;
    f.rows = rows;
    f.tokens = tokens;
    f.rows_per_blk = kBM * mt;
    f.bn = bn;
    f.n_nblk = p.n_nblk;
    f.num_kb = p.num_kb;
    if (p.ws == nullptr || plane_bytes > ws_bytes) return cudaErrorInvalidValue;
    const int max_splits = static_cast<int>(std::min<size_t>(64, ws_bytes / plane_bytes));
    int splits = force_splits > 0 ? force_splits
                 : (mt == 2 && tiles < sm_count) ? std::min((sm_count + tiles - 1) / tiles, std::max(1, p.num_kb / 8))
                                                 : 0;
    if (splits > 0) {
      splits = std::min(splits, max_splits);
      p.kb_per_split = (p.num_kb + splits - 1) / splits;
      p.splits = (p.num_kb + p.kb_per_split - 1) / p.kb_per_split;
      grid = std::max(1, std::min(tiles * p.splits, sm_count));
      f.kind = p.splits > 1 ? 1 : 0;
      f.splits = p.splits;
    } else {
      grid = std::max(1, std::min(tiles, sm_count));
      if (tiles % sm_count != 0 && tiles < 8 * sm_count) {
        // stream-K: equal (tile, k-block) ranges per CTA (no wave tail)
        const int G = static_cast<int>(std::min<long long>(sm_count, iters));
        const long long per_min = iters / G;
        const int max_pieces = static_cast<int>((p.num_kb + per_min - 1) / per_min) + 1;
        if (max_pieces <= max_splits) {
          p.streamk = 1;
          p.max_pieces = max_pieces;
          grid = G;
          f.kind = 2;
          f.grid = G;
          f.total = iters;
        }
      }
    }
    *fold = f;
  } else if (force_splits > 0) {
    // explicit split-K (tests / experiments)
    p.kb_per_split = (p.num_kb + force_splits - 1) / force_splits;
    p.splits = (p.num_kb + p.kb_per_split - 1) / p.kb_per_split;
    if (static_cast<size_t>(p.splits) * tokens * rows * 4 > ws_bytes) return cudaErrorInvalidValue;
    grid = std::max(1, std::min(tiles * p.splits, sm_count));
  } else if (mt == 2 && ws != nullptr && tiles < sm_count) {
    // small partition: K splits until every SM has a unit (balanced, no fix-up)
    int splits = std::min((sm_count + tiles - 1) / tiles, std::max(1, p.num_kb / 8));
    while (splits > 1 && static_cast<size_t>(splits) * tokens * rows * 4 > ws_bytes) --splits;
    p.kb_per_split = (p.num_kb + splits - 1) / splits;
    p.splits = (p.num_kb + p.kb_per_split - 1) / p.kb_per_split;
    grid = std::max(1, std::min(tiles * p.splits, sm_count));
  } else if (tokens <= 256 && ws != nullptr && tiles % sm_count != 0 &&
             tiles <= kGemmMaxCounterTiles) {
    // Stream-K: equal (tile, k-block) ranges per CTA remove the wave tail
    // of decode-shaped launches (weight streaming: every CTA busy to the end).
    const int G = static_cast<int>(std::min<long long>(sm_count, iters));
    const long long per_min = iters / G;
    p.max_pieces = static_cast<int>((p.num_kb + per_min - 1) / per_min) + 1;
    const size_t need = static_cast<size_t>(tiles) * p.max_pieces * mt * bn * kBM * 4;
    if (need <= ws_bytes && tiles < 8 * G) {
      p.streamk = 1;
      grid = G;
    } else {
      grid = std::max(1, std::min(tiles, sm_count));
    }
  } else if (tokens > 256 && ws != nullptr && tiles > sm_count && tiles % sm_count != 0 &&
             static_cast<double>(tiles % sm_count) / sm_count < hybrid_max_frac()) {
    // Hybrid: whole waves data-parallel, the partial last wave stream-K
    // (e.g. o / down at T = 2048 on 112 SMs: 256 tiles = 2.29 waves, not 3).
    const int rem = tiles % sm_count;
    const long long rem_iters = static_cast<long long>(rem) * p.num_kb;
    const long long per_min = std::max<long long>(1, rem_iters / sm_count);
    p.max_pieces = static_cast<int>((p.num_kb + per_min - 1) / per_min) + 1;
    const size_t need = static_cast<size_t>(rem) * p.max_pieces * mt * bn * kBM * 4;
    grid = sm_count;
    if (need <= ws_bytes && rem <= kGemmMaxCounterTiles) {
      p.streamk = 1;
      p.sk_tile0 = tiles - rem;
    }
  } else {
    grid = std::max(1, std::min(tiles, sm_count));
  }
  cudaError_t e;
  switch (bn * 4 + mt) {
    case 32 * 4 + 1: e = launch_bn<32, 1>(w_map, x_map_for_bn, p, grid, stream); break;
    case 32 * 4 + 2: e = launch_bn<32, 2>(w_map, x_map_for_bn, p, grid, stream); break;
    case 64 * 4 + 1: e = launch_bn<64, 1>(w_map, x_map_for_bn, p, grid, stream); break;
    case 64 * 4 + 2: e = launch_bn<64, 2>(w_map, x_map_for_bn, p, grid, stream); break;
    case 128 * 4 + 1: e = launch_bn<128, 1>(w_map, x_map_for_bn, p, grid, stream); break;
    case 256 * 4 + 1: e = launch_bn<256, 1>(w_map, x_map_for_bn, p, grid, stream); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  if (fold || p.streamk || p.splits == 1) return cudaSuccess;
  const int out_cols = mode == kEpiSwiGLU ? rows / 2 : rows;
  const int work = tokens * (out_cols / 8);
  ++g_kernel_launches;
  return launch_pdl(splitk_reduce_kernel, dim3((work + 255) / 256), dim3(256), 0, stream, p, mode);
}

template <int BN, int MT>
static void prepare_one() {
  cudaFuncSetAttribute(gemm_tc_kernel<BN, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       Cfg<BN, MT>::kSmem);
}

void prepare_gemm_kernels() {
  prepare_one<32, 1>();
  prepare_one<32, 2>();
  prepare_one<64, 1>();
  prepare_one<64, 2>();
  prepare_one<128, 1>();
  prepare_one<256, 1>();
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, pack_weights_kernel);
  cudaFuncGetAttributes(&fa, unpack_weights_kernel);
  cudaFuncGetAttributes(&fa, splitk_reduce_kernel);
}

size_t gemm_trace_read(unsigned long long* host, size_t n) {
  const size_t cap = sizeof(g_gemm_trace) / sizeof(unsigned long long);
  if (n > cap) n = cap;
  if (cudaMemcpyFromSymbol(host, g_gemm_trace, n * sizeof(unsigned long long)) != cudaSuccess) return 0;
  return n;
}

}  // namespace nxd
