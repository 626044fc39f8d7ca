// Bandwidth-bound helpers of the forward pass: embedding gather, RMSNorm,
// RoPE + paged KV write, row argmax (greedy sampling), weight init, and the
// TMA descriptor encoder. All loads/stores are 16-byte vectors.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cudaTypedefs.h>

#include <cfloat>
#include <cstdlib>

#include "device.cuh"

namespace nxd {

unsigned long long g_kernel_launches = 0;

namespace {

__global__ void embed_kernel(const int32_t* __restrict__ tok, const __nv_bfloat16* __restrict__ table,
                             int hidden, __nv_bfloat16* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x;
  const uint4* src = reinterpret_cast<const uint4*>(table + static_cast<size_t>(tok[t]) * hidden);
  uint4* dst = reinterpret_cast<uint4*>(out + static_cast<size_t>(t) * hidden);
  for (int i = threadIdx.x; i < hidden / 8; i += blockDim.x) dst[i] = src[i];
}

// One CTA (128 threads) per row, up to kNormVec 16 B chunks per thread, read
// once into registers. Small CTAs keep ~16 rows in flight per SM (a 2048-token
// prefill batch is ~1 wave instead of ~3 of latency-bound 512-thread rows).
constexpr int kNormVec = 8;
__global__ void __launch_bounds__(128) rmsnorm_kernel(const __nv_bfloat16* __restrict__ x,
                                                      const int32_t* __restrict__ rows, int hidden,
                                                      const __nv_bfloat16* __restrict__ w, float eps,
                                                      __nv_bfloat16* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  const int src_row = rows ? rows[r] : r;
  const uint4* xr = reinterpret_cast<const uint4*>(x + static_cast<size_t>(src_row) * hidden);
  const int nvec = hidden / 8;
  uint4 v[kNormVec];
  float ss = 0.f;
#pragma unroll
  for (int c = 0; c < kNormVec; ++c) {
    const int i = threadIdx.x + c * blockDim.x;
    v[c] = i < nvec ? xr[i] : make_uint4(0, 0, 0, 0);
    const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&v[c]);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float f = __bfloat162float(b[k]);
      ss += f * f;
    }
  }
  __shared__ float red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffff, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
  for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) tot += red[i];
  const float inv = rsqrtf(tot / hidden + eps);
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  uint4* dst = reinterpret_cast<uint4*>(out + static_cast<size_t>(r) * hidden);
#pragma unroll
  for (int c = 0; c < kNormVec; ++c) {
    const int i = threadIdx.x + c * blockDim.x;
    if (i >= nvec) continue;
    const uint4 ww = wr[i];
    const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&v[c]);
    const __nv_bfloat16* wb = reinterpret_cast<const __nv_bfloat16*>(&ww);
    __align__(16) __nv_bfloat16 o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k)
      o[k] = __float2bfloat16(__bfloat162float(b[k]) * inv * __bfloat162float(wb[k]));
    dst[i] = *reinterpret_cast<uint4*>(o);
  }
}

// cos/sin of pos * inv_freq[j] for every token of the batch, computed once
// per forward and shared by all layers: table[t][j] = (cos, sin).
__global__ void rope_table_kernel(const int32_t* __restrict__ pos, const float* __restrict__ inv_freq,
                                  int half, float2* __restrict__ table) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x;
  const float p = static_cast<float>(pos[t]);
  for (int j = threadIdx.x; j < half; j += blockDim.x) {
    float sn, cs;
    sincosf(p * inv_freq[j], &sn, &cs);
    table[static_cast<size_t>(t) * half + j] = make_float2(cs, sn);
  }
}

// One token's RoPE + paged KV write. Work items: (q or k head, chunk pair p)
// rotates dims [8p, 8p+8) with [64+8p, 64+8p+8) (rotate-half, hd = 128)
// using 16 B vectors; q goes to qdst (the qkv row the attention reads), k and
// v go to the paged cache in its UMMA atom layout (kv_chunk_elem, device.cuh). `row` may live in global or shared memory.
__device__ __forceinline__ void rope_kv_token(const __nv_bfloat16* row, __nv_bfloat16* qdst, int s,
                                              const float2* __restrict__ cs, int n_heads, int n_kv_heads,
                                              int page_tokens, __nv_bfloat16* __restrict__ kplane,
                                              __nv_bfloat16* __restrict__ vplane) {
  constexpr int hd = 128, half = 64;
  const int page = s / page_tokens, off = s % page_tokens;
  const int rot_items = (n_heads + n_kv_heads) * 8;
  const int v_items = n_kv_heads * 16;
  for (int it = threadIdx.x; it < rot_items + v_items; it += blockDim.x) {
    if (it < rot_items) {
      const int head = it >> 3, p = it & 7;
      const __nv_bfloat16* h = row + head * hd;
      const uint4 va = *reinterpret_cast<const uint4*>(h + 8 * p);
      const uint4 vb = *reinterpret_cast<const uint4*>(h + half + 8 * p);
      const __nv_bfloat16* a = reinterpret_cast<const __nv_bfloat16*>(&va);
      const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&vb);
      __align__(16) __nv_bfloat16 ra[8], rb[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float2 c = cs[8 * p + i];
        const float x = __bfloat162float(a[i]), y = __bfloat162float(b[i]);
        ra[i] = __float2bfloat16(x * c.x - y * c.y);
        rb[i] = __float2bfloat16(y * c.x + x * c.y);
      }
      if (head < n_heads) {
        *reinterpret_cast<uint4*>(qdst + head * hd + 8 * p) = *reinterpret_cast<uint4*>(ra);
        *reinterpret_cast<uint4*>(qdst + head * hd + half + 8 * p) = *reinterpret_cast<uint4*>(rb);
      } else {
        __nv_bfloat16* dst =  // [page][kv head][K | V] blocks of 4 KB atoms (kv_chunk_elem)
            kplane + (static_cast<size_t>(page) * n_kv_heads + (head - n_heads)) * 2 * page_tokens * hd;
        *reinterpret_cast<uint4*>(dst + kv_chunk_elem(off, p)) = *reinterpret_cast<uint4*>(ra);
        *reinterpret_cast<uint4*>(dst + kv_chunk_elem(off, p + 8)) = *reinterpret_cast<uint4*>(rb);
      }
    } else {
      const int i = it - rot_items;
      const int kh = i >> 4, c = i & 15;
      const __nv_bfloat16* src = row + (n_heads + n_kv_heads + kh) * hd + c * 8;
      __nv_bfloat16* dst = vplane + (static_cast<size_t>(page) * n_kv_heads + kh) * 2 * page_tokens * hd;
      *reinterpret_cast<uint4*>(dst + kv_chunk_elem(off, c)) = *reinterpret_cast<const uint4*>(src);
    }
  }
}

// One CTA per token: RoPE on q (in place) and k, k/v -> paged cache.
__global__ void rope_kv_kernel(__nv_bfloat16* __restrict__ qkv, const int32_t* __restrict__ slot,
                               const float2* __restrict__ table, int n_heads, int n_kv_heads,
                               int page_tokens, __nv_bfloat16* __restrict__ kplane,
                               __nv_bfloat16* __restrict__ vplane) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x;
  __nv_bfloat16* row = qkv + static_cast<size_t>(t) * (n_heads + 2 * n_kv_heads) * 128;
  rope_kv_token(row, row, slot[t], table + static_cast<size_t>(t) * 64, n_heads, n_kv_heads, page_tokens,
                kplane, vplane);
}

// ---- consumers of deferred-fold GEMM planes ---------------------------------
// Sum of the fp32 partials of elements [row, row + 8) of token t, in piece
// order (deterministic for a given partition). The loads of up to 8 pieces
// are issued before the first add, so a fold costs one L2 round trip, not
// one per piece.
__device__ __forceinline__ void fold8(const GemmFold& f, int row, int t, float (&v)[8]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = 0.f;
  const int n = fold_pieces(f, row, t);
  const size_t plane = static_cast<size_t>(f.tokens) * f.rows;
  const float* src = f.planes + static_cast<size_t>(t) * f.rows + row;
  for (int q0 = 0; q0 < n; q0 += 8) {
    float4 a[8], b[8];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q0 + q < n) {
        a[q] = __ldcg(reinterpret_cast<const float4*>(src + (q0 + q) * plane));
        b[q] = __ldcg(reinterpret_cast<const float4*>(src + (q0 + q) * plane + 4));
      }
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q0 + q < n) {
        v[0] += a[q].x, v[1] += a[q].y, v[2] += a[q].z, v[3] += a[q].w;
        v[4] += b[q].x, v[5] += b[q].y, v[6] += b[q].z, v[7] += b[q].w;
      }
  }
}

// One CTA per token, one 8-feature chunk per thread (blockDim = hidden / 8,
// <= 512; kFoldVec chunks per thread beyond that).
constexpr int kFoldVec = 2;
__global__ void __launch_bounds__(512) fold_residual_rmsnorm_kernel(GemmFold f, __nv_bfloat16* __restrict__ x,
                                                                     const __nv_bfloat16* __restrict__ w, float eps,
                                                                     __nv_bfloat16* __restrict__ h) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x, d = f.rows;
  __nv_bfloat16* xr = x + static_cast<size_t>(t) * d;
  float keep[kFoldVec][8];
  float ss = 0.f;
#pragma unroll
  for (int c = 0; c < kFoldVec; ++c) {
    const int row = (threadIdx.x + c * blockDim.x) * 8;
    if (row >= d) break;
    float v[8];
    fold8(f, row, t, v);
    const uint4 rv = *reinterpret_cast<const uint4*>(xr + row);
    const __nv_bfloat16* rb = reinterpret_cast<const __nv_bfloat16*>(&rv);
    __align__(16) __nv_bfloat16 o[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      o[i] = __float2bfloat16(v[i] + __bfloat162float(rb[i]));  // the GEMM residual epilogue
      keep[c][i] = __bfloat162float(o[i]);
      ss += keep[c][i] * keep[c][i];
    }
    *reinterpret_cast<uint4*>(xr + row) = *reinterpret_cast<uint4*>(o);
  }
  if (w == nullptr) return;
  __shared__ float red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffff, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
  for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) tot += red[i];
  const float inv = rsqrtf(tot / d + eps);
  __nv_bfloat16* hr = h + static_cast<size_t>(t) * d;
#pragma unroll
  for (int c = 0; c < kFoldVec; ++c) {
    const int row = (threadIdx.x + c * blockDim.x) * 8;
    if (row >= d) break;
    const uint4 wv = *reinterpret_cast<const uint4*>(w + row);
    const __nv_bfloat16* wb = reinterpret_cast<const __nv_bfloat16*>(&wv);
    __align__(16) __nv_bfloat16 o[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = __float2bfloat16(keep[c][i] * inv * __bfloat162float(wb[i]));
    *reinterpret_cast<uint4*>(hr + row) = *reinterpret_cast<uint4*>(o);
  }
}

// out[t][r] = sum planes (fp32): the plain fold (tests, diagnostics).
__global__ void __launch_bounds__(256) fold_store_f32_kernel(GemmFold f, float* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.y;
  const int row = (blockIdx.x * 256 + threadIdx.x) * 8;
  if (row >= f.rows) return;
  float v[8];
  fold8(f, row, t, v);
  float4* dst = reinterpret_cast<float4*>(out + static_cast<size_t>(t) * f.rows + row);
  dst[0] = make_float4(v[0], v[1], v[2], v[3]);
  dst[1] = make_float4(v[4], v[5], v[6], v[7]);
}

__device__ __forceinline__ float silu_f(float g) { return g / (1.0f + __expf(-g)); }

// grid (ceil(ffn / 2048), tokens): thread = 8 consecutive outputs.
__global__ void __launch_bounds__(256) fold_swiglu_kernel(GemmFold f, __nv_bfloat16* __restrict__ act) {
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.y;
  const int ffn = f.rows / 2;
  const int j = (blockIdx.x * 256 + threadIdx.x) * 8;
  if (j >= ffn) return;
  const int rg = (j >> 6) * 128 + (j & 63);  // gate rows of 128-row block j / 64; up = +64
  float g[8], u[8];
  fold8(f, rg, t, g);  // the g and u loads are independent: both in flight
  fold8(f, rg + 64, t, u);
  __align__(16) __nv_bfloat16 o[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) o[i] = __float2bfloat16(silu_f(g[i]) * u[i]);
  *reinterpret_cast<uint4*>(act + static_cast<size_t>(t) * ffn + j) = *reinterpret_cast<uint4*>(o);
}

// One CTA per token: the qkv row is folded into shared memory (+ bias,
// rounded to bf16 exactly like the GEMM's bias/store epilogue), then RoPE
// and the paged KV write run on it.
__global__ void __launch_bounds__(512) fold_rope_kv_kernel(GemmFold f, const __nv_bfloat16* __restrict__ bias,
                                                           __nv_bfloat16* __restrict__ qkv,
                                                           const int32_t* __restrict__ slot,
                                                           const float2* __restrict__ table, int n_heads,
                                                           int n_kv_heads, int page_tokens,
                                                           __nv_bfloat16* __restrict__ kplane,
                                                           __nv_bfloat16* __restrict__ vplane) {
  extern __shared__ __align__(16) __nv_bfloat16 srow[];
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x;
  for (int row = threadIdx.x * 8; row < f.rows; row += blockDim.x * 8) {
    float v[8];
    fold8(f, row, t, v);
    if (bias) {
      const uint4 bv = *reinterpret_cast<const uint4*>(bias + row);
      const __nv_bfloat16* bb = reinterpret_cast<const __nv_bfloat16*>(&bv);
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] += __bfloat162float(bb[i]);
    }
    __align__(16) __nv_bfloat16 o[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = __float2bfloat16(v[i]);
    *reinterpret_cast<uint4*>(srow + row) = *reinterpret_cast<uint4*>(o);
  }
  __syncthreads();
  rope_kv_token(srow, qkv + static_cast<size_t>(t) * f.rows, slot[t], table + static_cast<size_t>(t) * 64,
                n_heads, n_kv_heads, page_tokens, kplane, vplane);
}

// Greedy sampling, two passes: kArgChunks CTAs per row reduce a slice of
// the vocabulary to one (value, index) pair; one warp per row folds them.
// Ties resolve to the lowest index (numpy argmax).
constexpr int kArgChunks = 16;

__device__ __forceinline__ void arg_better(float& best, int& idx, float v, int i) {
  if (v > best || (v == best && i < idx)) {
    best = v;
    idx = i;
  }
}

__global__ void argmax_partial_kernel(const float* __restrict__ logits, int ld, int valid,
                                      float2* __restrict__ part) {
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.y, chunk = blockIdx.x;
  const int per = (valid + kArgChunks - 1) / kArgChunks;
  const int lo = chunk * per, hi = min(valid, lo + per);
  const float* r = logits + static_cast<size_t>(row) * ld;
  float best = -FLT_MAX;
  int idx = 0x7fffffff;
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) arg_better(best, idx, r[i], i);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    arg_better(best, idx, __shfl_xor_sync(0xffffffff, best, o), __shfl_xor_sync(0xffffffff, idx, o));
  __shared__ float sv[32];
  __shared__ int si[32];
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = best;
    si[threadIdx.x >> 5] = idx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) arg_better(best, idx, sv[w], si[w]);
    part[row * kArgChunks + chunk] = make_float2(best, __int_as_float(idx));
  }
}

__global__ void argmax_final_kernel(const float2* __restrict__ part, int rows, int offset,
                                    int32_t* __restrict__ out, float2* __restrict__ pair_out) {
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  float best = -FLT_MAX;
  int idx = 0x7fffffff;
  if (lane < kArgChunks) {
    const float2 p = part[row * kArgChunks + lane];
    best = p.x;
    idx = __float_as_int(p.y);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    arg_better(best, idx, __shfl_xor_sync(0xffffffff, best, o), __shfl_xor_sync(0xffffffff, idx, o));
  if (lane == 0) {
    if (out) out[row] = idx + offset;
    if (pair_out) pair_out[row] = make_float2(best, __int_as_float(idx + offset));
  }
}

// TP: fold the all-gathered [tp][rows] (max, global idx) pairs.
__global__ void argmax_fold_kernel(const float2* __restrict__ pairs, int tp, int rows,
                                   int32_t* __restrict__ out) {
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= rows) return;
  float best = -FLT_MAX;
  int idx = 0x7fffffff;
  for (int r = 0; r < tp; ++r) {
    const float2 p = pairs[static_cast<size_t>(r) * rows + row];
    arg_better(best, idx, p.x, __float_as_int(p.y));
  }
  out[row] = idx;
}

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

__global__ void fill_random_kernel(__nv_bfloat16* p, size_t n, uint64_t seed, float scale,
                                   float offset) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const uint64_t h = mix64(seed ^ mix64(i));
    const float u = static_cast<float>(h >> 40) * (1.0f / 16777216.0f);  // [0, 1)
    p[i] = __float2bfloat16(offset + scale * (2.f * u - 1.f));
  }
}

// Row/column slice of a larger logical matrix: element (r, c) of the slice
// takes the value of global element (rowmap(r), col0 + c), so a TP shard holds
// exactly the corresponding entries of the unsharded model.
__global__ void fill_random_slice_kernel(__nv_bfloat16* p, int rows, int cols, RowMap m,
                                         size_t full_cols, size_t col0, uint64_t seed,
                                         float scale, float offset) {
  const size_t n = static_cast<size_t>(rows) * cols;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int lr = static_cast<int>(i / cols), c = static_cast<int>(i % cols);
    int sg = 0;
    for (int k = 1; k < m.nseg; ++k)
      if (lr >= m.local0[k]) sg = k;
    const size_t gr = static_cast<size_t>(m.global0[sg] + (lr - m.local0[sg]));
    const uint64_t h = mix64(seed ^ mix64(gr * full_cols + col0 + c));
    const float u = static_cast<float>(h >> 40) * (1.0f / 16777216.0f);
    p[i] = __float2bfloat16(offset + scale * (2.f * u - 1.f));
  }
}

}  // namespace

cudaError_t fill_random_slice(__nv_bfloat16* p, int rows, int cols, const RowMap& m,
                              size_t full_cols, size_t col0, uint64_t seed, float scale,
                              float offset, cudaStream_t s) {
  fill_random_slice_kernel<<<1184, 256, 0, s>>>(p, rows, cols, m, full_cols, col0, seed, scale,
                                                offset);
  return cudaGetLastError();
}

cudaError_t embed(const int32_t* tokens, int n, const __nv_bfloat16* table, int hidden,
                  __nv_bfloat16* out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  ++g_kernel_launches;
  return launch_pdl(embed_kernel, dim3(n), dim3(128), 0, s, tokens, table, hidden, out);
}

cudaError_t rmsnorm(const __nv_bfloat16* x, const int32_t* rows, int n, int hidden,
                    const __nv_bfloat16* w, float eps, __nv_bfloat16* out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  ++g_kernel_launches;
  if (hidden % 8 || hidden > kNormVec * 8 * 128) return cudaErrorInvalidValue;
  return launch_pdl(rmsnorm_kernel, dim3(n), dim3(128), 0, s, x, rows, hidden, w, eps, out);
}

cudaError_t rope_table(const int32_t* pos, int n_tokens, const float* inv_freq, int head_dim,
                       float2* table, cudaStream_t s) {
  if (n_tokens == 0) return cudaSuccess;
  ++g_kernel_launches;
  const cudaError_t e0 = launch_pdl(rope_table_kernel, dim3(n_tokens), dim3(64), 0, s, pos, inv_freq,
                                    head_dim / 2, table);
  if (e0 != cudaSuccess) return e0;
  return cudaGetLastError();
}

cudaError_t fold_residual_rmsnorm(const GemmFold& f, __nv_bfloat16* x, const __nv_bfloat16* w, float eps,
                                  __nv_bfloat16* h, cudaStream_t s) {
  if (f.tokens == 0) return cudaSuccess;
  if (f.rows % 256 || f.rows > 512 * 8 * kFoldVec) return cudaErrorInvalidValue;
  ++g_kernel_launches;
  return launch_pdl(fold_residual_rmsnorm_kernel, dim3(f.tokens), dim3(std::min(512, f.rows / 8)), 0, s, f, x, w,
                    eps, h);
}

cudaError_t fold_store_f32(const GemmFold& f, float* out, cudaStream_t s) {
  if (f.tokens == 0) return cudaSuccess;
  if (f.rows % 8) return cudaErrorInvalidValue;
  ++g_kernel_launches;
  return launch_pdl(fold_store_f32_kernel, dim3((f.rows + 2047) / 2048, f.tokens), dim3(256), 0, s, f, out);
}

cudaError_t fold_swiglu(const GemmFold& f, __nv_bfloat16* act, cudaStream_t s) {
  if (f.tokens == 0) return cudaSuccess;
  const int ffn = f.rows / 2;
  if (f.rows % 128) return cudaErrorInvalidValue;
  ++g_kernel_launches;
  return launch_pdl(fold_swiglu_kernel, dim3((ffn + 2047) / 2048, f.tokens), dim3(256), 0, s, f, act);
}

cudaError_t fold_rope_kv(const GemmFold& f, const __nv_bfloat16* bias, __nv_bfloat16* qkv,
                         const int32_t* slot, const float2* table, int n_heads, int n_kv_heads,
                         int page_tokens, __nv_bfloat16* kplane, __nv_bfloat16* vplane, cudaStream_t s) {
  if (f.tokens == 0) return cudaSuccess;
  if (f.rows != (n_heads + 2 * n_kv_heads) * 128) return cudaErrorInvalidValue;
  ++g_kernel_launches;
  return launch_pdl(fold_rope_kv_kernel, dim3(f.tokens), dim3(std::min(512, f.rows / 8)),
                    static_cast<size_t>(f.rows) * 2, s, f, bias,
                    qkv, slot, table, n_heads, n_kv_heads, page_tokens, kplane, vplane);
}

cudaError_t rope_kv_write(__nv_bfloat16* qkv, int n_tokens, const int32_t* slot,
                          const float2* table, int n_heads, int n_kv_heads, int head_dim,
                          int page_tokens, __nv_bfloat16* kplane, __nv_bfloat16* vplane,
                          cudaStream_t s) {
  if (n_tokens == 0) return cudaSuccess;
  if (head_dim != 128) return cudaErrorInvalidValue;
  ++g_kernel_launches;
  return launch_pdl(rope_kv_kernel, dim3(n_tokens), dim3(256), 0, s, qkv, slot, table, n_heads, n_kv_heads,
                    page_tokens, kplane, vplane);
}

cudaError_t argmax_rows(const float* logits, int n, int ld, int valid, int offset, int32_t* out,
                        float2* pair_out, float2* scratch, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  g_kernel_launches += 2;
  const cudaError_t e = launch_pdl(argmax_partial_kernel, dim3(kArgChunks, n), dim3(256), 0, s, logits, ld,
                                   valid, scratch);
  if (e != cudaSuccess) return e;
  return launch_pdl(argmax_final_kernel, dim3((n + 7) / 8), dim3(256), 0, s, scratch, n, offset, out, pair_out);
}

cudaError_t argmax_fold(const float2* pairs, int tp, int rows, int32_t* out, cudaStream_t s) {
  if (rows == 0) return cudaSuccess;
  ++g_kernel_launches;
  return launch_pdl(argmax_fold_kernel, dim3((rows + 127) / 128), dim3(128), 0, s, pairs, tp, rows, out);
}

cudaError_t fill_random(__nv_bfloat16* p, size_t n, uint64_t seed, float scale, float offset,
                        cudaStream_t s) {
  fill_random_kernel<<<1184, 256, 0, s>>>(p, n, seed, scale, offset);
  return cudaGetLastError();
}

bool encode_kmajor(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                   uint64_t row_stride_bytes, uint32_t box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        !fn)
      return false;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {row_stride_bytes};
  const cuuint32_t box[2] = {64, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

// Kernel loading is lazy by default (CUDA_MODULE_LOADING=LAZY): the first
// launch of a kernel loads its module, which can wait for the context to go
// idle. A TP rank spinning in a peer collective never lets it go idle, so
// every kernel (and its smem opt-in, which is per device) is prepared up
// front on each device the library runs on.
bool g_pdl = [] {
  const char* e = std::getenv("NX_PDL");
  return !(e && e[0] == '0');
}();

cudaError_t ensure_kernels_prepared() {
  static std::atomic<uint64_t> mask{0};
  static cudaError_t failed[64] = {};
  int d = 0;
  cudaGetDevice(&d);
  const uint64_t bit = 1ull << (d & 63);
  if (mask.load(std::memory_order_acquire) & bit) return failed[d & 63];
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (mask.load() & bit) return failed[d & 63];
  prepare_gemm_kernels();
  prepare_gemm_decode_kernel();
  prepare_gemm_pair_kernel();
  // a rejected smem opt-in would make every launch of that kernel fail later
  // with no clear cause: remember it and hand it to the launch wrappers
  failed[d & 63] = prepare_attention_kernels();
  prepare_tp_kernels();
  const void* fns[] = {reinterpret_cast<const void*>(fill_random_kernel),
                       reinterpret_cast<const void*>(fill_random_slice_kernel),
                       reinterpret_cast<const void*>(embed_kernel),
                       reinterpret_cast<const void*>(rmsnorm_kernel),
                       reinterpret_cast<const void*>(rope_table_kernel),
                       reinterpret_cast<const void*>(rope_kv_kernel),
                       reinterpret_cast<const void*>(fold_residual_rmsnorm_kernel),
                       reinterpret_cast<const void*>(fold_swiglu_kernel),
                       reinterpret_cast<const void*>(fold_store_f32_kernel),
                       reinterpret_cast<const void*>(fold_rope_kv_kernel),
                       reinterpret_cast<const void*>(argmax_partial_kernel),
                       reinterpret_cast<const void*>(argmax_final_kernel),
                       reinterpret_cast<const void*>(argmax_fold_kernel)};
  cudaFuncAttributes fa;
  for (const void* f : fns) cudaFuncGetAttributes(&fa, f);
  cudaGetLastError();
  mask.fetch_or(bit);
  return failed[d & 63];
}

}  // namespace nxd
