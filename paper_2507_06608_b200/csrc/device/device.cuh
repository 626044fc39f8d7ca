// Internal device API of the B200 executor (kernels + launch helpers).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace nxd {

// Count of kernels launched by this library (host-side, all streams).
extern unsigned long long g_kernel_launches;

// Programmatic dependent launch: every kernel of a forward is launched with
// programmatic stream serialization, calls pdl_trigger() on entry (its
// successor may be scheduled once all of its CTAs are resident) and
// pdl_wait() before touching anything an upstream kernel wrote. Work that
// needs no upstream data (barrier init, TMEM alloc, weight prefetch) runs
// in the shadow of the previous kernel. NX_PDL=0 disables it.
extern bool g_pdl;
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#endif
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Load every kernel and set its shared-memory opt-in on the current device
// (once per device; see kernels.cu).
cudaError_t ensure_kernels_prepared();
void prepare_gemm_kernels();
cudaError_t prepare_attention_kernels();
void prepare_tp_kernels();

// ---- GEMM (gemm_tc.cu) -------------------------------------------------------
enum EpiMode {
  kEpiStore = 0,         // out = acc (bf16)
  kEpiBias = 1,          // out = acc + bias
  kEpiResidual = 2,      // out = acc + residual (may alias out)
  kEpiBiasResidual = 3,  // out = acc + bias + residual
  kEpiSwiGLU = 4,        // out[f] = silu(acc[gate f]) * acc[up f]  (interleaved 64-row blocks)
  kEpiPartial = 5,       // internal: fp32 K-split partials
  kEpiF32 = 6,           // out = acc (fp32), e.g. logits
  kEpiRopeKV = 7,        // QKV: bf16(acc + bias) -> RoPE on q / k; q -> out, k / v -> paged cache (pair kernel)
};

struct GemmParams {
  int rows, tokens, K;
  int n_mblk, n_nblk, splits, kb_per_split, num_kb;
  int mode;
  void* out;
  int ldo;
  const __nv_bfloat16* bias;
  const __nv_bfloat16* residual;
  int ldr;
  float* ws;
  int streamk;     // 1: stream-K partition of the (tile, k-block) iterations
  int max_pieces;  // stream-K: partial slots per tile
  int bn;          // token tile (for the stream-K fix-up)
  int* tile_count; // stream-K: per-tile arrival counters (zero between launches)
  int n_tiles128;  // 128-row weight blocks (n_mblk counts MT-block work tiles)
  int coresident;  // stream-K: parallel reduce-scatter fix-up (see gemm())
  int dbg;         // experiments only (NX_GEMM_DBG): 1 skip X loads, 2 skip MMAs
  int fold;        // 1: every work item writes fp32 planes, no fix-up (see GemmFold)
  int sk_tile0;    // stream-K covers tiles [sk_tile0, tiles); earlier tiles run data-parallel
  int bn_rt;       // token tile width (MMA N) of this launch, <= the template BN
};

int gemm_pick_bn(int tokens);
// Experiments: copies the per-CTA milestone stamps (NX_GEMM_DBG & 16).
size_t gemm_trace_read(unsigned long long* host, size_t n);
// y[tokens, rows] = epi(x[tokens, K] . w[rows, K]^T). `x_map` must have been
// encoded with box rows == bn. sm_count sizes the persistent grid (the lane's
// green-context partition); force_splits > 0 overrides the K-split choice.
// Weights are used in the packed tile layout (pack_weights): each 128 x 64
// tile is a contiguous, pre-swizzled 16 KB chunk streamed by cp.async.bulk.
size_t packed_weight_elems(int rows, int K);
cudaError_t pack_weights(const __nv_bfloat16* src, __nv_bfloat16* dst, int rows, int K,
                         cudaStream_t s);
cudaError_t unpack_weights(const __nv_bfloat16* src, __nv_bfloat16* dst, int rows, int K,
                           cudaStream_t s);
// ws must start with gemm_counter_bytes() of zeroed int counters (kept zero
// by the kernel itself between launches on the same stream).
// Deferred-fold output of a decode-shaped GEMM: instead of a cross-CTA
// fix-up inside the GEMM (a chain of dependent global round trips, ~5 us of
// its critical path), every work item writes its fp32 accumulator to plane
// `piece` ([piece][tokens][rows]) and the consumer kernel (fold_*) sums the
// planes of each element in piece order, applying the epilogue there.
struct GemmFold {
  const float* planes = nullptr;
  int rows = 0, tokens = 0;
  int kind = 0;      // 0: one plane; 1: `splits` uniform K splits; 2: stream-K pieces
  int splits = 1;
  int n_nblk = 1, num_kb = 1, grid = 1, rows_per_blk = 128, bn = 32;
  long long total = 1;  // stream-K (tile, k-block) iterations
};
#ifdef __CUDACC__
// Number of planes holding a partial of element (row, token t).
__device__ __forceinline__ int fold_pieces(const GemmFold& f, int row, int t) {
  if (f.kind == 0) return 1;
  if (f.kind == 1) return f.splits;
  const int tile = (row / f.rows_per_blk) * f.n_nblk + t / f.bn;
  const long long it0 = static_cast<long long>(tile) * f.num_kb;
  const int first = static_cast<int>(((it0 + 1) * f.grid - 1) / f.total);
  const int last = static_cast<int>(((it0 + f.num_kb) * f.grid - 1) / f.total);
  return last - first + 1;
}
#endif
// fold != nullptr: deferred-fold mode (mode/out/bias/residual are ignored;
// the consumer applies them); *fold describes the planes written.
cudaError_t gemm(const __nv_bfloat16* w_packed, const CUtensorMap& x_map, int bn, int rows, int tokens,
                 int K, int mode, void* out, int ldo, const __nv_bfloat16* bias,
                 const __nv_bfloat16* residual, int ldr, float* ws, size_t ws_bytes, int sm_count,
                 cudaStream_t stream, int force_splits = 0, bool coresident = false,
                 GemmFold* fold = nullptr);
// coresident: the launch owns its SMs (green-context partition, or nothing
// else running), so every CTA of the persistent grid is resident at once and
// stream-K pieces may wait for each other (parallel fix-up); otherwise the
// last arriving piece folds the tile alone.
constexpr size_t gemm_counter_bytes() { return 64 * 1024; }
// Decode-shaped GEMM (tokens <= 128; gemm_decode.cu): tokens are the MMA's
// M = 128 side and 256 weight rows its N side (the tensor floor for small
// token counts). fold != nullptr: fp32 planes for a fold_* consumer (ws as
// for gemm()); otherwise fp32 out[t * ldo + f] (lm_head logits). x_map's
// box must hold box_rows <= 128 token rows.
cudaError_t gemm_decode(const __nv_bfloat16* w_packed, const CUtensorMap& x_map, int box_rows, int rows,
                        int tokens, int K, float* out, int ldo, float* ws, size_t ws_bytes, int sm_count,
                        cudaStream_t stream, GemmFold* fold);
void prepare_gemm_decode_kernel();
// Prefill GEMM on CTA pairs (cta_group::2, gemm_tc2.cu): 256 weight rows x 256
// tokens per pair, each CTA staging half of the activation tile. x_map128 is
// the activations' K-major map with 128-row boxes. The forward uses it for every
// prefill-shaped GEMM unless NX_GEMM_2CTA=0 (gemm_pair_enabled()).
bool gemm_pair_enabled();
bool gemm_bn_fit_enabled();  // runtime prefill token-tile width (NX_BN_FIT=0: always 256)
// kEpiRopeKV: the QKV projection's epilogue also applies RoPE and writes k / v
// into the paged cache (`rope` describes it), so no separate RoPE kernel runs.
struct RopeKV {
  const int32_t* slot = nullptr;   // per token: page * page_tokens + offset
  const float2* table = nullptr;   // [tokens][64] (cos, sin)
  __nv_bfloat16* kplane = nullptr; // layer K view ([page][kv head][K | V][page_tokens][128])
  __nv_bfloat16* vplane = nullptr; // layer V view (kplane + page_tokens * 128)
  int n_heads = 0, n_kv_heads = 0, page_tokens = 16;
};
cudaError_t gemm_pair(const __nv_bfloat16* w_packed, const CUtensorMap& x_map128, int rows, int tokens, int K,
                      int mode, void* out, int ldo, const __nv_bfloat16* bias, const __nv_bfloat16* residual, int ldr,
                      int sm_count, cudaStream_t stream, const RopeKV* rope = nullptr);
void prepare_gemm_pair_kernel();
constexpr int kGemmMaxCounterTiles = 8192;  // [arrive | depart] int counters

// K-major bf16 [rows, cols] tensor map with a 64 x box_rows, 128B-swizzled box.
bool encode_kmajor(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols,
                   uint64_t row_stride_bytes, uint32_t box_rows);

// ---- attention (attention.cu) ----------------------------------------------
struct AttnGeom {
  int n_heads, n_kv_heads, group, head_dim;
  int page_tokens;
  int qkv_stride;  // elements per token row of the qkv buffer
  int out_stride;  // elements per token row of the attention output
  float scale_log2;
};

// Paged KV cache, per layer [page][kv head][K | V] blocks of 16 token rows
// x 128 dims (8 KB). Each K (V) half is 4 KB = four 1 KB SWIZZLE_128B atoms:
// atom (r / 8, c / 8) -- 8 token rows x 64 dims -- sits at (2 (r / 8) + c / 8)
// KB, and 16 B chunk c of token row r at kv_chunk_elem(r, c) (elements).
// The K (V) halves of consecutive pages copied 4 KB apart into shared memory
// form one uniform UMMA operand (8-token atoms 2 KB apart, 64-dim halves
// 1 KB apart): K-major for S = Q K^T, MN-major for O = P V.
__host__ __device__ __forceinline__ int kv_chunk_elem(int r, int c) {
  return ((((r >> 3) << 1) | (c >> 3)) << 9) + ((r & 7) << 6) + ((((c & 7) ^ (r & 7))) << 3);
}

struct AttnSeq {
  int q_start;   // first row of this sequence in the batch
  int q_len;     // new tokens this launch
  int kv_len;    // keys after this launch (start + q_len)
  int page_off;  // offset of the sequence's page list in the batch page array
};

// Prefill attention (attn_prefill.cu, tcgen05): work[i] = {sequence index,
// first token} of items of prefill_attn_tokens_per_item(group) tokens (x G
// heads = up to 128 query rows), longest first; qmap = encode_q_heads_map over
// the lane's qkv buffer; kvplane = the layer's [page][kv head][K | V] blocks.
int prefill_attn_tokens_per_item(int group);
bool encode_q_heads_map(CUtensorMap* map, const void* qkv, int tokens, int n_heads, int group,
                        int row_stride_elems);
cudaError_t prefill_attention(const AttnGeom& g, const CUtensorMap& qmap, const __nv_bfloat16* kvplane,
                              const AttnSeq* seqs, const int2* work, int n_work, const int32_t* pages,
                              __nv_bfloat16* out, int sm_count, cudaStream_t s);
cudaError_t prepare_prefill_attention_kernel();
// Decode attention over 32-key tiles (kDecTileKeys): seq_prefix[s] = first
// tile of sequence s, sum_{s' < s} ceil(kv_len(s') / 32) (n_seq + 1 entries,
// device memory); total_tiles = seq_prefix[n_seq] * n_kv_heads.
constexpr int kDecTileKeys = 32;
cudaError_t decode_attention(const AttnGeom& g, const __nv_bfloat16* qkv,
                             const __nv_bfloat16* kplane, const __nv_bfloat16* vplane,
                             const AttnSeq* seqs, int n_seq, const int* seq_prefix,
                             long long total_tiles, int max_seq_tiles, const int32_t* pages,
                             __nv_bfloat16* out, float* part_o, float* part_ml, size_t part_cap,
                             int* item_done, int sm_count, cudaStream_t s);

// ---- elementwise / norm / sampling (kernels.cu) ----------------------------
cudaError_t embed(const int32_t* tokens, int n, const __nv_bfloat16* table, int hidden,
                  __nv_bfloat16* out, cudaStream_t s);
// out[r] = x[rows ? rows[r] : r] * rsqrt(mean(x^2) + eps) * w
cudaError_t rmsnorm(const __nv_bfloat16* x, const int32_t* rows, int n, int hidden,
                    const __nv_bfloat16* w, float eps, __nv_bfloat16* out, cudaStream_t s);
// Per-batch RoPE cos/sin table [n_tokens][head_dim / 2].
cudaError_t rope_table(const int32_t* pos, int n_tokens, const float* inv_freq, int head_dim,
                       float2* table, cudaStream_t s);
// Rotary embedding on q and k (rotate-half pairs), then k, v -> paged cache
// in the pre-swizzled page layout the attention kernels bulk-copy.
// Consumers of deferred-fold GEMM planes (one launch each, PDL):
//  x = bf16(x + sum planes); h = rmsnorm(x) * w (skipped when w == nullptr)
cudaError_t fold_residual_rmsnorm(const GemmFold& f, __nv_bfloat16* x, const __nv_bfloat16* w, float eps,
                                  __nv_bfloat16* h, cudaStream_t s);
//  out[t][r] = sum planes (fp32)
cudaError_t fold_store_f32(const GemmFold& f, float* out, cudaStream_t s);
//  act[t][64 b + i] = silu(sum gate row 128 b + i) * (sum up row 128 b + 64 + i)
cudaError_t fold_swiglu(const GemmFold& f, __nv_bfloat16* act, cudaStream_t s);
//  qkv row = bf16(sum planes + bias), then RoPE + paged KV write as rope_kv_write
cudaError_t fold_rope_kv(const GemmFold& f, const __nv_bfloat16* bias, __nv_bfloat16* qkv,
                         const int32_t* slot, const float2* table, int n_heads, int n_kv_heads,
                         int page_tokens, __nv_bfloat16* kplane, __nv_bfloat16* vplane, cudaStream_t s);
cudaError_t rope_kv_write(__nv_bfloat16* qkv, int n_tokens, const int32_t* slot,
                          const float2* table, int n_heads, int n_kv_heads, int head_dim,
                          int page_tokens, __nv_bfloat16* kplane, __nv_bfloat16* vplane,
                          cudaStream_t s);
// out[r] = offset + argmax_{j < valid} logits[r * ld + j] (lowest index on
// ties); pair_out (optional) gets (max, offset + argmax); scratch holds 16
// float2 per row.
cudaError_t argmax_rows(const float* logits, int n, int ld, int valid, int offset, int32_t* out,
                        float2* pair_out, float2* scratch, cudaStream_t s);
// TP: fold all-gathered [tp][rows] (max, global idx) pairs into tokens.
cudaError_t argmax_fold(const float2* pairs, int tp, int rows, int32_t* out, cudaStream_t s);
// Deterministic random bf16 fill: uniform(-scale, scale) + offset from a hash of (seed, i).
// Local row r of a slice maps to global row global0[k] + (r - local0[k]) for
// the last segment k with local0[k] <= r (QKV shards have three segments).
struct RowMap {
  int nseg = 1;
  int local0[3] = {0, 0, 0};
  long long global0[3] = {0, 0, 0};
};
cudaError_t fill_random_slice(__nv_bfloat16* p, int rows, int cols, const RowMap& m,
                              size_t full_cols, size_t col0, uint64_t seed, float scale,
                              float offset, cudaStream_t s);
cudaError_t fill_random(__nv_bfloat16* p, size_t n, uint64_t seed, float scale, float offset,
                        cudaStream_t s);

}  // namespace nxd
