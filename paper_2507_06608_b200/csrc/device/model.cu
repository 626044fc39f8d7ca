// The device executor: model weights, paged KV cache, per-lane workspaces,
// green-context SM layouts, and the forward pass of one scheduled batch.
//
// One lane's batch = one launch sequence on the lane's stream:
//   H2D(metadata) -> embed -> L x [rmsnorm, QKV gemm, rope+KV write,
//   paged attention, O gemm(+residual), rmsnorm, gate/up gemm(SwiGLU),
//   down gemm(+residual)] -> rmsnorm(sampled rows) -> lm_head gemm (fp32)
//   -> argmax -> D2H(tokens)
// bracketed by CUDA events; the host engine polls the end event.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <initializer_list>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "device.cuh"
#include "model.cuh"

namespace nxd {

namespace {
void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
}  // namespace

// ---------------------------------------------------------------------------
// Green-context layouts.
// ---------------------------------------------------------------------------
void Partitions::init(int device, bool enable) {
  cudaDeviceProp prop{};
  ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  total_sm = prop.multiProcessorCount;
  ck(cudaStreamCreateWithFlags(&full_stream, cudaStreamNonBlocking), "stream");
  ck(cudaStreamCreateWithFlags(&plain_stream[0], cudaStreamNonBlocking), "stream");
  ck(cudaStreamCreateWithFlags(&plain_stream[1], cudaStreamNonBlocking), "stream");
  // Kernels launched on green-context streams cannot be replayed by Nsight
  // Compute (the profiled process dies at the first such launch). Under a
  // profiler's injection library the lanes therefore run on plain streams
  // (same kernels, no SM partitions) unless NX_GREEN_UNDER_PROFILER=1.
  const bool profiler = std::getenv("NV_NSIGHT_INJECTION_TRANSPORT_TYPE") ||
                        std::getenv("NV_COMPUTE_PROFILER_PERFWORKS_DIR") || std::getenv("CUDA_INJECTION64_PATH");
  if (const char* e = std::getenv("NX_GREEN"); e && e[0] == '0') enable = false;  // plain streams (tools)
  if (enable && profiler && !std::getenv("NX_GREEN_UNDER_PROFILER")) {
    std::fprintf(stderr, "nexus_b200: profiler injection detected, green-context partitions disabled\n");
    enable = false;
  }
  if (!enable) return;
  auto sym = [](const char* name) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || !p)
      throw std::runtime_error(std::string("driver entry point missing: ") + name);
    return p;
  };
  auto get_res = reinterpret_cast<PFN_cuDeviceGetDevResource>(sym("cuDeviceGetDevResource"));
  auto split = reinterpret_cast<PFN_cuDevSmResourceSplitByCount>(sym("cuDevSmResourceSplitByCount"));
  auto gen = reinterpret_cast<PFN_cuDevResourceGenerateDesc>(sym("cuDevResourceGenerateDesc"));
  auto create = reinterpret_cast<PFN_cuGreenCtxCreate>(sym("cuGreenCtxCreate"));
  auto mkstream = reinterpret_cast<PFN_cuGreenCtxStreamCreate>(sym("cuGreenCtxStreamCreate"));
  auto get_dev = reinterpret_cast<PFN_cuDeviceGet>(sym("cuDeviceGet"));
  CUdevice dev;
  if (get_dev(&dev, device) != CUDA_SUCCESS) throw std::runtime_error("cuDeviceGet");
  CUdevResource all;
  if (get_res(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS)
    throw std::runtime_error("cuDeviceGetDevResource");
  auto add_layout = [&](const CUdevResource* dec, unsigned n_dec, const CUdevResource* pre, unsigned n_pre) {
    CUdevResourceDesc dg, dr;
    CUgreenCtx gg, gr;
    CUstream sg, sr;
    if (gen(&dg, const_cast<CUdevResource*>(dec), n_dec) != CUDA_SUCCESS ||
        gen(&dr, const_cast<CUdevResource*>(pre), n_pre) != CUDA_SUCCESS ||
        create(&gg, dg, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
        create(&gr, dr, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
        mkstream(&sg, gg, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS ||
        mkstream(&sr, gr, CU_STREAM_NON_BLOCKING, 0) != CUDA_SUCCESS)
      throw std::runtime_error("green context creation failed");
    Layout l;
    for (unsigned i = 0; i < n_dec; ++i) l.decode_sms += static_cast<int>(dec[i].sm.smCount);
    for (unsigned i = 0; i < n_pre; ++i) l.prefill_sms += static_cast<int>(pre[i].sm.smCount);
    l.decode_stream = reinterpret_cast<cudaStream_t>(sg);
    l.prefill_stream = reinterpret_cast<cudaStream_t>(sr);
    layouts.push_back(l);
  };
  // Decode lane takes a group of 8k SMs (the green-context granularity on
  // sm_90+), the prefill lane the remaining SMs of the same split.
  for (int k = 1; 8 * k + 8 <= static_cast<int>(all.sm.smCount) && k <= 31; ++k) {
    CUdevResource grp, rest;
    unsigned n = 1;
    if (split(&grp, &n, &all, &rest, 0, 8 * k) != CUDA_SUCCESS || n != 1) break;
    add_layout(&grp, 1, &rest, 1);
  }
  enabled = !layouts.empty();
}

// Percent -> partition: the integer share maps to an SM target share/100 *
// total_sm and the layout whose lane size is nearest wins (ties: fewer SMs).
Partitions::Pick Partitions::pick(int lane_kind, int sm_pct) const {
  Pick p;
  if (lane_kind == 3 /*mixed*/ || !enabled || sm_pct >= 100) {
    p.stream = (lane_kind == 3 || (enabled && sm_pct >= 100)) ? full_stream
                                                               : plain_stream[lane_kind == 2 ? 1 : 0];
    p.sm_count = total_sm;
    p.layout = -1;
    p.exclusive = enabled || lane_kind == 3;
    return p;
  }
  const double target = sm_pct / 100.0 * total_sm;
  int best = 0;
  double best_err = 1e30;
  for (size_t i = 0; i < layouts.size(); ++i) {
    const int sms = lane_kind == 2 ? layouts[i].decode_sms : layouts[i].prefill_sms;
    const double err = std::fabs(sms - target);
    if (err < best_err - 1e-9) {
      best_err = err;
      best = static_cast<int>(i);
    }
  }
  const Layout& l = layouts[best];
  p.stream = lane_kind == 2 ? l.decode_stream : l.prefill_stream;
  p.sm_count = lane_kind == 2 ? l.decode_sms : l.prefill_sms;
  p.layout = best;
  p.exclusive = true;
  return p;
}

// ---------------------------------------------------------------------------
// Model.
// ---------------------------------------------------------------------------
namespace {
// Makes `dev` current for the scope (ranks of one process live on several GPUs).
struct DevGuard {
  int prev = -1, dev;
  explicit DevGuard(int d) : dev(d) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DevGuard() {
    if (prev >= 0 && prev != dev) cudaSetDevice(prev);
  }
};
}  // namespace

Model::Model(const nx_device_config& cfg, std::shared_ptr<PeerGroup> group)
    : cfg_(cfg), a_(cfg.arch), group_(std::move(group)), dev_(cfg.device) {
  if (a_.head_dim != 128) throw std::invalid_argument("head_dim must be 128");
  if (a_.hidden % 128 || a_.ffn % 64 || a_.vocab % 128 || (2 * a_.ffn) % 128)
    throw std::invalid_argument("hidden/vocab must be multiples of 128, ffn of 64");
  if (a_.n_heads % a_.n_kv_heads || a_.n_heads / a_.n_kv_heads > 8)
    throw std::invalid_argument("GQA group must divide heads and be <= 8");
  if (cfg.page_tokens != 16 || cfg.num_pages < 1)
    throw std::invalid_argument("page_tokens must be 16 (8 KB pre-swizzled K|V blocks)");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= cfg.device)
    throw NoDevice("no CUDA device");
  ck(cudaSetDevice(cfg.device), "cudaSetDevice");
  cudaDeviceProp prop{};
  ck(cudaGetDeviceProperties(&prop, cfg.device), "props");
  if (prop.major != 10) throw NoDevice("sm_100 device required");
  ensure_kernels_prepared();
  parts_.init(cfg.device, cfg.green_contexts != 0);
  tp_ = cfg.tp_size > 1 ? cfg.tp_size : 1;
  rank_ = tp_ > 1 ? cfg.tp_rank : 0;
  const nx_tp_shard sh = tp_plan(a_, tp_, rank_);
  hq_ = sh.n_q_heads;
  hkv_ = sh.n_kv_heads;
  ffn_ = sh.ffn_local;
  vocab_l_ = tp_ > 1 ? sh.vocab_local : a_.vocab;
  vocab_valid_ = tp_ > 1 ? sh.vocab_valid : a_.vocab;
  vocab0_ = tp_ > 1 ? sh.vocab0 : 0;
  const bool peer_mode = tp_ > 1 && (cfg.tp_mode == NX_TP_PEER || cfg.tp_mode == NX_TP_PEER_COLOCATED);
  if (tp_ > 1 && !peer_mode) {
    if (cfg.tp_mode != NX_TP_NCCL) throw std::invalid_argument("unknown tp_mode");
    Nccl& nc = Nccl::get();
    comm_[0] = nc.comm_init(tp_, cfg.nccl_id[0], rank_);
    comm_[1] = nc.comm_init(tp_, cfg.nccl_id[1], rank_);
  }
  if (peer_mode && !group_) {
    // rank 0 of a one-process group: owns the group and builds ranks 1..tp-1
    if (cfg.tp_rank != 0) throw std::invalid_argument("peer TP group is created through rank 0");
    if (cfg.tp_mode == NX_TP_PEER && cfg.device + tp_ > ndev)
      throw NoDevice("NX_TP_PEER needs tp_size GPUs starting at `device`");
    group_ = std::make_shared<PeerGroup>(tp_, cfg.tp_mode == NX_TP_PEER_COLOCATED);
  }
  qkv_rows_ = (hq_ + 2 * hkv_) * a_.head_dim;
  attn_cols_ = hq_ * a_.head_dim;
  alloc_weights();
  alloc_kv();
  lanes_[0].init(this, cfg.max_prefill_tokens);
  lanes_[1].init(this, cfg.max_decode_batch);
  lanes_[0].slot_index = 0;
  lanes_[1].slot_index = 1;
  if (group_) {
    group_->register_lane(rank_, 0, static_cast<size_t>(lanes_[0].t_max) * a_.hidden);
    group_->register_lane(rank_, 1, static_cast<size_t>(lanes_[1].t_max) * a_.hidden);
  }
  // RoPE inverse frequencies theta^(-2i/hd), computed in double, stored fp32.
  std::vector<float> inv(a_.head_dim / 2);
  for (int i = 0; i < a_.head_dim / 2; ++i)
    inv[i] = static_cast<float>(std::pow(static_cast<double>(a_.rope_theta),
                                         -2.0 * i / static_cast<double>(a_.head_dim)));
  ck(cudaMalloc(&inv_freq_, inv.size() * sizeof(float)), "malloc inv_freq");
  ck(cudaMemcpy(inv_freq_, inv.data(), inv.size() * sizeof(float), cudaMemcpyHostToDevice),
     "copy inv_freq");
  ck(cudaDeviceSynchronize(), "init sync");
  if (group_ && rank_ == 0) {
    for (int r = 1; r < tp_; ++r) {
      nx_device_config c = cfg_;
      c.tp_rank = r;
      if (cfg_.tp_mode == NX_TP_PEER) c.device = cfg_.device + r;
      peers_.push_back(std::make_unique<Model>(c, group_));
    }
    if (cfg_.tp_mode == NX_TP_PEER)  // every rank reads every other rank's slots
      for (int i = 0; i < tp_; ++i) {
        ck(cudaSetDevice(cfg_.device + i), "cudaSetDevice");
        for (int j = 0; j < tp_; ++j) {
          if (i == j) continue;
          int ok = 0;
          ck(cudaDeviceCanAccessPeer(&ok, cfg_.device + i, cfg_.device + j), "peer query");
          if (!ok) throw NoDevice("GPUs of the TP group lack peer access");
          const cudaError_t e = cudaDeviceEnablePeerAccess(cfg_.device + j, 0);
          if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
          else ck(e, "enable peer access");
        }
      }
    ck(cudaSetDevice(dev_), "cudaSetDevice");
  }
}

void Model::all_reduce(LaneWs& ws, __nv_bfloat16* x, size_t n) {
  if (group_) group_->all_reduce_bf16(rank_, ws.slot_index, x, n, ws.sm_count, ws.stream);
  else Nccl::get().all_reduce_bf16(comm_[ws.slot_index], x, n, ws.stream);
}

Model::~Model() {
  peers_.clear();
  DevGuard g(dev_);
  cudaDeviceSynchronize();
  for (void* c : comm_)
    if (c) Nccl::get().destroy(c);
  if (group_) group_->release_rank(rank_);
  for (void* p : allocs_) cudaFree(p);
  for (auto& l : lanes_) l.release();
}

__nv_bfloat16* Model::dalloc_bf16(size_t n) {
  void* p = nullptr;
  ck(cudaMalloc(&p, n * 2), "cudaMalloc");
  allocs_.push_back(p);
  return static_cast<__nv_bfloat16*>(p);
}

void Model::alloc_weights() {
  const size_t d = a_.hidden, L = a_.n_layers;
  // Same seed sequence on every rank: a TP shard is generated as the exact
  // slice of the unsharded model's tensors (fill_random_slice).
  uint64_t seed = cfg_.weight_seed;
  auto next_seed = [&]() { return seed = seed * 6364136223846793005ULL + 1442695040888963407ULL; };
  const float g = cfg_.weight_gain > 0 ? cfg_.weight_gain : 1.0f;
  auto uni = [&](size_t k) { return g * std::sqrt(3.0f / static_cast<float>(k)); };
  const nx_tp_shard sh = tp_plan(a_, tp_, rank_);
  const int hd = a_.head_dim;
  // row maps of the column-parallel tensors
  RowMap qkv_map;  // [q heads | k heads | v heads] -> this rank's heads of each
  qkv_map.nseg = 3;
  qkv_map.local0[1] = hq_ * hd;
  qkv_map.local0[2] = (hq_ + hkv_) * hd;
  qkv_map.global0[0] = static_cast<long long>(sh.q_head0) * hd;
  qkv_map.global0[1] = static_cast<long long>(a_.n_heads + sh.kv_head0) * hd;
  qkv_map.global0[2] = static_cast<long long>(a_.n_heads + a_.n_kv_heads + sh.kv_head0) * hd;
  RowMap gu_map;  // 128-row blocks of (64 gate | 64 up) features
  gu_map.global0[0] = 2LL * sh.ffn0;
  RowMap lm_map;
  lm_map.global0[0] = sh.vocab0;
  const RowMap whole;
  // staging buffer for the logical (row-major) random init before packing
  const size_t max_mat = std::max({static_cast<size_t>(qkv_rows_) * d, d * attn_cols_,
                                   2 * static_cast<size_t>(ffn_) * d,
                                   static_cast<size_t>(vocab_l_) * d});
  __nv_bfloat16* stage = nullptr;
  ck(cudaMalloc(&stage, max_mat * 2), "weight staging");
  auto plain = [&](size_t n, float scale, float offset, const RowMap& m = RowMap()) {
    __nv_bfloat16* p = dalloc_bf16(n);
    ck(fill_random_slice(p, static_cast<int>(n), 1, m, 1, 0, next_seed(), scale, offset, nullptr),
       "init weights");
    weight_bytes_ += n * 2;
    return p;
  };
  auto packed = [&](int rows, int K, float scale, const RowMap& m, size_t full_k, size_t k0) {
    const size_t n = static_cast<size_t>(rows) * K;
    ck(fill_random_slice(stage, rows, K, m, full_k, k0, next_seed(), scale, 0.f, nullptr),
       "init weights");
    __nv_bfloat16* p = dalloc_bf16(packed_weight_elems(rows, K));
    ck(pack_weights(stage, p, rows, K, nullptr), "pack weights");
    weight_bytes_ += n * 2;
    return p;
  };
  emb_ = dalloc_bf16(static_cast<size_t>(a_.vocab) * d);
  ck(fill_random(emb_, static_cast<size_t>(a_.vocab) * d, next_seed(), 1.0f, 0.f, nullptr),
     "init weights");
  weight_bytes_ += static_cast<size_t>(a_.vocab) * d * 2;
  const size_t q_cols = static_cast<size_t>(a_.n_heads) * hd;
  layers_.resize(L);
  for (size_t l = 0; l < L; ++l) {
    LayerW& w = layers_[l];
    w.attn_norm = plain(d, 0.1f, 1.0f);
    w.qkv = packed(qkv_rows_, static_cast<int>(d), uni(d), qkv_map, d, 0);
    w.qkv_bias = a_.qkv_bias ? plain(qkv_rows_, 0.1f, 0.f, qkv_map) : nullptr;
    w.o = packed(static_cast<int>(d), attn_cols_, uni(q_cols), whole, q_cols,
                 static_cast<size_t>(sh.q_head0) * hd);
    w.ffn_norm = plain(d, 0.1f, 1.0f);
    w.gate_up = packed(2 * ffn_, static_cast<int>(d), uni(d), gu_map, d, 0);
    w.down = packed(static_cast<int>(d), ffn_, uni(a_.ffn) * 2.0f, whole, a_.ffn, sh.ffn0);
  }
  final_norm_ = plain(d, 0.1f, 1.0f);
  const float lm_gain = cfg_.lm_head_gain > 0 ? cfg_.lm_head_gain : 1.0f;
  lm_head_ = packed(vocab_l_, static_cast<int>(d), lm_gain * std::sqrt(3.0f / d), lm_map, d, 0);
  ck(cudaDeviceSynchronize(), "weights");
  cudaFree(stage);
}

void Model::alloc_kv() {
  plane_elems_ = static_cast<size_t>(cfg_.num_pages) * hkv_ * cfg_.page_tokens *
                 a_.head_dim;
  const size_t total = plane_elems_ * 2 * a_.n_layers;
  kv_ = dalloc_bf16(total);
  ck(cudaMemset(kv_, 0, total * 2), "kv memset");  // stale pages stay finite
  kv_bytes_ = total * 2;
}

// ---------------------------------------------------------------------------
// Per-lane workspace.
// ---------------------------------------------------------------------------
void LaneWs::init(Model* m, int max_tokens) {
  const nx_arch& a = m->a_;
  t_max = std::max(max_tokens, 1);
  const size_t T = t_max;
  auto alloc = [&](size_t bytes) {
    void* p = nullptr;
    ck(cudaMalloc(&p, align_up(bytes, 256)), "lane alloc");
    owned.push_back(p);
    return p;
  };
  x = static_cast<__nv_bfloat16*>(alloc(T * a.hidden * 2));
  h = static_cast<__nv_bfloat16*>(alloc(T * a.hidden * 2));
  qkv = static_cast<__nv_bfloat16*>(alloc(T * m->qkv_rows_ * 2));
  attn = static_cast<__nv_bfloat16*>(alloc(T * m->attn_cols_ * 2));
  act = static_cast<__nv_bfloat16*>(alloc(T * m->ffn_ * 2));
  sample_cap = std::min<int>(t_max, 256);
  hs = static_cast<__nv_bfloat16*>(alloc(static_cast<size_t>(sample_cap) * a.hidden * 2));
  logits = static_cast<float*>(alloc(static_cast<size_t>(sample_cap) * m->vocab_l_ * 4));
  out_dev = alloc(T * 4);
  tp_pairs = static_cast<float2*>(alloc(static_cast<size_t>(sample_cap) * (m->tp_ + 1) * sizeof(float2)));
  rope_cs = static_cast<float2*>(alloc(T * (a.head_dim / 2) * sizeof(float2)));
  ws_bytes = 96u << 20;
  ws = static_cast<float*>(alloc(ws_bytes));
  ck(cudaMemset(ws, 0, gemm_counter_bytes()), "zero gemm counters");
  part_cap = static_cast<size_t>(8) << 20;  // floats
  part_o = static_cast<float*>(alloc(part_cap * 4));
  part_ml = static_cast<float*>(alloc(part_cap / a.head_dim * 2 * 4 + 1024));
  item_done = static_cast<int*>(alloc(static_cast<size_t>(T) * m->hkv_ * 4));
  ck(cudaMemset(item_done, 0, static_cast<size_t>(T) * m->hkv_ * 4), "item counters");
  // metadata (device + pinned mirror)
  meta_bytes = align_up(T * 12 + T * 16 + T * 8 + (static_cast<size_t>(T) + 1) * 4 * 64 +
                            static_cast<size_t>(m->cfg_.num_pages) * 4 + 4096,
                        4096);
  meta_dev = static_cast<uint8_t*>(alloc(meta_bytes));
  ck(cudaMallocHost(&meta_host, meta_bytes), "pinned meta");
  ck(cudaMallocHost(&out_host, static_cast<size_t>(T) * 4), "pinned out");
  ck(cudaEventCreate(&ev_start), "event");
  ck(cudaEventCreate(&ev_end), "event");
  ev_pool.resize(2048);
  for (auto& e : ev_pool) ck(cudaEventCreate(&e), "event");
  for (int i = 0; i < 4; ++i) {
    const uint32_t bn = 32u << i;
    if (!encode_kmajor(&map_h[i], h, T, a.hidden, static_cast<size_t>(a.hidden) * 2, bn) ||
        !encode_kmajor(&map_attn[i], attn, T, m->attn_cols_, static_cast<size_t>(m->attn_cols_) * 2,
                       bn) ||
        !encode_kmajor(&map_act[i], act, T, m->ffn_, static_cast<size_t>(m->ffn_) * 2, bn) ||
        !encode_kmajor(&map_hs[i], hs, sample_cap, a.hidden, static_cast<size_t>(a.hidden) * 2, bn))
      throw std::runtime_error("cuTensorMapEncodeTiled failed (activations)");
  }
  if (!encode_q_heads_map(&map_q, qkv, T, m->hq_, m->hq_ / m->hkv_, m->qkv_rows_))
    throw std::runtime_error("cuTensorMapEncodeTiled failed (prefill attention q)");
}

void LaneWs::release() {
  for (void* p : owned) cudaFree(p);
  owned.clear();
  if (meta_host) cudaFreeHost(meta_host);
  if (out_host) cudaFreeHost(out_host);
  meta_host = nullptr;
  out_host = nullptr;
}

static int bn_index(int bn) { return bn == 32 ? 0 : bn == 64 ? 1 : bn == 128 ? 2 : 3; }

// ---------------------------------------------------------------------------
// Forward.
// ---------------------------------------------------------------------------
void Model::launch(int slot, const nxb::ExecBatch& b) {
  for (auto& p : peers_) p->launch(slot, b);
  DevGuard guard(dev_);
  LaneWs& ws = lanes_[slot];
  const Partitions::Pick pk = parts_.pick(b.lane_kind, b.sm_pct);
  ws.stream = pk.stream;
  ws.sm_count = pk.sm_count;
  ws.layout = pk.layout;
  ws.exclusive = pk.exclusive;
  // ---- pack metadata into the pinned mirror ----
  int T = 0, n_sample = 0, n_pages_total = 0;
  for (const auto& m : b.members) {
    T += m.n_tokens;
    n_sample += m.sample ? 1 : 0;
    n_pages_total += m.n_pages;
  }
  if (T > ws.t_max) throw std::runtime_error("batch exceeds lane token capacity");
  const int n_seq = static_cast<int>(b.members.size());
  uint8_t* hp = ws.meta_host;
  size_t off = 0;
  auto carve = [&](size_t bytes) {
    const size_t o = off;
    off = align_up(off + bytes, 16);
    if (off > ws.meta_bytes) throw std::runtime_error("metadata overflow");
    return o;
  };
  const size_t o_tok = carve(T * 4), o_pos = carve(T * 4), o_slot = carve(T * 4);
  const size_t o_seq = carve(n_seq * sizeof(AttnSeq));
  const size_t o_pages = carve(n_pages_total * 4 + 4);
  const size_t o_rows = carve(n_sample * 4 + 4);
  const size_t o_dpre = carve((n_seq + 1) * 4);
  const int tq = prefill_attn_tokens_per_item(hq_ / hkv_);
  int max_work = 0;
  for (const auto& m : b.members)
    max_work += (m.n_tokens + tq - 1) / tq;
  const size_t o_work = carve(static_cast<size_t>(max_work) * sizeof(int2) + 8);
  int32_t* tok = reinterpret_cast<int32_t*>(hp + o_tok);
  int32_t* pos = reinterpret_cast<int32_t*>(hp + o_pos);
  int32_t* slt = reinterpret_cast<int32_t*>(hp + o_slot);
  AttnSeq* seqs = reinterpret_cast<AttnSeq*>(hp + o_seq);
  int32_t* pages = reinterpret_cast<int32_t*>(hp + o_pages);
  int32_t* rows = reinterpret_cast<int32_t*>(hp + o_rows);
  int2* work = reinterpret_cast<int2*>(hp + o_work);
  int32_t* dpre = reinterpret_cast<int32_t*>(hp + o_dpre);
  int t = 0, pg = 0, ns = 0, nw = 0;
  ws.dec_seq_count = 0;
  ws.max_dec_kv = 0;
  ws.max_dec_tiles = 0;
  ws.dec_kv_tokens = ws.pre_kv_tokens = ws.pre_pairs = 0;
  ws.is_decode_lane = slot == nxb::kLaneDecode;
  // decode members (q_len == 1) first in the seq table so the decode kernel
  // can take a prefix; the batch lists them first already.
  for (int i = 0; i < n_seq; ++i) {
    const auto& m = b.members[i];
    AttnSeq& s = seqs[i];
    s.q_start = t;
    s.q_len = m.n_tokens;
    s.kv_len = static_cast<int>(m.start_pos) + m.n_tokens;
    s.page_off = pg;
    for (int k = 0; k < m.n_pages; ++k) pages[pg + k] = m.pages[k];
    for (int k = 0; k < m.n_tokens; ++k) {
      const int p = static_cast<int>(m.start_pos) + k;
      tok[t + k] = m.tokens[k];
      pos[t + k] = p;
      slt[t + k] = m.pages[p / cfg_.page_tokens] * cfg_.page_tokens + p % cfg_.page_tokens;
    }
    if (m.sample) rows[ns++] = t + m.n_tokens - 1;
    if (!m.is_prefill) {
      if (i != ws.dec_seq_count) throw std::runtime_error("decode members must come first");
      const int tiles = (s.kv_len + kDecTileKeys - 1) / kDecTileKeys;
      if (i == 0) dpre[0] = 0;
      dpre[i + 1] = dpre[i] + tiles;
      ws.max_dec_tiles = std::max(ws.max_dec_tiles, tiles);
      ws.dec_seq_count++;
      ws.max_dec_kv = std::max(ws.max_dec_kv, s.kv_len);
      ws.dec_kv_tokens += s.kv_len;
    } else {
      const double st = static_cast<double>(m.start_pos), q = m.n_tokens;
      ws.pre_kv_tokens += s.kv_len;
      ws.pre_pairs += q * st + q * (q + 1) / 2;
      for (int t0 = 0; t0 < m.n_tokens; t0 += tq) work[nw++] = make_int2(i, t0);
    }
    t += m.n_tokens;
    pg += m.n_pages;
  }
  // prefill attention items longest first (persistent CTAs take them round robin)
  auto item_tiles = [&](const int2& w) {
    const AttnSeq& q = seqs[w.x];
    return q.kv_len - q.q_len + std::min(q.q_len, w.y + tq);
  };
  std::stable_sort(work, work + nw, [&](const int2& a, const int2& c) { return item_tiles(a) > item_tiles(c); });
  ws.tokens = T;
  ws.n_seq = n_seq;
  ws.n_work = nw;
  ws.n_sample = ns;
  cudaStream_t s = ws.stream;
  ws.prof = sample_every_ > 0 && (ws.batch_counter++ % static_cast<uint64_t>(sample_every_)) == 0;
  ws.recs.clear();
  ws.ev_used = 0;
  // Two lanes never share SMs: when this batch or the other lane's batch still
  // in flight runs on the whole GPU (a decode batch while the prefill lane is
  // idle, Engine::dispatch_device), this one is ordered after it.
  if (parts_.enabled && slot < 2) {
    const LaneWs& other = lanes_[1 - slot];
    if (other.pending && (other.layout < 0 || ws.layout < 0))
      ck(cudaStreamWaitEvent(s, other.ev_end, 0), "lane order");
  }
  ck(cudaEventRecord(ws.ev_start, s), "event record");
  ck(cudaMemcpyAsync(ws.meta_dev, hp, off, cudaMemcpyHostToDevice, s), "meta h2d");
  const uint8_t* dp = ws.meta_dev;
  ws.d_tok = reinterpret_cast<const int32_t*>(dp + o_tok);
  ws.d_pos = reinterpret_cast<const int32_t*>(dp + o_pos);
  ws.d_slot = reinterpret_cast<const int32_t*>(dp + o_slot);
  ws.d_seqs = reinterpret_cast<const AttnSeq*>(dp + o_seq);
  ws.d_pages = reinterpret_cast<const int32_t*>(dp + o_pages);
  ws.d_rows = reinterpret_cast<const int32_t*>(dp + o_rows);
  ws.d_work = reinterpret_cast<const int2*>(dp + o_work);
  ws.d_dec_prefix = reinterpret_cast<const int32_t*>(dp + o_dpre);
  ws.dec_total_tiles = ws.dec_seq_count ? static_cast<long long>(dpre[ws.dec_seq_count]) * hkv_ : 0;
  forward(ws);
  ck(cudaMemcpyAsync(ws.out_host, ws.d_out_tokens, static_cast<size_t>(ns) * 4,
                     cudaMemcpyDeviceToHost, s),
     "tokens d2h");
  ck(cudaEventRecord(ws.ev_end, s), "event record");
  ws.pending = true;
}

void Model::forward(LaneWs& ws) {
  cudaStream_t s = ws.stream;
  // Sampled profiling: an event pair around each launch, with its
  // algorithmic bytes / FLOPs, folded into kstats_ when the batch finishes.
  int op = -1;  // reference operator (NX_OP_*) the next launches belong to; -1 = none
  auto timed = [&](int kind, double bytes, double flops, auto&& fn) {
    if (!ws.prof || ws.ev_used + 2 > ws.ev_pool.size()) {
      fn();
      return;
    }
    cudaEvent_t a = ws.ev_pool[ws.ev_used++], b = ws.ev_pool[ws.ev_used++];
    cudaEventRecord(a, s);
    fn();
    cudaEventRecord(b, s);
    ws.recs.push_back({kind, op, a, b, bytes, flops});
  };
  const int T = ws.tokens;
  const double Td = T;
  const int d = a_.hidden;
  const int bn = gemm_pick_bn(T);
  const int bi = bn_index(bn);
  const int sm = ws.sm_count;
  const int gk = ws.is_decode_lane ? NX_K_GEMM_DECODE : NX_K_GEMM_PREFILL;
  // algorithmic GEMM traffic: weights once + activations in + out (+ residual)
  auto gbytes = [&](double rows, double K, double out_b, bool res) {
    return rows * K * 2 + Td * K * 2 + Td * rows * out_b + (res ? Td * rows * 2 : 0);
  };
  auto gflops = [&](double rows, double K) { return 2.0 * Td * rows * K; };
  AttnGeom g;
  g.n_heads = hq_;
  g.n_kv_heads = hkv_;
  g.group = hq_ / hkv_;
  g.head_dim = a_.head_dim;
  g.page_tokens = cfg_.page_tokens;
  g.qkv_stride = qkv_rows_;
  g.out_stride = attn_cols_;
  g.scale_log2 = 1.4426950408889634f / std::sqrt(static_cast<float>(a_.head_dim));
  const double kvtok = 2.0 * hkv_ * a_.head_dim * 2;  // K+V bytes per token per layer
  const double qo = 2.0 * attn_cols_ * 2;                       // q in + out per token
  timed(NX_K_OTHER, Td * d * 2 + Td * 4, 0, [&] { ck(embed(ws.d_tok, T, emb_, d, ws.x, s), "embed"); });
  timed(NX_K_OTHER, Td * a_.head_dim * 4, 0, [&] {
    ck(rope_table(ws.d_pos, T, inv_freq_, a_.head_dim, ws.rope_cs, s), "rope table");
  });
  // Decode-shaped batches defer the GEMMs' cross-CTA K fold to the consumer
  // kernel (GemmFold): residual + RMSNorm, SwiGLU and bias + RoPE + KV write
  // each read the fp32 planes, so no GEMM waits on a fix-up round trip and
  // the separate RMSNorm / RoPE launches disappear.
  const bool fold = fold_enabled_ && tp_ == 1 && T <= 128;
  // prefill-shaped GEMMs on CTA pairs (cta_group::2) when enabled
  const bool pair = !fold && bn == 256 && sm >= 2 && gemm_pair_enabled();
  GemmFold fq, fo, fg, fd;
  // bytes of the planes a fold reads: pieces <= ~max planes; count one plane
  auto pbytes = [&](double rows) { return Td * rows * 4; };
  for (int l = 0; l < a_.n_layers; ++l) {
    const LayerW& w = layers_[l];
    // layer l: [page][kv head][K | V] blocks of 16 x 128 (one contiguous 8 KB
    // block per (page, kv head), kv_chunk_elem atoms); the V view starts one K
    // half-block on
    __nv_bfloat16* kplane = kv_ + (2 * static_cast<size_t>(l)) * plane_elems_;
    __nv_bfloat16* vplane = kplane + static_cast<size_t>(cfg_.page_tokens) * a_.head_dim;
    RopeKV rope;
    rope.slot = ws.d_slot;
    rope.table = ws.rope_cs;
    rope.kplane = kplane;
    rope.vplane = vplane;
    rope.n_heads = hq_;
    rope.n_kv_heads = hkv_;
    rope.page_tokens = cfg_.page_tokens;
    op = NX_OP_QKV_PROJ;
    if (!fold || l == 0)
      timed(NX_K_OTHER, Td * d * 4, 0, [&] {
        ck(rmsnorm(ws.x, nullptr, T, d, w.attn_norm, a_.rms_eps, ws.h, s), "rmsnorm");
      });
    timed(gk, gbytes(qkv_rows_, d, fold ? 4 : 2, false), gflops(qkv_rows_, d), [&] {
      ck(fold ? gemm_decode(w.qkv, ws.map_h[bi], bn, qkv_rows_, T, d, nullptr, 0, ws.ws, ws.ws_bytes, sm, s, &fq)
              : pair ? gemm_pair(w.qkv, ws.map_h[2], qkv_rows_, T, d, kEpiRopeKV, ws.qkv, qkv_rows_, w.qkv_bias,
                                 nullptr, 0, sm, s, &rope)
              : gemm(w.qkv, ws.map_h[bi], bn, qkv_rows_, T, d, w.qkv_bias ? kEpiBias : kEpiStore,
                     ws.qkv, qkv_rows_, w.qkv_bias, nullptr, 0, ws.ws, ws.ws_bytes, sm, s, 0, ws.exclusive),
         "qkv gemm");
    });
    if (pair) {
      // RoPE + paged KV write ran in the QKV epilogue
    } else if (fold)
      timed(NX_K_OTHER, pbytes(qkv_rows_) + Td * qkv_rows_ * 2, 0, [&] {
        ck(fold_rope_kv(fq, w.qkv_bias, ws.qkv, ws.d_slot, ws.rope_cs, hq_, hkv_, cfg_.page_tokens, kplane,
                        vplane, s),
           "fold rope");
      });
    else
      timed(NX_K_OTHER, Td * qkv_rows_ * 4, 0, [&] {
        ck(rope_kv_write(ws.qkv, T, ws.d_slot, ws.rope_cs, hq_, hkv_, a_.head_dim,
                         cfg_.page_tokens, kplane, vplane, s),
           "rope");
      });
    op = NX_OP_ATTN_DECODE;
    if (ws.dec_seq_count > 0)
      timed(NX_K_ATTN_DECODE, ws.dec_kv_tokens * kvtok + ws.dec_seq_count * qo,
            4.0 * ws.dec_kv_tokens * attn_cols_, [&] {
              ck(decode_attention(g, ws.qkv, kplane, vplane, ws.d_seqs, ws.dec_seq_count,
                                  ws.d_dec_prefix, ws.dec_total_tiles, ws.max_dec_tiles, ws.d_pages,
                                  ws.attn, ws.part_o, ws.part_ml, ws.part_cap, ws.item_done, sm, s),
                 "decode attention");
            });
    op = NX_OP_ATTN_PREFILL;
    if (ws.n_work > 0)
      timed(NX_K_ATTN_PREFILL, ws.pre_kv_tokens * kvtok + (Td - ws.dec_seq_count) * qo,
            4.0 * ws.pre_pairs * attn_cols_, [&] {
              ck(prefill_attention(g, ws.map_q, kplane, ws.d_seqs, ws.d_work, ws.n_work, ws.d_pages,
                                   ws.attn, sm, s),
                 "prefill attention");
            });
    // Row-parallel under TP: rank 0 adds the residual, the others store
    // their partial; the all-reduce then yields x + sum_r o_r on every rank.
    const int res_mode = (tp_ == 1 || rank_ == 0) ? kEpiResidual : kEpiStore;
    op = NX_OP_ATTN_OUT_PROJ;
    timed(gk, gbytes(d, attn_cols_, fold ? 4 : 2, !fold), gflops(d, attn_cols_), [&] {
      ck(fold ? gemm_decode(w.o, ws.map_attn[bi], bn, d, T, attn_cols_, nullptr, 0, ws.ws, ws.ws_bytes, sm, s, &fo)
              : pair ? gemm_pair(w.o, ws.map_attn[2], d, T, attn_cols_, res_mode, ws.x, d, nullptr, ws.x, d, sm, s)
              : gemm(w.o, ws.map_attn[bi], bn, d, T, attn_cols_, res_mode, ws.x, d, nullptr, ws.x,
                     d, ws.ws, ws.ws_bytes, sm, s, 0, ws.exclusive),
         "o gemm");
    });
    if (tp_ > 1) timed(NX_K_OTHER, Td * d * 2 * 2, 0, [&] { all_reduce(ws, ws.x, static_cast<size_t>(T) * d); });
    if (fold)
      timed(NX_K_OTHER, pbytes(d) + Td * d * 6, 0, [&] {
        ck(fold_residual_rmsnorm(fo, ws.x, w.ffn_norm, a_.rms_eps, ws.h, s), "fold o");
      });
    else
      timed(NX_K_OTHER, Td * d * 4, 0, [&] {
        ck(rmsnorm(ws.x, nullptr, T, d, w.ffn_norm, a_.rms_eps, ws.h, s), "rmsnorm");
      });
    op = NX_OP_FFN;
    timed(gk, gbytes(2.0 * ffn_, d, fold ? 8 : 1, false), gflops(2.0 * ffn_, d), [&] {
      ck(fold ? gemm_decode(w.gate_up, ws.map_h[bi], bn, 2 * ffn_, T, d, nullptr, 0, ws.ws, ws.ws_bytes, sm, s, &fg)
              : pair ? gemm_pair(w.gate_up, ws.map_h[2], 2 * ffn_, T, d, kEpiSwiGLU, ws.act, ffn_, nullptr, nullptr, 0,
                                 sm, s)
              : gemm(w.gate_up, ws.map_h[bi], bn, 2 * ffn_, T, d, kEpiSwiGLU, ws.act, ffn_, nullptr,
                     nullptr, 0, ws.ws, ws.ws_bytes, sm, s, 0, ws.exclusive),
         "gate/up gemm");
    });
    if (fold)
      timed(NX_K_OTHER, pbytes(2.0 * ffn_) + Td * ffn_ * 2, 0, [&] {
        ck(fold_swiglu(fg, ws.act, s), "fold swiglu");
      });
    timed(gk, gbytes(d, ffn_, fold ? 4 : 2, !fold), gflops(d, ffn_), [&] {
      ck(fold ? gemm_decode(w.down, ws.map_act[bi], bn, d, T, ffn_, nullptr, 0, ws.ws, ws.ws_bytes, sm, s, &fd)
              : pair ? gemm_pair(w.down, ws.map_act[2], d, T, ffn_, res_mode, ws.x, d, nullptr, ws.x, d, sm, s)
              : gemm(w.down, ws.map_act[bi], bn, d, T, ffn_, res_mode, ws.x, d, nullptr, ws.x, d,
                     ws.ws, ws.ws_bytes, sm, s, 0, ws.exclusive),
         "down gemm");
    });
    if (tp_ > 1) timed(NX_K_OTHER, Td * d * 2 * 2, 0, [&] { all_reduce(ws, ws.x, static_cast<size_t>(T) * d); });
    if (fold) {
      // the next layer's attention RMSNorm rides along (none after the last)
      const __nv_bfloat16* next_norm = l + 1 < a_.n_layers ? layers_[l + 1].attn_norm : nullptr;
      timed(NX_K_OTHER, pbytes(d) + Td * d * 6, 0, [&] {
        ck(fold_residual_rmsnorm(fd, ws.x, next_norm, a_.rms_eps, ws.h, s), "fold down");
      });
    }
  }
  op = -1;
  // lm_head over the sampled rows, in chunks of the logits buffer.
  ws.d_out_tokens = ws.logits_tokens_dev();
  for (int r0 = 0; r0 < ws.n_sample; r0 += ws.sample_cap) {
    const int n = std::min(ws.sample_cap, ws.n_sample - r0);
    const double nd = n;
    timed(NX_K_OTHER, nd * d * 4, 0, [&] {
      ck(rmsnorm(ws.x, ws.d_rows + r0, n, d, final_norm_, a_.rms_eps, ws.hs, s), "final norm");
    });
    const int sbn = gemm_pick_bn(n);
    timed(gk, static_cast<double>(vocab_l_) * d * 2 + nd * d * 2 + nd * vocab_l_ * 4,
          2.0 * nd * vocab_l_ * d, [&] {
            ck(tp_ == 1 && n <= 128
                   ? gemm_decode(lm_head_, ws.map_hs[bn_index(sbn)], sbn, vocab_l_, n, d, ws.logits, vocab_l_,
                                 ws.ws, ws.ws_bytes, sm, s, nullptr)
                   : gemm(lm_head_, ws.map_hs[bn_index(sbn)], sbn, vocab_l_, n, d, kEpiF32, ws.logits,
                          vocab_l_, nullptr, nullptr, 0, ws.ws, ws.ws_bytes, sm, s, 0, ws.exclusive),
               "lm_head gemm");
          });
    timed(NX_K_OTHER, nd * vocab_l_ * 4, 0, [&] {
      if (tp_ == 1) {
        ck(argmax_rows(ws.logits, n, vocab_l_, vocab_l_, 0, ws.d_out_tokens + r0, nullptr,
                       reinterpret_cast<float2*>(ws.part_ml), s),
           "argmax");
        return;
      }
      // vocab-parallel: local (max, global idx) pairs -> all-gather -> fold
      float2* mine = ws.tp_pairs + static_cast<size_t>(n) * tp_;
      ck(argmax_rows(ws.logits, n, vocab_l_, vocab_valid_, vocab0_, nullptr, mine,
                     reinterpret_cast<float2*>(ws.part_ml), s),
         "argmax");
      if (group_) {
        group_->argmax_gather(rank_, ws.slot_index, mine, n, ws.d_out_tokens + r0, s);
        return;
      }
      Nccl::get().all_gather_f2(comm_[ws.slot_index], mine, ws.tp_pairs, 2 * static_cast<size_t>(n), s);
      ck(argmax_fold(ws.tp_pairs, tp_, n, ws.d_out_tokens + r0, s), "argmax fold");
    });
  }
}

int32_t* LaneWs::logits_tokens_dev() {
  if (!out_dev) {
    ck(cudaMalloc(&out_dev, static_cast<size_t>(t_max) * 4), "out tokens");
    owned.push_back(out_dev);
  }
  return static_cast<int32_t*>(out_dev);
}

bool Model::done(int slot) {
  for (auto& p : peers_)
    if (!p->done(slot)) return false;
  DevGuard guard(dev_);
  LaneWs& ws = lanes_[slot];
  if (!ws.pending) return true;
  const cudaError_t e = cudaEventQuery(ws.ev_end);
  if (e == cudaErrorNotReady) return false;
  ck(e, "device batch");
  finish(ws);
  return true;
}

void Model::wait(int slot) {
  for (auto& p : peers_) p->wait(slot);
  DevGuard guard(dev_);
  LaneWs& ws = lanes_[slot];
  if (!ws.pending) return;
  ck(cudaEventSynchronize(ws.ev_end), "device batch");
  finish(ws);
}

void Model::finish(LaneWs& ws) {
  ws.pending = false;
  if (group_ && group_->error())
    throw std::runtime_error("TP peer collective timed out (a rank never arrived)");
  kstats_.batches += 1;
  ws.sampled.assign(ws.out_host, ws.out_host + ws.n_sample);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ws.ev_start, ws.ev_end);
  ws.last_ms = ms;
  if (ws.prof) {
    for (const auto& r : ws.recs) {
      float t = 0.f;
      cudaEventElapsedTime(&t, r.a, r.b);
      kstats_.ms[r.kind] += t;
      kstats_.sm_ms[r.kind] += t * ws.sm_count;
      kstats_.bytes[r.kind] += r.bytes;
      kstats_.flops[r.kind] += r.flops;
      kstats_.launches[r.kind] += 1;
      if (r.op >= 0) {
        kstats_.op_ms[r.op] += t;
        kstats_.op_launches[r.op] += 1;
      }
    }
    kstats_.batches_sampled += 1;
    kstats_.batch_ms_sampled += ms;
    ws.recs.clear();
    ws.prof = false;
  }
}

void Model::copy_logits(int slot, float* host, size_t n_floats) {
  DevGuard guard(dev_);
  LaneWs& ws = lanes_[slot];
  const size_t rows = static_cast<size_t>(std::min(ws.n_sample, ws.sample_cap));
  if (!group_) {
    const size_t want = std::min<size_t>(n_floats, rows * vocab_l_);
    ck(cudaMemcpy(host, ws.logits, want * 4, cudaMemcpyDeviceToHost), "logits d2h");
    return;
  }
  // one-process TP group: stitch every rank's vocab slice into [rows][vocab]
  std::vector<float> part(rows * vocab_l_);
  for (int r = 0; r < tp_; ++r) {
    Model* m = r == 0 ? this : peers_[r - 1].get();
    DevGuard g(m->dev_);
    ck(cudaMemcpy(part.data(), m->lanes_[slot].logits, part.size() * 4, cudaMemcpyDeviceToHost),
       "logits d2h");
    for (size_t i = 0; i < rows; ++i)
      for (int j = 0; j < m->vocab_valid_; ++j) {
        const size_t dst = i * a_.vocab + m->vocab0_ + j;
        if (dst < n_floats) host[dst] = part[i * vocab_l_ + j];
      }
  }
}

size_t Model::weight_to_host(int tensor, int layer, void* host, size_t cap) const {
  DevGuard guard(dev_);
  const size_t d = a_.hidden;
  if (tensor != 0 && tensor != 8 && tensor != 9 && (layer < 0 || layer >= a_.n_layers))
    throw std::invalid_argument("unknown layer");
  const __nv_bfloat16* p = nullptr;
  size_t elems = 0;
  int rows = 0, K = 0;  // > 0: packed matrix
  switch (tensor) {
    case 0: p = emb_; elems = static_cast<size_t>(a_.vocab) * d; break;
    case 1: p = layers_[layer].attn_norm; elems = d; break;
    case 2: p = layers_[layer].qkv; rows = qkv_rows_; K = static_cast<int>(d); break;
    case 3: p = layers_[layer].qkv_bias; elems = a_.qkv_bias ? qkv_rows_ : 0; break;
    case 4: p = layers_[layer].o; rows = static_cast<int>(d); K = attn_cols_; break;
    case 5: p = layers_[layer].ffn_norm; elems = d; break;
    case 6: p = layers_[layer].gate_up; rows = 2 * ffn_; K = static_cast<int>(d); break;
    case 7: p = layers_[layer].down; rows = static_cast<int>(d); K = ffn_; break;
    case 8: p = final_norm_; elems = d; break;
    case 9: p = lm_head_; rows = vocab_l_; K = static_cast<int>(d); break;
    default: throw std::invalid_argument("unknown tensor");
  }
  if (rows) elems = static_cast<size_t>(rows) * K;
  if (!host) return elems * 2;
  if (cap < elems * 2) throw std::invalid_argument("buffer too small");
  if (!elems) return 0;
  if (!rows) {
    ck(cudaMemcpy(host, p, elems * 2, cudaMemcpyDeviceToHost), "weight d2h");
    return elems * 2;
  }
  __nv_bfloat16* tmp = nullptr;
  ck(cudaMalloc(&tmp, elems * 2), "unpack staging");
  ck(unpack_weights(p, tmp, rows, K, nullptr), "unpack");
  const cudaError_t e = cudaMemcpy(host, tmp, elems * 2, cudaMemcpyDeviceToHost);
  cudaFree(tmp);
  ck(e, "weight d2h");
  return elems * 2;
}

}  // namespace nxd
