// Device executor declarations (see model.cu).
#pragma once

#include <cstdlib>

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <stdexcept>
#include <vector>

#include "device.cuh"
#include "executor.hpp"
#include "tp.cuh"
#include <memory>
#include "nexus_b200.h"

namespace nxd {

struct NoDevice : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Pre-instantiated green-context SM layouts: layout k gives the decode lane
// a group of 8(k+1) SMs and the prefill lane the rest of the same split.
struct Partitions {
  struct Layout {
    int decode_sms = 0, prefill_sms = 0;
    cudaStream_t decode_stream = nullptr, prefill_stream = nullptr;
  };
  struct Pick {
    cudaStream_t stream = nullptr;
    int sm_count = 0;
    int layout = -1;
    bool exclusive = false;  // the stream owns its SMs (green partition / whole GPU)
  };
  void init(int device, bool enable);
  Pick pick(int lane_kind, int sm_pct) const;
  bool enabled = false;
  int total_sm = 0;
  std::vector<Layout> layouts;
  cudaStream_t full_stream = nullptr;          // monolithic lane: whole GPU
  cudaStream_t plain_stream[2] = {nullptr, nullptr};  // no partitioning
};

class Model;

struct LaneWs {
  void init(Model* m, int max_tokens);
  void release();
  int32_t* logits_tokens_dev();

  int t_max = 0;
  __nv_bfloat16 *x = nullptr, *h = nullptr, *qkv = nullptr, *attn = nullptr, *act = nullptr,
                *hs = nullptr;
  float* logits = nullptr;
  float2* rope_cs = nullptr;  // per-batch RoPE table [t_max][64]
  float2* tp_pairs = nullptr;  // TP: (max, argmax) per sampled row, gathered [tp][rows]
  int slot_index = 0;
  int sample_cap = 0;
  float* ws = nullptr;
  size_t ws_bytes = 0;
  float *part_o = nullptr, *part_ml = nullptr;
  int* item_done = nullptr;  // decode attention: partials written per (sequence, kv head), zero between launches
  size_t part_cap = 0;
  CUtensorMap map_h[4], map_attn[4], map_act[4], map_hs[4];
  CUtensorMap map_q;  // q heads of the qkv buffer for prefill attention (encode_q_heads_map)
  uint8_t* meta_dev = nullptr;
  uint8_t* meta_host = nullptr;
  size_t meta_bytes = 0;
  int32_t* out_host = nullptr;
  void* out_dev = nullptr;
  cudaEvent_t ev_start = nullptr, ev_end = nullptr;
  std::vector<void*> owned;
  // current batch
  cudaStream_t stream = nullptr;
  int sm_count = 0, layout = -1;
  bool exclusive = false;
  int tokens = 0, n_seq = 0, n_work = 0, n_sample = 0, dec_seq_count = 0, max_dec_kv = 0;
  int max_dec_tiles = 0;
  long long dec_total_tiles = 0;
  const int32_t* d_dec_prefix = nullptr;
  const int32_t *d_tok = nullptr, *d_pos = nullptr, *d_slot = nullptr, *d_pages = nullptr,
                *d_rows = nullptr;
  const AttnSeq* d_seqs = nullptr;
  const int2* d_work = nullptr;
  int32_t* d_out_tokens = nullptr;
  bool pending = false;
  std::vector<int32_t> sampled;
  float last_ms = 0.f;
  // sampled per-kernel-class profiling
  struct ProfRec {
    int kind, op;
    cudaEvent_t a, b;
    double bytes, flops;
  };
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<ProfRec> recs;
  bool prof = false;
  uint64_t batch_counter = 0;
  double dec_kv_tokens = 0, pre_kv_tokens = 0, pre_pairs = 0;
  bool is_decode_lane = false;
};

// Projection weights are held in the packed tile layout (pack_weights).
struct LayerW {
  __nv_bfloat16 *attn_norm, *qkv, *qkv_bias, *o, *ffn_norm, *gate_up, *down;
};

class Model : public nxb::Executor {
 public:
  // group: the peer-memory TP group this rank belongs to (NX_TP_PEER*); rank 0
  // creates it and the other ranks' Models, and fans every batch out to them.
  explicit Model(const nx_device_config& cfg, std::shared_ptr<PeerGroup> group = nullptr);
  ~Model() override;

  void launch(int slot, const nxb::ExecBatch& b) override;
  bool done(int slot) override;
  void wait(int slot) override;
  const std::vector<int32_t>& sampled(int slot) override { return lanes_[slot].sampled; }
  double device_ms(int slot) override { return lanes_[slot].last_ms; }
  int32_t vocab() const override { return a_.vocab; }
  int32_t page_tokens() const override { return cfg_.page_tokens; }
  int32_t num_pages() const override { return cfg_.num_pages; }

  void copy_logits(int slot, float* host, size_t n_floats);
  // Logical (row-major) copy of a weight tensor into host memory.
  size_t weight_to_host(int tensor, int layer, void* host, size_t cap) const;
  const Partitions& partitions() const { return parts_; }
  uint64_t weight_bytes() const { return weight_bytes_; }
  uint64_t kv_bytes() const { return kv_bytes_; }
  int last_layout(int slot) const { return lanes_[slot].layout; }
  int last_sm_count(int slot) const { return lanes_[slot].sm_count; }
  void set_profiling(int every) { sample_every_ = every; }
  nx_kernel_stats kernel_stats() const {
    nx_kernel_stats k = kstats_;
    k.kernel_launches = g_kernel_launches;
    return k;
  }
  void reset_kernel_stats() { kstats_ = nx_kernel_stats{}; }

 private:
  friend struct LaneWs;
  void alloc_weights();
  void alloc_kv();
  void forward(LaneWs& ws);
  void finish(LaneWs& ws);
  __nv_bfloat16* dalloc_bf16(size_t n);

  nx_device_config cfg_;
  nx_arch a_;
  int qkv_rows_ = 0, attn_cols_ = 0;
  // tensor-parallel shard (tp_ = 1: whole model on this GPU)
  int tp_ = 1, rank_ = 0;
  int hq_ = 0, hkv_ = 0, ffn_ = 0;        // local q heads, kv heads, ffn features
  int vocab_l_ = 0, vocab_valid_ = 0, vocab0_ = 0;  // local lm_head rows (padded), valid, offset
  void* comm_[2] = {nullptr, nullptr};    // NCCL communicator per lane
  std::shared_ptr<PeerGroup> group_;      // peer-memory TP group (one process)
  std::vector<std::unique_ptr<Model>> peers_;  // ranks 1..tp-1 (rank 0 only)
  int dev_ = 0;
  void all_reduce(LaneWs& ws, __nv_bfloat16* x, size_t n);
  Partitions parts_;
  std::vector<void*> allocs_;
  __nv_bfloat16 *emb_ = nullptr, *final_norm_ = nullptr, *lm_head_ = nullptr, *kv_ = nullptr;
  std::vector<LayerW> layers_;
  float* inv_freq_ = nullptr;
  size_t plane_elems_ = 0;
  uint64_t weight_bytes_ = 0, kv_bytes_ = 0;
  LaneWs lanes_[2];
  int sample_every_ = 0;
  // deferred-fold decode GEMMs (GemmFold); NX_FOLD=0 restores the in-GEMM fix-up
  bool fold_enabled_ = [] {
    const char* e = std::getenv("NX_FOLD");
    return !(e && e[0] == '0');
  }();
  nx_kernel_stats kstats_{};
};

}  // namespace nxd
