// Tensor parallelism: Megatron-style sharding of the decoder
// across tp ranks of one node, NCCL over NVLink / NVSwitch.
//
//   QKV      column-parallel by heads: rank r owns q heads [r*H/tp, ...) and
//            kv heads [r*Hkv/tp, ...); the KV cache holds only those heads.
//   O        row-parallel -> all-reduce (sum) of the [T, d] output
//   gate/up  column-parallel (ffn/tp features, SwiGLU stays local)
//   down     row-parallel -> all-reduce
//   lm_head  vocab-parallel (vocab padded to a multiple of 128 * tp); each
//            rank's (max, argmax) pairs are all-gathered and folded with the
//            lowest-global-index tie rule.
// The residual add folds into the all-reduce: rank 0's projection epilogue
// adds the residual (x + o_0), the others store o_r, and sum(x) = x + sum o_r.
// One NCCL communicator per lane (prefill, decode) so the lanes never
// serialize on a shared NCCL stream; NCCL kernels run inside the issuing
// lane's green-context SMs.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "nexus_b200.h"

namespace nxd {

// Shard geometry of one rank (pure host arithmetic; also exported through
// nx_tp_shard_plan for the CPU tests).
nx_tp_shard tp_plan(const nx_arch& a, int tp_size, int rank);

// Thin dlopen() binding of libnccl.so.2 (no link-time dependency, so the
// library still loads on GPU-less hosts).
class Nccl {
 public:
  static Nccl& get();  // throws std::runtime_error if NCCL is unavailable
  void unique_id(uint8_t out[128]);
  void* comm_init(int nranks, const uint8_t id[128], int rank);
  void all_reduce_bf16(void* comm, void* buf, size_t count, cudaStream_t s);
  void all_gather_f2(void* comm, const void* send, void* recv, size_t count_floats, cudaStream_t s);
  void broadcast_bytes(void* comm, void* buf, size_t bytes, int root, cudaStream_t s);
  void destroy(void* comm);

 private:
  Nccl();
  void check(int rc, const char* what);
  void* lib_ = nullptr;
  void* sym_[8] = {};
};

// Peer-memory collectives for a TP group driven by ONE process (NX_TP_PEER:
// rank r on GPU device+r with peer access over NVLink; NX_TP_PEER_COLOCATED:
// all ranks on one GPU, for tests). Every collective is a single kernel per
// rank: publish the local partial into its own double-buffered slot, push an
// epoch flag per chunk into every rank's flag row, wait for all ranks' flags
// of the same chunk, then reduce the chunk in fixed rank order (so all ranks
// hold bitwise-identical results). No NCCL, no host round trip.
constexpr int kPeerMaxRanks = 8;
constexpr int kPeerMaxChunks = 1024;

class PeerGroup {
 public:
  // colocated: every rank on one GPU (tests) — collectives then use a few
  // CTAs so spinning ranks never starve the ranks they wait for of SMs.
  PeerGroup(int tp, bool colocated);
  ~PeerGroup();
  // Rank `rank` registers its per-lane exchange buffers (on its own device).
  void register_lane(int rank, int lane, size_t max_elems);
  void release_rank(int rank);
  // x[0:n) <- sum over ranks of x_r[0:n) (bf16 in, fp32 sum, bf16 out), with
  // at most max_ctas CTAs (the lane's SM count).
  void all_reduce_bf16(int rank, int lane, __nv_bfloat16* x, size_t n, int max_ctas, cudaStream_t s);
  // tokens[i] <- global argmax from each rank's (max, global idx) pair i.
  void argmax_gather(int rank, int lane, const float2* mine, int n, int32_t* out, cudaStream_t s);
  // Non-zero once a peer wait timed out (a rank never arrived).
  int error() const { return *err_host_; }
  int size() const { return tp_; }

 private:
  struct Slot {
    void* buf[2] = {nullptr, nullptr};  // epoch parity
    uint32_t* flags = nullptr;          // [kPeerMaxRanks][kPeerMaxChunks]
    uint32_t epoch = 0;
  };
  int tp_;
  bool colocated_;
  Slot slot_[kPeerMaxRanks][2];
  int* err_host_ = nullptr;
  int* err_dev_ = nullptr;
};

}  // namespace nxd
