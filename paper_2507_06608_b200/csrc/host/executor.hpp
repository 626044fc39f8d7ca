// The seam between the host step executor and the device.
//
// In the reference a batch's latency is *predicted* (simulator.cpp:361-366,
// 391-393). Here the engine hands each launched batch to an Executor, which
// runs the real prefill/decode kernels on the lane's green-context SM
// partition and reports completion; the engine's clock mode decides whether
// the measured time or the cost model drives the event loop.
#pragma once

#include <cstdint>
#include <vector>

namespace nxb {

enum LaneSlot { kLanePrefill = 0, kLaneDecode = 1 };

struct ExecMember {
  uint64_t id = 0;
  int32_t n_tokens = 0;       // chunk tokens (prefill) or 1 (decode)
  int64_t start_pos = 0;      // KV position of the first input token
  int32_t sample = 0;         // 1: emit the next token after this launch
  int32_t is_prefill = 0;
  const int32_t* tokens = nullptr;  // n_tokens input ids (host memory)
  const int32_t* pages = nullptr;   // page table covering start_pos + n_tokens
  int32_t n_pages = 0;
};

struct ExecBatch {
  int lane_kind = 0;   // NX_LANE_PREFILL / NX_LANE_DECODE / NX_LANE_MIXED
  int sm_pct = 100;    // this lane's share of the GPU, integer percent
  std::vector<ExecMember> members;  // decode members first, then prefill (log order)
};

class Executor {
 public:
  virtual ~Executor() = default;
  // Enqueue the batch on the lane's stream; must not block on the device.
  virtual void launch(int slot, const ExecBatch& b) = 0;
  // Non-blocking completion probe.
  virtual bool done(int slot) = 0;
  // Block until the lane's batch finished.
  virtual void wait(int slot) = 0;
  // After completion: sampled tokens of the sampling members, in member order.
  virtual const std::vector<int32_t>& sampled(int slot) = 0;
  // Device-timed duration (ms) of the lane's last batch (CUDA events).
  virtual double device_ms(int slot) = 0;
  virtual int32_t vocab() const = 0;
  // Page geometry the executor's KV cache was built with.
  virtual int32_t page_tokens() const = 0;
  virtual int32_t num_pages() const = 0;
};

}  // namespace nxb
