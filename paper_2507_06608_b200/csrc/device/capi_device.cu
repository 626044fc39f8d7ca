// Device half of the C-ABI (include/nexus_b200.h, "device executor" section).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>
#include <memory>
#include <string>

#include "capi_internal.hpp"
#include "device.cuh"
#include "model.cuh"
#include "tp.cuh"

struct nx_device {
  std::unique_ptr<nxd::Model> m;
};

namespace {

int dfail(int code, const std::string& what) {
  nxb::last_error() = what;
  return code;
}

template <class F>
int dguard(F&& f) {
  try {
    nxb::last_error().clear();
    return f();
  } catch (const nxd::NoDevice& e) {
    return dfail(NX_ENODEV, e.what());
  } catch (const std::invalid_argument& e) {
    return dfail(NX_EINVAL, e.what());
  } catch (const std::bad_alloc&) {
    return dfail(NX_ENOMEM, "out of memory");
  } catch (const std::exception& e) {
    return dfail(NX_ERUNTIME, e.what());
  }
}

int cuda_rc(cudaError_t e) {
  if (e == cudaSuccess) return NX_OK;
  return dfail(e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver ? NX_ENODEV : NX_ERUNTIME,
               cudaGetErrorString(e));
}

}  // namespace

extern "C" {

int nx_device_create(const nx_device_config* cfg, nx_device** out) {
  return dguard([&] {
    auto d = std::make_unique<nx_device>();
    d->m = std::make_unique<nxd::Model>(*cfg);
    *out = d.release();
    return NX_OK;
  });
}

void nx_device_destroy(nx_device* dev) { delete dev; }

int nx_tp_shard_plan(const nx_arch* arch, int32_t tp_size, int32_t rank, nx_tp_shard* out) {
  return dguard([&] {
    if (!arch || !out) throw std::invalid_argument("nx_tp_shard_plan: null argument");
    *out = nxd::tp_plan(*arch, tp_size, rank);
    return NX_OK;
  });
}

int nx_nccl_unique_id(uint8_t out[128]) {
  return dguard([&] {
    nxd::Nccl::get().unique_id(out);
    return NX_OK;
  });
}

int nx_device_get_info(const nx_device* dev, nx_device_info* out) {
  std::memset(out, 0, sizeof(*out));
  const nxd::Partitions& p = dev->m->partitions();
  out->sm_count = p.total_sm;
  out->n_layouts = static_cast<int32_t>(p.layouts.size());
  for (size_t i = 0; i < p.layouts.size() && i < 32; ++i) {
    out->layout_decode_sms[i] = p.layouts[i].decode_sms;
    out->layout_prefill_sms[i] = p.layouts[i].prefill_sms;
  }
  out->weight_bytes = dev->m->weight_bytes();
  out->kv_bytes = dev->m->kv_bytes();
  return NX_OK;
}

int nx_engine_bind_device(nx_engine* eng, nx_device* dev) {
  return dguard([&] {
    eng->e.bind(dev->m.get(), /*owns=*/false);
    return NX_OK;
  });
}

int nx_device_weight(const nx_device* dev, int32_t tensor, int32_t layer, void* host,
                     size_t cap_bytes, size_t* bytes) {
  return dguard([&] {
    *bytes = dev->m->weight_to_host(tensor, layer, nullptr, 0);
    if (host) dev->m->weight_to_host(tensor, layer, host, cap_bytes);
    return NX_OK;
  });
}

int nx_device_launch(nx_device* dev, const nx_batch_desc* b) {
  return dguard([&] {
    nxb::ExecBatch eb;
    eb.lane_kind = b->lane == 1 ? NX_LANE_DECODE : NX_LANE_PREFILL;
    eb.sm_pct = b->sm_pct;
    size_t tok_off = 0, page_off = 0;
    bool any_prefill = false, any_decode = false;
    for (int i = 0; i < b->n_members; ++i) {
      nxb::ExecMember m;
      m.id = static_cast<uint64_t>(i);
      m.n_tokens = b->n_tokens[i];
      m.start_pos = b->start_pos[i];
      m.sample = b->sample[i];
      // Leading single-token members run through the decode kernel (same math).
      m.is_prefill = (b->lane == 1 || (m.n_tokens == 1 && !any_prefill)) ? 0 : 1;
      m.tokens = b->tokens + tok_off;
      m.pages = b->pages + page_off;
      m.n_pages = b->n_pages[i];
      tok_off += m.n_tokens;
      page_off += m.n_pages;
      any_prefill |= m.is_prefill != 0;
      any_decode |= m.is_prefill == 0;
      eb.members.push_back(m);
    }
    if (b->lane == 0 && any_decode && any_prefill) eb.lane_kind = NX_LANE_MIXED;
    dev->m->launch(b->lane == 1 ? nxb::kLaneDecode : nxb::kLanePrefill, eb);
    return NX_OK;
  });
}

int nx_device_wait(nx_device* dev, int32_t lane, int32_t* sampled, float* logits,
                   double* device_ms) {
  return dguard([&] {
    const int slot = lane == 1 ? nxb::kLaneDecode : nxb::kLanePrefill;
    dev->m->wait(slot);
    const std::vector<int32_t>& s = dev->m->sampled(slot);
    if (sampled) std::memcpy(sampled, s.data(), s.size() * 4);
    if (logits) dev->m->copy_logits(slot, logits, s.size() * static_cast<size_t>(dev->m->vocab()));
    if (device_ms) *device_ms = dev->m->device_ms(slot);
    return NX_OK;
  });
}

int nx_device_forward(nx_device* dev, const nx_batch_desc* b, int32_t* sampled, float* logits,
                      double* device_ms) {
  const int rc = nx_device_launch(dev, b);
  if (rc != NX_OK) return rc;
  return nx_device_wait(dev, b->lane, sampled, logits, device_ms);
}

int nx_device_set_profiling(nx_device* dev, int32_t sample_every) {
  dev->m->set_profiling(sample_every);
  return NX_OK;
}

int nx_device_kernel_stats(const nx_device* dev, nx_kernel_stats* out) {
  *out = dev->m->kernel_stats();
  return NX_OK;
}

int nx_device_reset_kernel_stats(nx_device* dev) {
  dev->m->reset_kernel_stats();
  return NX_OK;
}

int nx_dev_malloc(size_t bytes, void** p) { return cuda_rc(cudaMalloc(p, bytes)); }
int nx_dev_free(void* p) { return cuda_rc(cudaFree(p)); }
int nx_dev_h2d(void* dst, const void* src, size_t n) {
  return cuda_rc(cudaMemcpy(dst, src, n, cudaMemcpyHostToDevice));
}
int nx_dev_d2h(void* dst, const void* src, size_t n) {
  return cuda_rc(cudaMemcpy(dst, src, n, cudaMemcpyDeviceToHost));
}
int nx_dev_sync(void) { return cuda_rc(cudaDeviceSynchronize()); }

size_t nx_dbg_gemm_trace(uint64_t* out, size_t n) {
  return nxd::gemm_trace_read(reinterpret_cast<unsigned long long*>(out), n);
}

// Decode GEMM (tokens <= 128): mode 16 = stream-K fold planes + fold_store_f32,
// mode 17 = direct fp32 (data-parallel). out is fp32 [tokens][rows].
static int op_gemm_decode(const void* x, const void* w, int32_t tokens, int32_t rows, int32_t K, int32_t mode,
                          void* out, int32_t sm_count, int32_t iters, float* ms) {
  const int bn = nxd::gemm_pick_bn(tokens);
  CUtensorMap xm;
  if (!nxd::encode_kmajor(&xm, x, tokens, K, static_cast<uint64_t>(K) * 2, bn))
    return dfail(NX_ERUNTIME, "tensor map encode failed");
  __nv_bfloat16* wp = nullptr;
  int rc = cuda_rc(cudaMalloc(&wp, nxd::packed_weight_elems(rows, K) * 2));
  if (rc) return rc;
  rc = cuda_rc(nxd::pack_weights(static_cast<const __nv_bfloat16*>(w), wp, rows, K, nullptr));
  int dev = 0, n_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  if (sm_count <= 0 || sm_count > n_sm) sm_count = n_sm;
  float* ws = nullptr;
  const size_t ws_bytes = 256u << 20;
  if (!rc) rc = cuda_rc(cudaMalloc(&ws, ws_bytes));
  const int n = iters > 0 ? iters : 1;
  std::vector<cudaEvent_t> ev(2 * n);
  for (auto& e : ev) cudaEventCreate(&e);
  cudaError_t err = rc ? cudaErrorUnknown : cudaSuccess;
  nxd::GemmFold f;
  for (int i = 0; i < n && err == cudaSuccess; ++i) {
    cudaEventRecord(ev[2 * i], nullptr);
    err = nxd::gemm_decode(wp, xm, bn, rows, tokens, K, static_cast<float*>(out), rows, ws, ws_bytes, sm_count,
                           nullptr, mode == 16 ? &f : nullptr);
    cudaEventRecord(ev[2 * i + 1], nullptr);
  }
  if (err == cudaSuccess && mode == 16) err = nxd::fold_store_f32(f, static_cast<float*>(out), nullptr);
  if (err == cudaSuccess) err = cudaDeviceSynchronize();
  std::vector<float> t(n, 0.f);
  for (int i = 0; i < n; ++i) cudaEventElapsedTime(&t[i], ev[2 * i], ev[2 * i + 1]);
  std::sort(t.begin(), t.end());
  if (ms) *ms = t[n / 2] * n;
  for (auto& e : ev) cudaEventDestroy(e);
  cudaFree(ws);
  cudaFree(wp);
  return rc ? rc : cuda_rc(err);
}

int nx_op_gemm(const void* x, const void* w, int32_t tokens, int32_t rows, int32_t K, int32_t mode,
               void* out, int32_t ldo, const void* bias, const void* residual, int32_t ldr,
               int32_t sm_count, int32_t splits, int32_t iters, float* ms) {
  return dguard([&] {
    if (mode == 16 || mode == 17) return op_gemm_decode(x, w, tokens, rows, K, mode, out, sm_count, iters, ms);
    const bool pair = splits == -2;  // CTA-pair prefill GEMM (gemm_tc2.cu)
    if (pair) splits = 0;
    const int bn = nxd::gemm_pick_bn(tokens);
    CUtensorMap xm;
    if (!nxd::encode_kmajor(&xm, x, tokens, K, static_cast<uint64_t>(K) * 2, bn))
      return dfail(NX_ERUNTIME, "tensor map encode failed");
    CUtensorMap xm128;
    if (!nxd::encode_kmajor(&xm128, x, tokens, K, static_cast<uint64_t>(K) * 2, 128))
      return dfail(NX_ERUNTIME, "tensor map encode failed");
    __nv_bfloat16* wp = nullptr;
    int prc = cuda_rc(cudaMalloc(&wp, nxd::packed_weight_elems(rows, K) * 2));
    if (prc) return prc;
    prc = cuda_rc(nxd::pack_weights(static_cast<const __nv_bfloat16*>(w), wp, rows, K, nullptr));
    if (prc) {
      cudaFree(wp);
      return prc;
    }
    int dev = 0;
    cudaGetDevice(&dev);
    int n_sm = 0;
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    if (sm_count <= 0 || sm_count > n_sm) sm_count = n_sm;
    float* ws = nullptr;
    const size_t ws_bytes = 256u << 20;
    int rc = cuda_rc(cudaMalloc(&ws, ws_bytes));
    if (rc) return rc;
    rc = cuda_rc(cudaMemset(ws, 0, nxd::gemm_counter_bytes()));
    if (rc) return rc;
    // Per-launch device time: an event pair around every launch, median
    // reported (host enqueue gaps between launches are excluded).
    const int n = iters > 0 ? iters : 1;
    std::vector<cudaEvent_t> ev(2 * n);
    for (auto& e : ev) cudaEventCreate(&e);
    cudaError_t err = cudaSuccess;
    for (int i = 0; i < n && err == cudaSuccess; ++i) {
      cudaEventRecord(ev[2 * i], nullptr);
      err = pair ? nxd::gemm_pair(wp, xm128, rows, tokens, K, mode, out, ldo,
                                  static_cast<const __nv_bfloat16*>(bias),
                                  static_cast<const __nv_bfloat16*>(residual), ldr, sm_count, nullptr)
                 : nxd::gemm(wp, xm, bn, rows, tokens, K, mode, out, ldo,
                             static_cast<const __nv_bfloat16*>(bias),
                             static_cast<const __nv_bfloat16*>(residual), ldr, ws, ws_bytes, sm_count,
                             nullptr, splits, /*coresident=*/true);
      cudaEventRecord(ev[2 * i + 1], nullptr);
    }
    if (err == cudaSuccess) err = cudaDeviceSynchronize();
    std::vector<float> t(n, 0.f);
    for (int i = 0; i < n; ++i) cudaEventElapsedTime(&t[i], ev[2 * i], ev[2 * i + 1]);
    std::sort(t.begin(), t.end());
    if (ms) *ms = t[n / 2] * n;  // median per launch, scaled so ms / iters = median
    for (auto& e : ev) cudaEventDestroy(e);
    cudaFree(ws);
    cudaFree(wp);
    return cuda_rc(err);
  });
}

}  // extern "C"
