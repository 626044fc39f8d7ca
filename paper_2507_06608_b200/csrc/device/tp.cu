// Tensor-parallel plumbing: shard plan + NCCL binding (see tp.cuh).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <stdexcept>

#include "device.cuh"
#include "tp.cuh"

namespace nxd {

nx_tp_shard tp_plan(const nx_arch& a, int tp, int r) {
  if (tp < 1 || r < 0 || r >= tp) throw std::invalid_argument("bad tp rank/size");
  if (a.n_heads % tp || a.n_kv_heads % tp)
    throw std::invalid_argument("heads and kv heads must divide by tp");
  if (a.ffn % (64 * tp)) throw std::invalid_argument("ffn must divide into 64-feature blocks per rank");
  nx_tp_shard s{};
  s.tp_size = tp;
  s.rank = r;
  s.n_q_heads = a.n_heads / tp;
  s.q_head0 = r * s.n_q_heads;
  s.n_kv_heads = a.n_kv_heads / tp;
  s.kv_head0 = r * s.n_kv_heads;
  s.ffn_local = a.ffn / tp;
  s.ffn0 = r * s.ffn_local;
  const int block = 128 * tp;
  s.vocab_padded = (a.vocab + block - 1) / block * block;
  s.vocab_local = s.vocab_padded / tp;
  s.vocab0 = r * s.vocab_local;
  s.vocab_valid = std::max(0, std::min(s.vocab_local, a.vocab - s.vocab0));
  return s;
}

namespace {
using GetId = ncclResult_t (*)(ncclUniqueId*);
using Init = ncclResult_t (*)(ncclComm_t*, int, ncclUniqueId, int);
using AllReduce = ncclResult_t (*)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                                   ncclComm_t, cudaStream_t);
using AllGather = ncclResult_t (*)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                                   cudaStream_t);
using Bcast = ncclResult_t (*)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                               cudaStream_t);
using Destroy = ncclResult_t (*)(ncclComm_t);
using ErrStr = const char* (*)(ncclResult_t);
const char* const kNames[] = {"ncclGetUniqueId", "ncclCommInitRank", "ncclAllReduce",
                              "ncclAllGather", "ncclBroadcast", "ncclCommDestroy",
                              "ncclGetErrorString"};
}  // namespace

Nccl::Nccl() {
  // RTLD_LOCAL: never let our NCCL interpose on another library's (torch
  // links its own); a copy already loaded under the same soname is reused.
  // NX_NCCL_LIB selects a specific libnccl.so.
  const char* env = std::getenv("NX_NCCL_LIB");
  if (env && *env) lib_ = dlopen(env, RTLD_NOW | RTLD_LOCAL);
  for (const char* so : {"libnccl.so.2", "libnccl.so"}) {
    if (lib_) break;
    lib_ = dlopen(so, RTLD_NOW | RTLD_LOCAL);
  }
  if (!lib_) throw std::runtime_error("NCCL (libnccl.so.2) not found");
  for (int i = 0; i < 7; ++i) {
    sym_[i] = dlsym(lib_, kNames[i]);
    if (!sym_[i]) throw std::runtime_error(std::string("NCCL symbol missing: ") + kNames[i]);
  }
}

Nccl& Nccl::get() {
  static Nccl n;
  return n;
}

void Nccl::check(int rc, const char* what) {
  if (rc != ncclSuccess)
    throw std::runtime_error(std::string(what) + ": " +
                             reinterpret_cast<ErrStr>(sym_[6])(static_cast<ncclResult_t>(rc)));
}

void Nccl::unique_id(uint8_t out[128]) {
  ncclUniqueId id;
  check(reinterpret_cast<GetId>(sym_[0])(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, 128);
}

void* Nccl::comm_init(int nranks, const uint8_t raw[128], int rank) {
  ncclUniqueId id;
  std::memcpy(id.internal, raw, 128);
  ncclComm_t c = nullptr;
  check(reinterpret_cast<Init>(sym_[1])(&c, nranks, id, rank), "ncclCommInitRank");
  return c;
}

void Nccl::all_reduce_bf16(void* comm, void* buf, size_t n, cudaStream_t s) {
  check(reinterpret_cast<AllReduce>(sym_[2])(buf, buf, n, ncclBfloat16, ncclSum,
                                            static_cast<ncclComm_t>(comm), s),
        "ncclAllReduce");
}

void Nccl::all_gather_f2(void* comm, const void* send, void* recv, size_t n, cudaStream_t s) {
  check(reinterpret_cast<AllGather>(sym_[3])(send, recv, n, ncclFloat32,
                                            static_cast<ncclComm_t>(comm), s),
        "ncclAllGather");
}

void Nccl::broadcast_bytes(void* comm, void* buf, size_t bytes, int root, cudaStream_t s) {
  check(reinterpret_cast<Bcast>(sym_[4])(buf, buf, bytes, ncclUint8, root,
                                        static_cast<ncclComm_t>(comm), s),
        "ncclBroadcast");
}

void Nccl::destroy(void* comm) {
  if (comm) reinterpret_cast<Destroy>(sym_[5])(static_cast<ncclComm_t>(comm));
}

// ---------------------------------------------------------------------------
// Peer-memory collectives.
// ---------------------------------------------------------------------------
namespace {

struct PeerArgs {
  const void* src[kPeerMaxRanks];  // every rank's slot buffer for this epoch
  void* mine;                      // this rank's slot buffer
  uint32_t* flag_dst[kPeerMaxRanks];  // rank p's flag row for *this* rank
  const uint32_t* flag_src;           // this rank's flags [rank][chunk]
  int tp, rank;
  uint32_t epoch;
  size_t n, chunk;  // elements (bf16: 8-element vectors), per-CTA chunk
  int* err;
};

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Threads 0..tp-1 push this chunk's flag to every rank, then wait for every
// rank's flag of the same chunk (bounded: 10 s, then flag an error and go on
// rather than hang the GPU).
__device__ __forceinline__ void peer_barrier(const PeerArgs& a, int chunk) {
  __syncthreads();
  if (threadIdx.x < a.tp) {
    __threadfence_system();
    st_release_sys(a.flag_dst[threadIdx.x] + chunk, a.epoch);
    const uint32_t* f = a.flag_src + threadIdx.x * kPeerMaxChunks + chunk;
    const uint64_t t0 = globaltimer();
    while (ld_acquire_sys(f) < a.epoch) {
      if (globaltimer() - t0 > 10000000000ull) {
        atomicExch(a.err, 1);
        break;
      }
    }
  }
  __syncthreads();
}

__global__ void peer_allreduce_kernel(PeerArgs a, __nv_bfloat16* x) {
  pdl_wait();
  const size_t v0 = (blockIdx.x * a.chunk) / 8, v1 = min(a.n, (blockIdx.x + 1) * a.chunk) / 8;
  uint4* mine = static_cast<uint4*>(a.mine);
  const uint4* xv = reinterpret_cast<const uint4*>(x);
  for (size_t i = v0 + threadIdx.x; i < v1; i += blockDim.x) mine[i] = xv[i];
  peer_barrier(a, blockIdx.x);
  uint4* out = reinterpret_cast<uint4*>(x);
  for (size_t i = v0 + threadIdx.x; i < v1; i += blockDim.x) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int r = 0; r < a.tp; ++r) {
      const uint4 v = __ldcg(static_cast<const uint4*>(a.src[r]) + i);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = __bfloat1622float2(h[k]);
        acc[2 * k] += f.x;
        acc[2 * k + 1] += f.y;
      }
    }
    uint4 o;
    __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int k = 0; k < 4; ++k) oh[k] = __floats2bfloat162_rn(acc[2 * k], acc[2 * k + 1]);
    out[i] = o;
  }
}

__global__ void peer_argmax_kernel(PeerArgs a, const float2* mine_pairs, int32_t* out) {
  pdl_wait();
  float2* mine = static_cast<float2*>(a.mine);
  for (int i = threadIdx.x; i < static_cast<int>(a.n); i += blockDim.x) mine[i] = mine_pairs[i];
  peer_barrier(a, 0);
  for (int i = threadIdx.x; i < static_cast<int>(a.n); i += blockDim.x) {
    float best = -3.402823466e38f;
    int idx = 0x7fffffff;
    for (int r = 0; r < a.tp; ++r) {
      const float2 p = __ldcg(static_cast<const float2*>(a.src[r]) + i);
      const int j = __float_as_int(p.y);
      if (p.x > best || (p.x == best && j < idx)) best = p.x, idx = j;
    }
    out[i] = idx;
  }
}

}  // namespace

PeerGroup::PeerGroup(int tp, bool colocated) : tp_(tp), colocated_(colocated) {
  if (tp < 2 || tp > kPeerMaxRanks) throw std::invalid_argument("peer TP group size must be 2..8");
  if (cudaHostAlloc(&err_host_, sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable) !=
      cudaSuccess)
    throw std::runtime_error("peer group: pinned error flag");
  *err_host_ = 0;
  if (cudaHostGetDevicePointer(reinterpret_cast<void**>(&err_dev_), err_host_, 0) != cudaSuccess)
    throw std::runtime_error("peer group: mapped error flag");
}

PeerGroup::~PeerGroup() {
  for (int r = 0; r < kPeerMaxRanks; ++r) release_rank(r);
  if (err_host_) cudaFreeHost(err_host_);
}

void PeerGroup::register_lane(int rank, int lane, size_t max_elems) {
  Slot& sl = slot_[rank][lane];
  const size_t bytes = (max_elems * 2 + 255) / 256 * 256;
  for (void*& b : sl.buf)
    if (cudaMalloc(&b, bytes) != cudaSuccess) throw std::runtime_error("peer group: buffer alloc");
  const size_t fb = sizeof(uint32_t) * kPeerMaxRanks * kPeerMaxChunks;
  if (cudaMalloc(&sl.flags, fb) != cudaSuccess || cudaMemset(sl.flags, 0, fb) != cudaSuccess)
    throw std::runtime_error("peer group: flag alloc");
  sl.epoch = 0;
}

void PeerGroup::release_rank(int rank) {
  for (Slot& sl : slot_[rank]) {
    for (void*& b : sl.buf) {
      if (b) cudaFree(b);
      b = nullptr;
    }
    if (sl.flags) cudaFree(sl.flags);
    sl.flags = nullptr;
  }
}

static PeerArgs make_args(int tp, int rank, uint32_t epoch, int* err, size_t n, size_t chunk,
                          void* (*bufs)[2], uint32_t** flags) {
  PeerArgs a{};
  const int parity = epoch & 1;
  for (int r = 0; r < tp; ++r) {
    a.src[r] = bufs[r][parity];
    a.flag_dst[r] = flags[r] + static_cast<size_t>(rank) * kPeerMaxChunks;
  }
  a.mine = bufs[rank][parity];
  a.flag_src = flags[rank];
  a.tp = tp;
  a.rank = rank;
  a.epoch = epoch;
  a.n = n;
  a.chunk = chunk;
  a.err = err;
  return a;
}

void PeerGroup::all_reduce_bf16(int rank, int lane, __nv_bfloat16* x, size_t n, int max_ctas,
                                cudaStream_t s) {
  if (n == 0) return;
  if (n % 8) throw std::invalid_argument("peer all-reduce: n must be a multiple of 8");
  void* bufs[kPeerMaxRanks][2];
  uint32_t* flags[kPeerMaxRanks];
  for (int r = 0; r < tp_; ++r) {
    bufs[r][0] = slot_[r][lane].buf[0];
    bufs[r][1] = slot_[r][lane].buf[1];
    flags[r] = slot_[r][lane].flags;
  }
  const size_t cap = static_cast<size_t>(std::max(1, colocated_ ? std::min(max_ctas, 4) : max_ctas));
  const size_t grid = std::min<size_t>({static_cast<size_t>(kPeerMaxChunks), cap,
                                        std::max<size_t>(1, (n + 8191) / 8192)});
  const size_t chunk = ((n + grid - 1) / grid + 7) / 8 * 8;
  const uint32_t epoch = ++slot_[rank][lane].epoch;
  PeerArgs a = make_args(tp_, rank, epoch, err_dev_, n, chunk, bufs, flags);
  ++g_kernel_launches;
  peer_allreduce_kernel<<<static_cast<unsigned>((n + chunk - 1) / chunk), 256, 0, s>>>(a, x);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("peer all-reduce: ") + cudaGetErrorString(e));
}

void PeerGroup::argmax_gather(int rank, int lane, const float2* mine, int n, int32_t* out,
                              cudaStream_t s) {
  if (n == 0) return;
  void* bufs[kPeerMaxRanks][2];
  uint32_t* flags[kPeerMaxRanks];
  for (int r = 0; r < tp_; ++r) {
    bufs[r][0] = slot_[r][lane].buf[0];
    bufs[r][1] = slot_[r][lane].buf[1];
    flags[r] = slot_[r][lane].flags;
  }
  const uint32_t epoch = ++slot_[rank][lane].epoch;
  PeerArgs a = make_args(tp_, rank, epoch, err_dev_, static_cast<size_t>(n), 0, bufs, flags);
  ++g_kernel_launches;
  peer_argmax_kernel<<<1, 256, 0, s>>>(a, mine, out);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("peer argmax: ") + cudaGetErrorString(e));
}

void prepare_tp_kernels() {
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, peer_allreduce_kernel);
  cudaFuncGetAttributes(&fa, peer_argmax_kernel);
}

}  // namespace nxd
