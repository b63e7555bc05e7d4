// NCCL and in-process loopback implementations of the executor's Comms (comm.hpp).
#include "runtime/comm.hpp"

#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <deque>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "lynx_ops_internal.h"

namespace lynx::rt {

namespace {

void cuda_ck(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  cudaGetLastError();
  if (e == cudaErrorMemoryAllocation) throw RtError(std::string(what) + ": out of device memory", kOutOfMemory);
  throw RtError(std::string(what) + ": " + cudaGetErrorString(e), kCudaError);
}

void nccl_ck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw RtError(std::string(what) + ": " + ncclGetErrorString(r), kCudaError);
}

int hex_val(char c) {
  if (c >= '0' && c <= '9') return c - '0';
  if (c >= 'a' && c <= 'f') return c - 'a' + 10;
  if (c >= 'A' && c <= 'F') return c - 'A' + 10;
  return -1;
}

// ------------------------------------------------------------------ NCCL
class NcclComms final : public Comms {
 public:
  NcclComms(const std::string& id_hex, int world_rank, int world_size, int pp_rank, int tp_rank) {
    ncclUniqueId id;
    if (id_hex.empty() && world_size == 1) {
      // Single rank with the TP template: the all-reduce windows run on a
      // one-rank communicator (identity reduction), exercising the same streams.
      nccl_ck(ncclGetUniqueId(&id), "ncclGetUniqueId");
    } else {
      if (id_hex.size() != 2 * sizeof(ncclUniqueId))
        throw RtError("parallel.nccl_id must be a hex ncclUniqueId", kValidation);
      for (size_t i = 0; i < sizeof(id); ++i) {
        const int hi = hex_val(id_hex[2 * i]), lo = hex_val(id_hex[2 * i + 1]);
        if (hi < 0 || lo < 0) throw RtError("parallel.nccl_id is not hex", kValidation);
        id.internal[i] = static_cast<char>(hi * 16 + lo);
      }
    }
    nccl_ck(ncclCommInitRank(&world_, world_size, id, world_rank), "ncclCommInitRank");
    // TP groups: ranks sharing a pipeline stage; PP groups: ranks sharing a TP rank.
    // Activations (s -> s+1) and gradients (s+1 -> s) use separate communicators and
    // streams, so the two directions of 1F1B never wait on each other.
    nccl_ck(ncclCommSplit(world_, pp_rank, tp_rank, &tp_, nullptr), "split tp");
    nccl_ck(ncclCommSplit(world_, tp_rank, pp_rank, &pa_, nullptr), "split pp act");
    nccl_ck(ncclCommSplit(world_, tp_rank, pp_rank, &pg_, nullptr), "split pp grad");
  }
  void allreduce_sum_bf16(void* buf, size_t count, cudaStream_t s) override {
    nccl_ck(ncclAllReduce(buf, buf, count, ncclBfloat16, ncclSum, tp_, s), "allreduce");
  }
  void allreduce_f32(float* buf, size_t count, bool max, cudaStream_t s) override {
    nccl_ck(ncclAllReduce(buf, buf, count, ncclFloat32, max ? ncclMax : ncclSum, tp_, s), "allreduce f32");
  }
  void send_bf16(const void* buf, size_t count, int peer, Channel ch, cudaStream_t s) override {
    nccl_ck(ncclSend(buf, count, ncclBfloat16, peer, ch == Channel::PP_ACT ? pa_ : pg_, s), "send");
  }
  void recv_bf16(void* buf, size_t count, int peer, Channel ch, cudaStream_t s) override {
    nccl_ck(ncclRecv(buf, count, ncclBfloat16, peer, ch == Channel::PP_ACT ? pa_ : pg_, s), "recv");
  }
  const char* kind() const override { return "nccl"; }

  // Staging slots and flags in cudaMalloc'd memory, exchanged as CUDA-IPC handles over the TP
  // communicator (ncclAllGather of the handle bytes) and opened as peer mappings.
  void fused_setup(size_t bytes) override {
    if (base_) return;
    bytes_ = bytes;
    int n = 0, me = 0;
    nccl_ck(ncclCommCount(tp_, &n), "comm count");
    nccl_ck(ncclCommUserRank(tp_, &me), "comm rank");
    if (n > kMaxTpRanks) throw RtError("tp_fused supports up to 8 TP ranks", kValidation);
    n_ = n;
    me_ = me;
    cuda_ck(cudaMalloc(&base_, 2 * bytes), "fused staging");
    cuda_ck(cudaMalloc(&flags_, kMaxTpRanks * sizeof(unsigned long long)), "fused flags");
    cuda_ck(cudaMemset(flags_, 0, kMaxTpRanks * sizeof(unsigned long long)), "fused flags");
    cudaIpcMemHandle_t h[2];
    cuda_ck(cudaIpcGetMemHandle(&h[0], base_), "ipc handle");
    cuda_ck(cudaIpcGetMemHandle(&h[1], flags_), "ipc handle");
    void *d_send = nullptr, *d_recv = nullptr;
    cuda_ck(cudaMalloc(&d_send, sizeof(h)), "ipc exchange");
    cuda_ck(cudaMalloc(&d_recv, sizeof(h) * n), "ipc exchange");
    cuda_ck(cudaMemcpy(d_send, h, sizeof(h), cudaMemcpyHostToDevice), "ipc exchange");
    nccl_ck(ncclAllGather(d_send, d_recv, sizeof(h), ncclUint8, tp_, nullptr), "ipc allgather");
    cuda_ck(cudaStreamSynchronize(nullptr), "ipc exchange");
    std::vector<cudaIpcMemHandle_t> all(2 * n);
    cuda_ck(cudaMemcpy(all.data(), d_recv, sizeof(h) * n, cudaMemcpyDeviceToHost), "ipc exchange");
    cudaFree(d_send);
    cudaFree(d_recv);
    for (int r = 0; r < n; ++r) {
      if (r == me) {
        peer_base_[r] = base_;
        peer_flags_.f[r] = static_cast<unsigned long long*>(flags_);
        continue;
      }
      cuda_ck(cudaIpcOpenMemHandle(&peer_base_[r], all[2 * r], cudaIpcMemLazyEnablePeerAccess), "ipc open");
      void* f = nullptr;
      cuda_ck(cudaIpcOpenMemHandle(&f, all[2 * r + 1], cudaIpcMemLazyEnablePeerAccess), "ipc open");
      peer_flags_.f[r] = static_cast<unsigned long long*>(f);
    }
  }
  void* fused_slot(int slot) override { return static_cast<char*>(base_) + slot * bytes_; }
  std::vector<const void*> fused_peers(int slot) override {
    std::vector<const void*> v;
    for (int r = 0; r < n_; ++r) v.push_back(static_cast<const char*>(peer_base_[r]) + slot * bytes_);
    return v;
  }
  void fused_barrier(long long k, cudaStream_t s) override {
    if (tp_signal_wait(peer_flags_, static_cast<const unsigned long long*>(flags_), n_, me_,
                       static_cast<unsigned long long>(k + 1), s) != kOk)
      throw RtError(last_error(), kCudaError);
  }
  ~NcclComms() override {
    if (base_ && tp_) {
      // Peers read this rank's staging slots in place: free them only after every TP rank got here.
      // Each executor synchronises its own streams before destroying its communicators, so once all
      // ranks passed this collective no consumer kernel reads a slot any more.
      void* one = nullptr;
      if (cudaMalloc(&one, sizeof(float)) == cudaSuccess) {
        if (ncclAllReduce(one, one, 1, ncclFloat, ncclSum, tp_, nullptr) == ncclSuccess) cudaStreamSynchronize(nullptr);
        cudaFree(one);
      }
    }
    for (int r = 0; r < n_; ++r)
      if (r != me_) {
        if (peer_base_[r]) cudaIpcCloseMemHandle(peer_base_[r]);
        if (peer_flags_.f[r]) cudaIpcCloseMemHandle(peer_flags_.f[r]);
      }
    if (base_) cudaFree(base_);
    if (flags_) cudaFree(flags_);
    for (ncclComm_t c : {tp_, pa_, pg_, world_})
      if (c) ncclCommDestroy(c);
  }

 private:
  ncclComm_t world_ = nullptr, tp_ = nullptr, pa_ = nullptr, pg_ = nullptr;
  void *base_ = nullptr, *flags_ = nullptr;
  size_t bytes_ = 0;
  int n_ = 0, me_ = 0;
  void* peer_base_[kMaxTpRanks] = {};
  TpFlags peer_flags_{};
};

// ------------------------------------------------------------------ loopback
constexpr int kMaxTp = 8;
constexpr auto kPeerTimeout = std::chrono::seconds(300);

struct PtrPack {
  __nv_bfloat16* p[kMaxTp];
};

// out = bf16(sum_r float(in_r)) in rank order, written to every rank's buffer.
__global__ void loopback_sum_kernel(PtrPack ptrs, int n, long long nvec, long long count) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long v = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; v < nvec; v += stride) {
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int r = 0; r < n; ++r) {
      float f[8];
      bf8_to_f(reinterpret_cast<const BF8*>(ptrs.p[r])[v], f);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += f[j];
    }
    const BF8 o = f_to_bf8(acc);
    for (int r = 0; r < n; ++r) reinterpret_cast<BF8*>(ptrs.p[r])[v] = o;
  }
  for (long long i = 8 * nvec + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < count; i += stride) {
    float acc = 0.f;
    for (int r = 0; r < n; ++r) acc += bf2f(ptrs.p[r][i]);
    for (int r = 0; r < n; ++r) ptrs.p[r][i] = f2bf(acc);
  }
}

struct PtrPackF {
  float* p[kMaxTp];
};

// fp32 MAX / SUM over the ranks in rank order, written to every rank's buffer.
__global__ void loopback_f32_kernel(PtrPackF ptrs, int n, long long count, int is_max) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    float acc = ptrs.p[0][i];
    for (int r = 1; r < n; ++r) acc = is_max ? fmaxf(acc, ptrs.p[r][i]) : acc + ptrs.p[r][i];
    for (int r = 0; r < n; ++r) ptrs.p[r][i] = acc;
  }
}

struct ArCall {
  int arrived = 0, left = 0;
  bool complete = false;
  size_t count = 0;
  int kind = 0;
  void* bufs[kMaxTp] = {};
  cudaEvent_t ready[kMaxTp] = {};
  cudaEvent_t done = nullptr;
};

struct TpGroup {
  std::mutex mu;
  std::condition_variable cv;
  std::map<long long, ArCall> calls;
};

struct Msg {
  void* staging;
  size_t bytes;
  cudaEvent_t ready;
};

struct Link {
  std::mutex mu;
  std::condition_variable cv;
  std::deque<Msg> q;
};

struct Grid {
  int tp = 1, pp = 1;
  std::vector<std::unique_ptr<TpGroup>> groups;  // one per stage
  std::vector<std::vector<void*>> fused;          // [stage][tp rank]: staging base (exec.tp_fused)
  std::mutex links_mu;
  std::map<std::tuple<int, int, int, int>, std::unique_ptr<Link>> links;  // (channel, src, dst, tp_rank)
  Link& link(Channel ch, int src, int dst, int tp_rank) {
    std::lock_guard<std::mutex> g(links_mu);
    auto& p = links[{static_cast<int>(ch), src, dst, tp_rank}];
    if (!p) p = std::make_unique<Link>();
    return *p;
  }
};

std::mutex g_grids_mu;
std::map<std::string, std::weak_ptr<Grid>> g_grids;

class LoopbackComms final : public Comms {
 public:
  LoopbackComms(const std::string& name, int tp, int pp, int pp_rank, int tp_rank)
      : tp_(tp), pp_rank_(pp_rank), tp_rank_(tp_rank) {
    if (tp < 1 || tp > kMaxTp || pp < 1 || pp_rank < 0 || pp_rank >= pp || tp_rank < 0 || tp_rank >= tp)
      throw RtError("loopback grid: rank out of range (tp <= 8)", kValidation);
    std::lock_guard<std::mutex> g(g_grids_mu);
    grid_ = g_grids[name].lock();
    if (!grid_) {
      grid_ = std::make_shared<Grid>();
      grid_->tp = tp;
      grid_->pp = pp;
      for (int s = 0; s < pp; ++s) grid_->groups.push_back(std::make_unique<TpGroup>());
      grid_->fused.assign(pp, std::vector<void*>(tp, nullptr));
      g_grids[name] = grid_;
    } else if (grid_->tp != tp || grid_->pp != pp) {
      throw RtError("loopback grid '" + name + "' exists with a different tp x pp shape", kValidation);
    }
  }

  void allreduce_sum_bf16(void* buf, size_t count, cudaStream_t s) override { reduce(buf, count, 0, s); }
  void allreduce_f32(float* buf, size_t count, bool max, cudaStream_t s) override {
    reduce(buf, count, max ? 2 : 1, s);
  }

  void fused_setup(size_t bytes) override {
    if (base_) return;
    bytes_ = bytes;
    cuda_ck(cudaMalloc(&base_, 2 * bytes), "fused staging");
    TpGroup& g = *grid_->groups[pp_rank_];
    std::lock_guard<std::mutex> lk(g.mu);
    grid_->fused[pp_rank_][tp_rank_] = base_;
    g.cv.notify_all();
  }
  void* fused_slot(int slot) override { return static_cast<char*>(base_) + slot * bytes_; }
  std::vector<const void*> fused_peers(int slot) override {
    TpGroup& g = *grid_->groups[pp_rank_];
    std::unique_lock<std::mutex> lk(g.mu);
    auto& row = grid_->fused[pp_rank_];
    if (!g.cv.wait_for(lk, kPeerTimeout, [&] {
          for (void* p : row)
            if (!p) return false;
          return true;
        }))
      throw RtError("loopback tp_fused: a TP peer never set up its staging", kCudaError);
    std::vector<const void*> v;
    for (void* p : row) v.push_back(static_cast<const char*>(p) + slot * bytes_);
    return v;
  }
  // every rank's stream waits for every rank's partial of call k (events only; no kernel)
  void fused_barrier(long long k, cudaStream_t s) override { reduce(nullptr, 0, 3, s); }
  ~LoopbackComms() override {
    if (base_) {
      cudaDeviceSynchronize();  // peers may still read this rank's slots
      cudaFree(base_);
    }
  }

  // kind 0: bf16 SUM (fp32 accumulation), 1: fp32 SUM, 2: fp32 MAX, 3: barrier only. Every rank of the
  // TP group calls
  // its collectives in the same order (identical programs), so the k-th call of each rank matches.
  void reduce(void* buf, size_t count, int kind, cudaStream_t s) {
    if (tp_ == 1) return;
    TpGroup& g = *grid_->groups[pp_rank_];
    const long long k = seq_++;
    cudaEvent_t ready;
    cuda_ck(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming), "event");
    cuda_ck(cudaEventRecord(ready, s), "event");
    std::unique_lock<std::mutex> lk(g.mu);
    ArCall& c = g.calls[k];
    if (c.arrived && (c.count != count || c.kind != kind))
      throw RtError("loopback all-reduce: ranks disagree on the size or type", kCudaError);
    c.count = count;
    c.kind = kind;
    c.bufs[tp_rank_] = buf;
    c.ready[tp_rank_] = ready;
    if (++c.arrived == tp_) {  // last to arrive reduces for everyone
      for (int r = 0; r < tp_; ++r) cuda_ck(cudaStreamWaitEvent(s, c.ready[r], 0), "wait");
      if (kind == 3) {
        // barrier: the waits above are the whole operation
      } else if (kind == 0) {
        PtrPack pk{};
        for (int r = 0; r < tp_; ++r) pk.p[r] = static_cast<__nv_bfloat16*>(c.bufs[r]);
        const long long nvec = static_cast<long long>(count / 8);
        long long blocks = (nvec + 255) / 256;
        blocks = blocks < 1 ? 1 : (blocks > 148 * 8 ? 148 * 8 : blocks);
        loopback_sum_kernel<<<static_cast<int>(blocks), 256, 0, s>>>(pk, tp_, nvec, static_cast<long long>(count));
      } else {
        PtrPackF pk{};
        for (int r = 0; r < tp_; ++r) pk.p[r] = static_cast<float*>(c.bufs[r]);
        long long blocks = (static_cast<long long>(count) + 255) / 256;
        blocks = blocks < 1 ? 1 : (blocks > 148 * 8 ? 148 * 8 : blocks);
        loopback_f32_kernel<<<static_cast<int>(blocks), 256, 0, s>>>(pk, tp_, static_cast<long long>(count),
                                                                     kind == 2 ? 1 : 0);
      }
      if (kind != 3 && check_launch("loopback_allreduce") != kOk) throw RtError(last_error(), kCudaError);
      cuda_ck(cudaEventCreateWithFlags(&c.done, cudaEventDisableTiming), "event");
      cuda_ck(cudaEventRecord(c.done, s), "event");
      c.complete = true;
      g.cv.notify_all();
    } else {
      if (!g.cv.wait_for(lk, kPeerTimeout, [&] { return c.complete; }))
        throw RtError("loopback all-reduce: a TP peer did not arrive", kCudaError);
      cuda_ck(cudaStreamWaitEvent(s, c.done, 0), "wait");
    }
    if (++c.left == tp_) {  // every rank has ordered its stream after the reduction
      for (int r = 0; r < tp_; ++r) cudaEventDestroy(c.ready[r]);
      cudaEventDestroy(c.done);
      g.calls.erase(k);
    }
  }

  void send_bf16(const void* buf, size_t count, int peer, Channel ch, cudaStream_t s) override {
    Link& L = grid_->link(ch, pp_rank_, peer, tp_rank_);
    const size_t bytes = count * 2;
    Msg m{nullptr, bytes, nullptr};
    cuda_ck(cudaMallocAsync(&m.staging, bytes, s), "loopback send staging");
    cuda_ck(cudaMemcpyAsync(m.staging, buf, bytes, cudaMemcpyDeviceToDevice, s), "loopback send");
    cuda_ck(cudaEventCreateWithFlags(&m.ready, cudaEventDisableTiming), "event");
    cuda_ck(cudaEventRecord(m.ready, s), "event");
    std::lock_guard<std::mutex> g(L.mu);
    L.q.push_back(m);
    L.cv.notify_all();
  }

  void recv_bf16(void* buf, size_t count, int peer, Channel ch, cudaStream_t s) override {
    Link& L = grid_->link(ch, peer, pp_rank_, tp_rank_);
    Msg m;
    {
      std::unique_lock<std::mutex> lk(L.mu);
      if (!L.cv.wait_for(lk, kPeerTimeout, [&] { return !L.q.empty(); }))
        throw RtError("loopback recv: the peer stage never sent", kCudaError);
      m = L.q.front();
      L.q.pop_front();
    }
    if (m.bytes != count * 2) throw RtError("loopback recv: message size mismatch", kCudaError);
    cuda_ck(cudaStreamWaitEvent(s, m.ready, 0), "wait");
    cuda_ck(cudaMemcpyAsync(buf, m.staging, m.bytes, cudaMemcpyDeviceToDevice, s), "loopback recv");
    cuda_ck(cudaFreeAsync(m.staging, s), "loopback recv free");
    cudaEventDestroy(m.ready);
  }

  const char* kind() const override { return "loopback"; }

 private:
  std::shared_ptr<Grid> grid_;
  int tp_, pp_rank_, tp_rank_;
  long long seq_ = 0;
  void* base_ = nullptr;
  size_t bytes_ = 0;
};

}  // namespace

std::unique_ptr<Comms> make_nccl_comms(const std::string& id_hex, int world_rank, int world_size, int pp_rank,
                                       int tp_rank) {
  return std::make_unique<NcclComms>(id_hex, world_rank, world_size, pp_rank, tp_rank);
}

std::unique_ptr<Comms> make_loopback_comms(const std::string& name, int tp, int pp, int pp_rank, int tp_rank) {
  return std::make_unique<LoopbackComms>(name, tp, pp, pp_rank, tp_rank);
}

std::string nccl_unique_id_hex() {
  ncclUniqueId id;
  nccl_ck(ncclGetUniqueId(&id), "ncclGetUniqueId");
  static const char* hx = "0123456789abcdef";
  std::string out(2 * sizeof(id), '0');
  for (size_t i = 0; i < sizeof(id); ++i) {
    const unsigned char c = static_cast<unsigned char>(id.internal[i]);
    out[2 * i] = hx[c >> 4];
    out[2 * i + 1] = hx[c & 15];
  }
  return out;
}

}  // namespace lynx::rt
