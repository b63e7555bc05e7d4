// Communication layer of the executor: the TP all-reduce windows and the 1F1B
// pipeline send / recv. Two implementations behind one interface:
//
//   * NcclComms — one process per GPU: a world communicator split into the TP
//     group (ranks of one stage) and two pipeline communicators (activations
//     s -> s+1, gradients s+1 -> s), each driven from its own CUDA stream.
//   * LoopbackComms — every rank of a TP x PP grid inside ONE process on one GPU,
//     one executor per rank, each driven by its own host thread. NCCL cannot put
//     two ranks on one device, so this is how the sharded numerics (column / row
//     split weights, all-reduce placement, pipeline hand-off) are checked against
//     the unsharded oracle on a single B200. The all-reduce sums every rank's
//     partial in fixed rank order in fp32 and rounds once to bf16 — the result a
//     two-rank NCCL ring produces — and writes it to every rank's buffer. Sends
//     are buffered (copied into a staging buffer, never block the host); receives
//     block the host thread until the matching send was issued, then order their
//     stream after it. With buffered sends the 1F1B programs cannot deadlock.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace lynx::rt {

struct RtError : std::runtime_error {
  RtError(const std::string& w, int c) : std::runtime_error(w), code(c) {}
  int code;
};

enum class Channel { TP = 0, PP_ACT = 1, PP_GRAD = 2 };

class Comms {
 public:
  virtual ~Comms() = default;
  // In-place sum over the TP group of `count` bf16 elements, stream-ordered on s.
  virtual void allreduce_sum_bf16(void* buf, size_t count, cudaStream_t s) = 0;
  // In-place fp32 MAX (max = true) or SUM over the TP group (the vocab-parallel cross-entropy's row
  // statistics), stream-ordered on s.
  virtual void allreduce_f32(float* buf, size_t count, bool max, cudaStream_t s) = 0;
  // Pipeline hand-off of `count` bf16 elements to / from stage `peer` (same TP rank).
  virtual void send_bf16(const void* buf, size_t count, int peer, Channel ch, cudaStream_t s) = 0;
  virtual void recv_bf16(void* buf, size_t count, int peer, Channel ch, cudaStream_t s) = 0;
  virtual const char* kind() const = 0;

  // Fused row-parallel reductions (exec.tp_fused): two staging slots of `bytes` per rank that every rank
  // of the TP group can read in place (the same device in the loopback grid, CUDA-IPC peer mappings over
  // NVLink across processes). A rank writes its partial into its own slot (call k uses slot k % 2); after
  // fused_barrier(k, s) — stream-ordered on s, no host wait on the device — every rank's slot of call k
  // is complete and readable. Two slots suffice: a rank rewrites slot k % 2 at call k + 2 only after its
  // own reduction of call k + 1, which waited for every peer's call k + 1 partial, written after that
  // peer's reduction of call k (stream order) had finished reading the slot.
  virtual void fused_setup(size_t bytes) = 0;
  virtual void* fused_slot(int slot) = 0;
  virtual std::vector<const void*> fused_peers(int slot) = 0;  // every rank's slot, rank order
  virtual void fused_barrier(long long k, cudaStream_t s) = 0;
};

// id_hex: hex ncclUniqueId ("" with world_size 1: a private one-rank world).
std::unique_ptr<Comms> make_nccl_comms(const std::string& id_hex, int world_rank, int world_size, int pp_rank,
                                       int tp_rank);
// All tp * pp ranks of the grid `name` must be created in this process (any order, any thread).
std::unique_ptr<Comms> make_loopback_comms(const std::string& name, int tp, int pp, int pp_rank, int tp_rank);

// Host-side hex <-> ncclUniqueId.
std::string nccl_unique_id_hex();

}  // namespace lynx::rt
