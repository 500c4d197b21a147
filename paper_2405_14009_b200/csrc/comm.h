// comm.h — NCCL communicators of one rank: world, per-stage live-peer group (DP
// all-reduce) and one communicator + stream per directed worker pair
// that the plan uses (ReRouteAct / ReRouteGrad).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <map>
#include <utility>
#include <vector>

#include "planner.h"

struct slip_comm {
  int rank = 0, world = 1;
  int role = 0;  // worker position k*N + i this process plays (default: its world rank)
  int p2p_ctas = 2;  // CTAs per pair-communicator kernel (0: NCCL's default)
  ncclComm_t world_comm = nullptr;
  bool ready = false;
  slip::Cluster cl;
  int my_stage = 0, my_pipe = 0;
  bool my_live = true;
  ncclComm_t stage_comm = nullptr;  // live peers of my stage (nullptr if singleton / failed)
  ncclComm_t live_comm = nullptr;   // all live ranks (validation flags; nullptr if failed / alone)
  // validated mode: point-to-point validation flags of preceding stages,
  // a communicator of its own (the flag all-reduce uses live_comm on another stream)
  ncclComm_t val_comm = nullptr;
  cudaStream_t val_stream = nullptr;
  std::vector<int> val_rank;  // role -> rank in val_comm (-1: failed)
  int stage_size = 1;
  cudaStream_t ar_stream = nullptr;
  // directed pair (src rank, dst rank) -> communicator in which src is rank 0, dst rank 1
  std::map<std::pair<int, int>, ncclComm_t> pair_comm;
  std::map<std::pair<int, int>, cudaStream_t> pair_stream;
  // DP = 2 all-reduce fused into AdamW (slip_comm_fuse_ar_adam): the peer's fp32
  // gradient and barrier flag, mapped over NVLink with CUDA IPC
  bool fused_ar = false;
  const float* peer_grad = nullptr;
  const float* fused_local = nullptr;  // ctx->grad when the mapping was made
  unsigned* flags = nullptr;       // own flag word (cudaMalloc, exported to the peer)
  unsigned* peer_flags = nullptr;  // the peer's flag word
  void* ipc_grad_base = nullptr;   // opened IPC mappings (closed by destroy_setup)
  void* ipc_flag_base = nullptr;
  unsigned epoch = 0;
  // push mode (slip_comm_fuse_ar_push): W writes its 2-D weight gradients into the peer's
  // receive buffer as well (TMA over NVLink); AdamW reads them from this rank's own
  bool push = false;
  const float* my_recv = nullptr;  // this rank's receive buffer (the peer writes it)
  float* peer_recv = nullptr;      // the peer's receive buffer (mapped)
  void* ipc_recv_base = nullptr;
};

#define SLIP_NCCL(expr)                                          \
  do {                                                           \
    ncclResult_t _r = (expr);                                    \
    if (_r != ncclSuccess) return ::slip::nccl_status(_r, #expr); \
  } while (0)

namespace slip {
// worker (stage i, pipeline k) <-> rank k*N + i
inline int rank_of(int N, int i, int k) { return k * N + i; }
slip_status nccl_status(ncclResult_t r, const char* where);
}  // namespace slip
