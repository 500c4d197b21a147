// comm.cpp — NCCL bootstrap, per-stage and per-pair communicators, the stage gradient
// all-reduce (slip_grad_allreduce).
#include "comm.h"

#include <cstring>
#include <cuda.h>
#include <set>
#include <string>

#include "common.h"
#include "stage.h"

namespace slip {
slip_status nccl_status(ncclResult_t r, const char* where) {
  if (r == ncclSuccess) return SLIP_OK;
  set_error(std::string(where) + ": " + ncclGetErrorString(r));
  return SLIP_ENCCL;
}
}  // namespace slip

using namespace slip;

namespace {

void close_fused(slip_comm* c) {
  if (c->ipc_grad_base) cudaIpcCloseMemHandle(c->ipc_grad_base);
  if (c->ipc_flag_base) cudaIpcCloseMemHandle(c->ipc_flag_base);
  if (c->ipc_recv_base) cudaIpcCloseMemHandle(c->ipc_recv_base);
  c->ipc_recv_base = nullptr;
  c->my_recv = nullptr;
  c->peer_recv = nullptr;
  c->push = false;
  if (c->flags) cudaFree(c->flags);
  c->ipc_grad_base = c->ipc_flag_base = nullptr;
  c->flags = c->peer_flags = nullptr;
  c->peer_grad = c->fused_local = nullptr;
  c->fused_ar = false;
  c->epoch = 0;
}

void destroy_setup(slip_comm* c) {
  close_fused(c);
  for (auto& kv : c->pair_comm)
    if (kv.second) ncclCommDestroy(kv.second);
  for (auto& kv : c->pair_stream)
    if (kv.second) cudaStreamDestroy(kv.second);
  c->pair_comm.clear();
  c->pair_stream.clear();
  if (c->stage_comm) ncclCommDestroy(c->stage_comm);
  c->stage_comm = nullptr;
  if (c->live_comm) ncclCommDestroy(c->live_comm);
  c->live_comm = nullptr;
  if (c->val_comm) ncclCommDestroy(c->val_comm);
  c->val_comm = nullptr;
  if (c->val_stream) cudaStreamDestroy(c->val_stream);
  c->val_stream = nullptr;
  c->val_rank.clear();
  if (c->ar_stream) cudaStreamDestroy(c->ar_stream);
  c->ar_stream = nullptr;
  c->ready = false;
}

}  // namespace

extern "C" {

slip_status slip_nccl_unique_id(uint8_t out_id[128]) {
  SLIP_CHECK(out_id, SLIP_EINVAL, "nccl_unique_id: out is NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  SLIP_NCCL(ncclGetUniqueId(&id));
  std::memcpy(out_id, &id, 128);
  return SLIP_OK;
}

slip_status slip_comm_create(slip_comm** out, int32_t rank, int32_t world, const uint8_t id[128]) {
  SLIP_CHECK(out && id && world >= 1 && rank >= 0 && rank < world, SLIP_EINVAL, "comm_create: bad arguments");
  ncclUniqueId uid;
  std::memcpy(&uid, id, 128);
  slip_comm* c = new slip_comm();
  c->rank = rank;
  c->role = rank;
  c->world = world;
  ncclResult_t r = ncclCommInitRank(&c->world_comm, world, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_status(r, "ncclCommInitRank");
  }
  *out = c;
  return SLIP_OK;
}

slip_status slip_comm_setup(slip_comm* c, const slip_cluster* cl) {
  SLIP_CHECK(c && c->world_comm, SLIP_EINVAL, "comm_setup: comm not created");
  Cluster cc;
  SLIP_TRY(read_cluster(cl, cc));
  SLIP_CHECK(cc.N * cc.DP == c->world, SLIP_EINVAL, "comm_setup: world size must equal N * DP");
  std::vector<int> ex;
  if (!assign(cc, ex)) {
    set_error("comm_setup: unrecoverable failure set");
    return SLIP_EUNRECOVERABLE;
  }
  destroy_setup(c);
  c->cl = cc;
  c->my_stage = c->role % cc.N;
  c->my_pipe = c->role / cc.N;
  c->my_live = cc.is_live(c->my_stage, c->my_pipe);
  SLIP_CUDA(cudaStreamCreateWithFlags(&c->ar_stream, cudaStreamNonBlocking));
  // stage communicator over the live peers (color = stage), failed ranks excluded
  int n_live = 0;
  for (int k = 0; k < cc.DP; ++k) n_live += cc.is_live(c->my_stage, k);
  ncclComm_t sc = nullptr;
  SLIP_NCCL(ncclCommSplit(c->world_comm, c->my_live ? c->my_stage : NCCL_SPLIT_NOCOLOR, c->my_pipe, &sc, nullptr));
  c->stage_size = c->my_live ? n_live : 0;
  if (sc && n_live <= 1) {
    ncclCommDestroy(sc);
    sc = nullptr;
  }
  c->stage_comm = sc;
  // all live ranks (post-step validation flags)
  int n_all = 0;
  for (uint8_t v : cc.live) n_all += v;
  ncclComm_t lc = nullptr;
  SLIP_NCCL(ncclCommSplit(c->world_comm, c->my_live ? 0 : NCCL_SPLIT_NOCOLOR, c->role, &lc, nullptr));
  if (lc && n_all <= 1) {
    ncclCommDestroy(lc);
    lc = nullptr;
  }
  c->live_comm = lc;
  // the same group again for the validation-flag P2P of preceding stages
  ncclComm_t vc = nullptr;
  SLIP_NCCL(ncclCommSplit(c->world_comm, c->my_live ? 0 : NCCL_SPLIT_NOCOLOR, c->role, &vc, nullptr));
  if (vc && n_all <= 1) {
    ncclCommDestroy(vc);
    vc = nullptr;
  }
  c->val_comm = vc;
  c->val_rank.assign(static_cast<size_t>(cc.N) * cc.DP, -1);
  for (int r = 0, q = 0; r < cc.N * cc.DP; ++r)  // split ranks follow the key (role) order
    if (cc.is_live(r % cc.N, r / cc.N)) c->val_rank[r] = q++;
  if (vc) SLIP_CUDA(cudaStreamCreateWithFlags(&c->val_stream, cudaStreamNonBlocking));
  // directed pairs used by the assignment (ACT i -> i+1, GRAD i+1 -> i), in a fixed order
  std::set<std::pair<int, int>> pairs;
  for (int k = 0; k < cc.DP; ++k)
    for (int j = 0; j < cc.m; ++j)
      for (int i = 0; i + 1 < cc.N; ++i) {
        const int a = rank_of(cc.N, i, ex[(static_cast<size_t>(i) * cc.m + j) * cc.DP + k]);
        const int b = rank_of(cc.N, i + 1, ex[(static_cast<size_t>(i + 1) * cc.m + j) * cc.DP + k]);
        pairs.insert({a, b});
        pairs.insert({b, a});
      }
  // Pair communicators carry one [T, h] activation / gradient at a time and their kernels
  // run concurrently with the persistent compute kernels: cap each at c->p2p_ctas CTAs
  // (SMs) so that the transfers a worker has outstanding fit in the SM reserve
  // (slip_set_sm_reserve) instead of starving the GEMM grids.
  ncclConfig_t pcfg = NCCL_CONFIG_INITIALIZER;
  if (c->p2p_ctas > 0) {
    pcfg.minCTAs = 1;
    pcfg.maxCTAs = c->p2p_ctas;
  }
  int color = 0;
  for (const auto& pr : pairs) {
    const bool member = c->role == pr.first || c->role == pr.second;
    ncclComm_t pc = nullptr;
    SLIP_NCCL(ncclCommSplit(c->world_comm, member ? color : NCCL_SPLIT_NOCOLOR, c->role == pr.first ? 0 : 1, &pc,
                            c->p2p_ctas > 0 ? &pcfg : nullptr));
    if (member) {
      c->pair_comm[pr] = pc;
      cudaStream_t st;
      SLIP_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
      c->pair_stream[pr] = st;
    }
    ++color;
  }
  c->ready = true;
  return SLIP_OK;
}

slip_status slip_comm_destroy(slip_comm* c) {
  if (!c) return SLIP_OK;
  destroy_setup(c);
  if (c->world_comm) ncclCommDestroy(c->world_comm);
  delete c;
  return SLIP_OK;
}

slip_status slip_comm_set_p2p_ctas(slip_comm* c, int32_t n) {
  SLIP_CHECK(c && n >= 0 && n <= 64, SLIP_EINVAL, "comm_set_p2p_ctas: n must be in [0, 64]");
  destroy_setup(c);
  c->p2p_ctas = n;
  return SLIP_OK;
}

slip_status slip_comm_set_role(slip_comm* c, int32_t role) {
  SLIP_CHECK(c && role >= 0 && role < c->world, SLIP_EINVAL, "comm_set_role: role out of range");
  destroy_setup(c);
  c->role = role;
  return SLIP_OK;
}

slip_status slip_migrate_state(slip_ctx* ctx, slip_comm* c, int32_t peer, int32_t send, int64_t opt_step,
                               slip_stream s) {
  SLIP_CHECK(ctx && ctx->bound && c && c->world_comm, SLIP_EINVAL, "migrate_state: ctx not bound or comm missing");
  SLIP_CHECK(peer >= 0 && peer < c->world && peer != c->rank, SLIP_EINVAL, "migrate_state: bad peer rank");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(s);
  const size_t n = static_cast<size_t>(ctx->n_params);
  // both sides first exchange their parameter counts: a receiver whose context holds a
  // different stage model (e.g. one without the sender's GPT end) fails on both sides
  // instead of leaving mismatched transfers in flight
  {
    int64_t* d_n = nullptr;
    SLIP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_n), 2 * sizeof(int64_t), st));
    const int64_t mine = ctx->n_params;
    SLIP_CUDA(cudaMemcpyAsync(d_n, &mine, sizeof(int64_t), cudaMemcpyHostToDevice, st));
    SLIP_NCCL(ncclGroupStart());
    ncclResult_t r1 = ncclSend(d_n, 1, ncclInt64, peer, c->world_comm, st);
    ncclResult_t r2 = ncclRecv(d_n + 1, 1, ncclInt64, peer, c->world_comm, st);
    SLIP_NCCL(ncclGroupEnd());
    if (r1 != ncclSuccess || r2 != ncclSuccess) return nccl_status(r1 != ncclSuccess ? r1 : r2, "migrate_state: sizes");
    int64_t theirs = -1;
    SLIP_CUDA(cudaMemcpyAsync(&theirs, d_n + 1, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SLIP_CUDA(cudaFreeAsync(d_n, st));
    SLIP_CUDA(cudaStreamSynchronize(st));
    SLIP_CHECK(theirs == mine, SLIP_EINVAL,
               ("migrate_state: the peer's stage holds " + std::to_string(theirs) + " parameters, this one " +
                std::to_string(mine) + " (bind the stage model of the role taken over first)")
                   .c_str());
  }
  float* bufs[3] = {ctx->master, ctx->adam_m, ctx->adam_v};
  // the sender's AdamW step count travels with the state, so the receiver continues
  // with the same bias correction as the peer it replicates
  int64_t* d_step = nullptr;
  SLIP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d_step), sizeof(int64_t), st));
  if (send) SLIP_CUDA(cudaMemcpyAsync(d_step, &ctx->opt_step, sizeof(int64_t), cudaMemcpyHostToDevice, st));
  SLIP_NCCL(ncclGroupStart());
  for (float* b : bufs) {
    ncclResult_t r = send ? ncclSend(b, n, ncclFloat32, peer, c->world_comm, st)
                          : ncclRecv(b, n, ncclFloat32, peer, c->world_comm, st);
    if (r != ncclSuccess) {
      ncclGroupEnd();
      return nccl_status(r, send ? "ncclSend(state)" : "ncclRecv(state)");
    }
  }
  {
    ncclResult_t r = send ? ncclSend(d_step, 1, ncclInt64, peer, c->world_comm, st)
                          : ncclRecv(d_step, 1, ncclInt64, peer, c->world_comm, st);
    if (r != ncclSuccess) {
      ncclGroupEnd();
      return nccl_status(r, "migrate_state: step count");
    }
  }
  SLIP_NCCL(ncclGroupEnd());
  int64_t sender_step = 0;
  SLIP_CUDA(cudaMemcpyAsync(&sender_step, d_step, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  SLIP_CUDA(cudaFreeAsync(d_step, st));
  SLIP_CUDA(cudaStreamSynchronize(st));
  if (!send) {
    ctx->opt_step = opt_step >= 0 ? opt_step : sender_step;
    SLIP_TRY(slip_weights_from_master(ctx, s));
  }
  return SLIP_OK;
}

namespace {
slip_status fuse_impl(slip_ctx* ctx, slip_comm* c, int32_t enable, float* recv);
}

slip_status slip_comm_fuse_ar_adam(slip_ctx* ctx, slip_comm* c, int32_t enable) {
  return fuse_impl(ctx, c, enable, nullptr);
}

slip_status slip_comm_fuse_ar_push(slip_ctx* ctx, slip_comm* c, float* recv, int32_t enable) {
  SLIP_CHECK(!enable || recv, SLIP_EINVAL, "comm_fuse_ar_push: recv is NULL");
  SLIP_CHECK(!enable || !ctx || ctx->dm.ends == 0, SLIP_EUNSUPPORTED,
             "comm_fuse_ar_push: stages with a GPT end (their embedding gradient is not written by W) use "
             "slip_comm_fuse_ar_adam");
  return fuse_impl(ctx, c, enable, enable ? recv : nullptr);
}

namespace {
slip_status fuse_impl(slip_ctx* ctx, slip_comm* c, int32_t enable, float* recv) {
  SLIP_CHECK(ctx && ctx->bound && c && c->ready, SLIP_EINVAL, "comm_fuse_ar_adam: ctx not bound or comm not set up");
  close_fused(c);
  if (!enable || !c->my_live || !c->stage_comm) return SLIP_OK;  // nothing to fuse (singleton group)
  if (c->stage_size != 2) {
    set_error("comm_fuse_ar_adam: only a stage group of 2 live peers can fuse its all-reduce");
    return SLIP_EUNSUPPORTED;
  }
  // base of the allocation holding the caller's gradient buffer (torch sub-allocates)
  using AddrRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static AddrRange range = nullptr;
  if (!range) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    SLIP_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q));
    SLIP_CHECK(q == cudaDriverEntryPointSuccess && f, SLIP_ECUDA, "comm_fuse_ar_adam: no cuMemGetAddressRange");
    range = reinterpret_cast<AddrRange>(f);
  }
  CUdeviceptr base = 0;
  size_t bytes = 0;
  SLIP_CHECK(range(&base, &bytes, reinterpret_cast<CUdeviceptr>(ctx->grad)) == CUDA_SUCCESS, SLIP_ECUDA,
             "comm_fuse_ar_adam: cuMemGetAddressRange(grad) failed");
  SLIP_CUDA(cudaMalloc(&c->flags, 256));
  SLIP_CUDA(cudaMemset(c->flags, 0, 256));
  struct Rec {
    cudaIpcMemHandle_t grad, flag, recv;
    int64_t grad_off, n_params, recv_off, has_recv;
  } mine{}, both[2];
  SLIP_CUDA(cudaIpcGetMemHandle(&mine.grad, reinterpret_cast<void*>(base)));
  SLIP_CUDA(cudaIpcGetMemHandle(&mine.flag, c->flags));
  mine.grad_off = static_cast<int64_t>(reinterpret_cast<CUdeviceptr>(ctx->grad) - base);
  mine.n_params = ctx->n_params;
  if (recv) {  // push mode: the receive buffer the peer's W launches write
    CUdeviceptr rbase = 0;
    size_t rbytes = 0;
    SLIP_CHECK(range(&rbase, &rbytes, reinterpret_cast<CUdeviceptr>(recv)) == CUDA_SUCCESS, SLIP_ECUDA,
               "comm_fuse_ar_push: cuMemGetAddressRange(recv) failed");
    SLIP_CUDA(cudaIpcGetMemHandle(&mine.recv, reinterpret_cast<void*>(rbase)));
    mine.recv_off = static_cast<int64_t>(reinterpret_cast<CUdeviceptr>(recv) - rbase);
    mine.has_recv = 1;
  }
  void* dbuf = nullptr;
  SLIP_CUDA(cudaMalloc(&dbuf, 3 * sizeof(Rec)));
  // ordered before the all-gather on the same stream (a pageable cudaMemcpy on the legacy
  // stream has no ordering with the non-blocking ar_stream)
  SLIP_CUDA(cudaMemcpyAsync(dbuf, &mine, sizeof(Rec), cudaMemcpyHostToDevice, c->ar_stream));
  ncclResult_t r = ncclAllGather(dbuf, static_cast<char*>(dbuf) + sizeof(Rec), sizeof(Rec), ncclUint8, c->stage_comm,
                                 c->ar_stream);
  cudaError_t e = r == ncclSuccess ? cudaStreamSynchronize(c->ar_stream) : cudaSuccess;
  if (e == cudaSuccess && r == ncclSuccess)
    e = cudaMemcpy(both, static_cast<char*>(dbuf) + sizeof(Rec), 2 * sizeof(Rec), cudaMemcpyDeviceToHost);
  cudaFree(dbuf);
  if (r != ncclSuccess) return nccl_status(r, "ncclAllGather(ipc handles)");
  SLIP_CUDA(e);
  int me = 0;
  SLIP_NCCL(ncclCommUserRank(c->stage_comm, &me));
  const Rec& peer = both[1 - me];
  // both peers fuse or neither: a one-sided failure would leave the other side spinning in
  // peer_barrier until its trap, so the local outcome is MIN-reduced over the pair first
  int32_t ok = peer.n_params == ctx->n_params ? 1 : 0;
  cudaError_t oe = cudaSuccess;
  if (ok) oe = cudaIpcOpenMemHandle(&c->ipc_grad_base, peer.grad, cudaIpcMemLazyEnablePeerAccess);
  if (oe != cudaSuccess) c->ipc_grad_base = nullptr;
  if (ok && oe == cudaSuccess) {
    oe = cudaIpcOpenMemHandle(&c->ipc_flag_base, peer.flag, cudaIpcMemLazyEnablePeerAccess);
    if (oe != cudaSuccess) c->ipc_flag_base = nullptr;
  }
  if (ok && recv && !peer.has_recv) ok = 0;  // push mode on one side only
  if (ok && oe == cudaSuccess && recv) {
    oe = cudaIpcOpenMemHandle(&c->ipc_recv_base, peer.recv, cudaIpcMemLazyEnablePeerAccess);
    if (oe != cudaSuccess) c->ipc_recv_base = nullptr;
  }
  if (oe != cudaSuccess) {
    ok = 0;
    cudaGetLastError();
  }
  int32_t* dok = nullptr;
  SLIP_CUDA(cudaMalloc(&dok, sizeof(int32_t)));
  SLIP_CUDA(cudaMemcpyAsync(dok, &ok, sizeof(int32_t), cudaMemcpyHostToDevice, c->ar_stream));
  r = ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, c->stage_comm, c->ar_stream);
  int32_t all_ok = 0;
  e = r == ncclSuccess ? cudaMemcpyAsync(&all_ok, dok, sizeof(int32_t), cudaMemcpyDeviceToHost, c->ar_stream)
                       : cudaSuccess;
  if (e == cudaSuccess && r == ncclSuccess) e = cudaStreamSynchronize(c->ar_stream);
  cudaFree(dok);
  if (r != ncclSuccess || e != cudaSuccess || !all_ok) {
    close_fused(c);
    if (r != ncclSuccess) return nccl_status(r, "ncclAllReduce(fuse agreement)");
    SLIP_CUDA(e);
    if (peer.n_params != ctx->n_params) {
      set_error("comm_fuse_ar_adam: peer holds a different stage size");
      return SLIP_EINVAL;
    }
    set_error(oe != cudaSuccess ? "comm_fuse_ar_adam: cudaIpcOpenMemHandle failed here"
                                : "comm_fuse_ar_adam: the peer could not map this rank's buffers");
    return SLIP_ECUDA;
  }
  c->peer_grad = reinterpret_cast<const float*>(static_cast<char*>(c->ipc_grad_base) + peer.grad_off);
  c->peer_flags = static_cast<unsigned*>(c->ipc_flag_base);
  c->fused_local = ctx->grad;
  c->fused_ar = true;
  if (recv) {
    c->my_recv = recv;
    c->peer_recv = reinterpret_cast<float*>(static_cast<char*>(c->ipc_recv_base) + peer.recv_off);
    c->push = true;
  }
  return SLIP_OK;
}
}  // namespace

slip_status slip_grad_allreduce(slip_ctx* ctx, slip_comm* c, slip_stream s) {
  SLIP_CHECK(ctx && ctx->bound && c && c->ready, SLIP_EINVAL, "grad_allreduce: ctx not bound or comm not set up");
  if (!c->my_live || !c->stage_comm) return SLIP_OK;  // failed rank or singleton group
  SLIP_NCCL(ncclAllReduce(ctx->grad, ctx->grad, static_cast<size_t>(ctx->n_params), ncclFloat32, ncclSum,
                          c->stage_comm, reinterpret_cast<cudaStream_t>(s)));
  return SLIP_OK;
}

}  // extern "C"
