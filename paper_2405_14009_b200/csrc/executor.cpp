// executor.cpp — slip_execute_schedule: runs this rank's share of the plan.
//
// The plan (planner.cpp) is computed identically on every rank.  This rank (worker
// (i, k), rank = k*N + i) walks its own ops in planned start order and enqueues:
//   F   : input  <- synth / host copy (stage 0)  or  ncclRecv on the (src -> me) pair stream
//         slip_stage_forward into a free slot; output -> slot.dy; ncclSend to the next stage
//   B   : grad   <- MSE head (last stage)        or  ncclRecv into slot.dy
//         slip_backward_input; dx (in place of slot.x) -> ncclSend to the previous stage
//   W   : slip_backward_weight (deferred weight gradients), frees the slot
//   BC  : coupled backward (B then W)
//   AR  : after the stage's last W of the iteration: slip_grad_allreduce on the AR stream
//   OPT : staggered AdamW step (§3.3); its F of the next iteration follows it
// Cross-stream dependencies are CUDA events; the host never blocks inside the loop.
// Every directed pair has its own communicator and stream, and receives are posted in
// the sender's send order (checked below), so re-routed traffic cannot deadlock.
#include <algorithm>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "comm.h"
#include "common.h"
#include "kernels.cuh"
#include "stage.h"

using namespace slip;

namespace {

struct EventPool {
  std::vector<cudaEvent_t> ev;
  size_t next = 0;
  ~EventPool() {
    for (auto e : ev) cudaEventDestroy(e);
  }
  cudaError_t get(cudaEvent_t* out) {
    if (next == ev.size()) {
      cudaEvent_t e;
      cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      if (r != cudaSuccess) return r;
      ev.push_back(e);
    }
    *out = ev[next++];
    return cudaSuccess;
  }
};

// events with timing enabled, for the per-phase breakdown of the timed run
struct TimedPool {
  std::vector<cudaEvent_t> ev;
  size_t next = 0;
  ~TimedPool() {
    for (auto e : ev) cudaEventDestroy(e);
  }
  cudaError_t get(cudaEvent_t* out) {
    if (next == ev.size()) {
      cudaEvent_t e;
      cudaError_t r = cudaEventCreate(&e);
      if (r != cudaSuccess) return r;
      ev.push_back(e);
    }
    *out = ev[next++];
    return cudaSuccess;
  }
};

struct SlotInfo {
  cudaEvent_t freed = nullptr;    // recorded on the compute stream when W released the slot
  cudaEvent_t sent_y = nullptr;   // F output (slot.dy) send completed
  cudaEvent_t sent_dx = nullptr;  // B output (slot.x) send completed
};

}  // namespace

extern "C" slip_status slip_execute_schedule(slip_ctx* ctx, slip_comm* comm, const slip_cluster* cluster,
                                             const slip_costs* costs, const slip_plan_opts* opts,
                                             const slip_adam* adam, int32_t warmup, int32_t iterations,
                                             uint64_t seed, const slip_io* io, slip_stream stream,
                                             slip_report* out) {
  SLIP_CHECK(ctx && ctx->bound, SLIP_EINVAL, "execute: ctx not bound");
  SLIP_CHECK(comm && comm->ready, SLIP_EINVAL, "execute: comm not set up (slip_comm_setup)");
  SLIP_CHECK(costs && opts && adam && out, SLIP_EINVAL, "execute: NULL argument");
  SLIP_CHECK(warmup >= 0 && iterations >= 1, SLIP_EINVAL, "execute: iterations must be >= 1");
  Cluster cl;
  SLIP_TRY(read_cluster(cluster, cl));
  SLIP_CHECK(cl.N == comm->cl.N && cl.DP == comm->cl.DP && cl.m == comm->cl.m && cl.live == comm->cl.live,
             SLIP_EINVAL, "execute: cluster differs from the one passed to slip_comm_setup");
  std::memset(out, 0, sizeof *out);
  const int N = cl.N, DP = cl.DP, m = cl.m;
  const int me_i = comm->my_stage, me_k = comm->my_pipe;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  if (!comm->my_live) return SLIP_OK;  // masked (failed) rank: idles
  const Dims& D = ctx->dm;
  const size_t Th = static_cast<size_t>(D.T) * D.h;
  const size_t bytes = Th * sizeof(bf16);
  const float grad_scale = 1.0f / static_cast<float>(DP * m);

  EventPool pool;
  cudaEvent_t t0, t1;
  SLIP_CUDA(cudaEventCreate(&t0));
  SLIP_CUDA(cudaEventCreate(&t1));
  struct EvGuard {
    cudaEvent_t a, b;
    ~EvGuard() {
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    }
  } guard{t0, t1};

  SLIP_CHECK(DP * m <= 1024, SLIP_EINVAL, "execute: DP * m must be <= 1024");
  float* d_losses = ctx->ws.losses;  // [1024] per-micro-batch losses (k*m + j)
  int64_t launches0 = ctx->launches;
  TimedPool tpool;
  std::vector<std::pair<int, size_t>> timed_marks;

  for (int phase_run = 0; phase_run < 2; ++phase_run) {
    const int H = phase_run == 0 ? warmup : iterations;
    if (H == 0) continue;
    slip_plan_opts po = *opts;
    po.horizon = H;
    Plan plan;
    SLIP_TRY(slip::plan(cl, *costs, po, plan));
    auto exec_of = [&](int i, int j, int k) { return plan.exec[(static_cast<size_t>(i) * m + j) * DP + k]; };
    // my compute ops in planned order, with the AR op of each iteration inserted after my
    // last W / BC of that iteration
    std::vector<slip_op> mine;
    for (const slip_op& o : plan.ops)
      if (o.phase != SLIP_AR && o.stage == me_i && o.exec == me_k) mine.push_back(o);
    std::vector<slip_op> seq;
    {
      std::vector<int> last_w(H, -1);
      for (size_t q = 0; q < mine.size(); ++q)
        if (mine[q].phase == SLIP_W || mine[q].phase == SLIP_BC) last_w[mine[q].iter] = static_cast<int>(q);
      for (size_t q = 0; q < mine.size(); ++q) {
        seq.push_back(mine[q]);
        for (int t = 0; t < H; ++t)
          if (last_w[t] == static_cast<int>(q)) seq.push_back({me_i, -1, -1, SLIP_AR, me_k, t, 0, 0});
      }
    }
    // verify per-pair FIFO: my receive order from each source equals its send order
    {
      std::map<std::pair<int, int>, std::vector<int64_t>> sends, recvs;
      std::vector<slip_op> byend(plan.ops.begin(), plan.ops.end());
      std::stable_sort(byend.begin(), byend.end(), [](const slip_op& a, const slip_op& b) { return a.end < b.end; });
      auto key = [&](const slip_op& o) { return (static_cast<int64_t>(o.iter) * m + o.mb) * DP + o.origin; };
      for (const slip_op& o : byend) {
        if (o.phase == SLIP_F && o.stage + 1 < N && o.stage + 1 == me_i &&
            exec_of(o.stage + 1, o.mb, o.origin) == me_k)
          sends[{rank_of(N, o.stage, o.exec), 0}].push_back(key(o));
        if ((o.phase == SLIP_B || o.phase == SLIP_BC) && o.stage == me_i + 1 &&
            exec_of(o.stage - 1, o.mb, o.origin) == me_k)
          sends[{rank_of(N, o.stage, o.exec), 1}].push_back(key(o));
      }
      for (const slip_op& o : mine) {
        if (o.phase == SLIP_F && me_i > 0)
          recvs[{rank_of(N, me_i - 1, exec_of(me_i - 1, o.mb, o.origin)), 0}].push_back(key(o));
        if ((o.phase == SLIP_B || o.phase == SLIP_BC) && me_i + 1 < N)
          recvs[{rank_of(N, me_i + 1, exec_of(me_i + 1, o.mb, o.origin)), 1}].push_back(key(o));
      }
      SLIP_CHECK(sends == recvs, SLIP_ESTATE, "execute: plan violates per-pair FIFO order");
    }

    // slot state
    std::vector<SlotInfo> slots(ctx->n_slots);
    std::vector<int> free_slots;
    for (int q = ctx->n_slots - 1; q >= 0; --q) free_slots.push_back(q);
    std::map<int64_t, int> slot_of;  // (t, j, k) -> slot
    std::vector<char> first_b(H, 1), first_w(H, 1);
    auto tjk = [&](const slip_op& o) { return (static_cast<int64_t>(o.iter) * m + o.mb) * DP + o.origin; };

    if (phase_run == 1) {
      SLIP_CUDA(cudaEventRecord(t0, cs));
      launches0 = ctx->launches;
    }
    const bool timed = phase_run == 1;
    std::vector<std::pair<int, size_t>> marks;  // (phase, index of the begin event in tpool)
    for (const slip_op& o : seq) {
      cudaEvent_t ev;
      if (timed) {
        cudaEvent_t tb;
        SLIP_CUDA(tpool.get(&tb));
        SLIP_CUDA(cudaEventRecord(tb, cs));
        marks.push_back({o.phase, tpool.next - 1});
      }
      if (o.phase == SLIP_W || o.phase == SLIP_BC) out->w_gemm_launches += timed ? 4 * ctx->L : 0;
      if (o.phase == SLIP_F) {
        SLIP_CHECK(!free_slots.empty(), SLIP_EINVAL,
                   "execute: not enough slots for the plan's in-flight micro-batches (raise n_slots)");
        const int slot = free_slots.back();
        free_slots.pop_back();
        slot_of[tjk(o)] = slot;
        SlotBufs& sb = ctx->slots[slot];
        SlotInfo& si = slots[slot];
        if (me_i == 0) {
          if (si.freed) SLIP_CUDA(cudaStreamWaitEvent(cs, si.freed, 0));
          if (si.sent_dx) SLIP_CUDA(cudaStreamWaitEvent(cs, si.sent_dx, 0));
          if (io && io->x_host) {
            SLIP_CUDA(cudaMemcpyAsync(sb.x, io->x_host[o.origin * m + o.mb], bytes, cudaMemcpyHostToDevice, cs));
          } else {
            SLIP_CUDA(synth_normal(sb.x, static_cast<int64_t>(Th), seed, o.origin, o.mb, cs));
            ctx->launches += 1;
          }
        } else {
          const int src = rank_of(N, me_i - 1, exec_of(me_i - 1, o.mb, o.origin));
          const std::pair<int, int> pr{src, comm->rank};
          cudaStream_t ps = comm->pair_stream.at(pr);
          if (si.freed) SLIP_CUDA(cudaStreamWaitEvent(ps, si.freed, 0));
          if (si.sent_dx) SLIP_CUDA(cudaStreamWaitEvent(ps, si.sent_dx, 0));
          {
            ncclResult_t r = ncclRecv(sb.x, Th, ncclBfloat16, 0, comm->pair_comm.at(pr), ps);
            if (r != ncclSuccess) return nccl_status(r, "ncclRecv act");
          }
          SLIP_CUDA(pool.get(&ev));
          SLIP_CUDA(cudaEventRecord(ev, ps));
          SLIP_CUDA(cudaStreamWaitEvent(cs, ev, 0));
        }
        if (si.sent_y) SLIP_CUDA(cudaStreamWaitEvent(cs, si.sent_y, 0));
        SLIP_TRY(slip_stage_forward(ctx, slot, sb.x, sb.dy, stream));
        if (me_i + 1 < N) {
          const int dst = rank_of(N, me_i + 1, exec_of(me_i + 1, o.mb, o.origin));
          const std::pair<int, int> pr{comm->rank, dst};
          cudaStream_t ps = comm->pair_stream.at(pr);
          SLIP_CUDA(pool.get(&ev));
          SLIP_CUDA(cudaEventRecord(ev, cs));
          SLIP_CUDA(cudaStreamWaitEvent(ps, ev, 0));
          {
            ncclResult_t r = ncclSend(sb.dy, Th, ncclBfloat16, 1, comm->pair_comm.at(pr), ps);
            if (r != ncclSuccess) return nccl_status(r, "ncclSend act");
          }
          SLIP_CUDA(pool.get(&si.sent_y));
          SLIP_CUDA(cudaEventRecord(si.sent_y, ps));
        } else {
          si.sent_y = nullptr;
        }
      } else if (o.phase == SLIP_B || o.phase == SLIP_BC) {
        const int slot = slot_of.at(tjk(o));
        SlotBufs& sb = ctx->slots[slot];
        SlotInfo& si = slots[slot];
        if (me_i + 1 == N) {
          bf16* target = ctx->ws.dy1;  // B's temporaries are free before the loss head runs
          if (io && io->target_host) {
            SLIP_CUDA(cudaMemcpyAsync(target, io->target_host[o.origin * m + o.mb], bytes, cudaMemcpyHostToDevice, cs));
          } else {
            SLIP_CUDA(synth_normal(target, static_cast<int64_t>(Th), seed + 1, o.origin, o.mb, cs));
            ctx->launches += 1;
          }
          const int li = o.origin * m + o.mb;
          SLIP_TRY(slip_loss_mse(ctx, sb.dy, target, sb.dy, d_losses + li, stream));
        } else {
          const int src = rank_of(N, me_i + 1, exec_of(me_i + 1, o.mb, o.origin));
          const std::pair<int, int> pr{src, comm->rank};
          cudaStream_t ps = comm->pair_stream.at(pr);
          if (si.sent_y) SLIP_CUDA(cudaStreamWaitEvent(ps, si.sent_y, 0));
          SLIP_CUDA(pool.get(&ev));
          SLIP_CUDA(cudaEventRecord(ev, cs));  // slot.dy no longer read by this rank's compute
          SLIP_CUDA(cudaStreamWaitEvent(ps, ev, 0));
          {
            ncclResult_t r = ncclRecv(sb.dy, Th, ncclBfloat16, 0, comm->pair_comm.at(pr), ps);
            if (r != ncclSuccess) return nccl_status(r, "ncclRecv grad");
          }
          SLIP_CUDA(pool.get(&ev));
          SLIP_CUDA(cudaEventRecord(ev, ps));
          SLIP_CUDA(cudaStreamWaitEvent(cs, ev, 0));
        }
        void* dx = me_i > 0 ? static_cast<void*>(sb.x) : nullptr;  // dx overwrites the consumed stage input
        const int acc_b = first_b[o.iter] ? 0 : 1;
        first_b[o.iter] = 0;
        if (o.phase == SLIP_BC) {
          const int acc_w = first_w[o.iter] ? 0 : 1;
          first_w[o.iter] = 0;
          SLIP_TRY(slip_backward_input(ctx, slot, sb.dy, dx, acc_b, stream));
          SLIP_TRY(slip_backward_weight(ctx, slot, acc_w, stream));
        } else {
          SLIP_TRY(slip_backward_input(ctx, slot, sb.dy, dx, acc_b, stream));
        }
        if (me_i > 0) {
          const int dst = rank_of(N, me_i - 1, exec_of(me_i - 1, o.mb, o.origin));
          const std::pair<int, int> pr{comm->rank, dst};
          cudaStream_t ps = comm->pair_stream.at(pr);
          SLIP_CUDA(pool.get(&ev));
          SLIP_CUDA(cudaEventRecord(ev, cs));
          SLIP_CUDA(cudaStreamWaitEvent(ps, ev, 0));
          {
            ncclResult_t r = ncclSend(sb.x, Th, ncclBfloat16, 1, comm->pair_comm.at(pr), ps);
            if (r != ncclSuccess) return nccl_status(r, "ncclSend grad");
          }
          SLIP_CUDA(pool.get(&si.sent_dx));
          SLIP_CUDA(cudaEventRecord(si.sent_dx, ps));
        } else {
          si.sent_dx = nullptr;
        }
        if (o.phase == SLIP_BC) {
          SLIP_CUDA(pool.get(&si.freed));
          SLIP_CUDA(cudaEventRecord(si.freed, cs));
          free_slots.push_back(slot);
          slot_of.erase(tjk(o));
        }
      } else if (o.phase == SLIP_W) {
        const int slot = slot_of.at(tjk(o));
        SlotInfo& si = slots[slot];
        const int acc_w = first_w[o.iter] ? 0 : 1;
        first_w[o.iter] = 0;
        SLIP_TRY(slip_backward_weight(ctx, slot, acc_w, stream));
        SLIP_CUDA(pool.get(&si.freed));
        SLIP_CUDA(cudaEventRecord(si.freed, cs));
        free_slots.push_back(slot);
        slot_of.erase(tjk(o));
      } else if (o.phase == SLIP_AR) {
        if (comm->stage_comm) {
          SLIP_CUDA(pool.get(&ev));
          SLIP_CUDA(cudaEventRecord(ev, cs));
          SLIP_CUDA(cudaStreamWaitEvent(comm->ar_stream, ev, 0));
          SLIP_TRY(slip_grad_allreduce(ctx, comm, reinterpret_cast<slip_stream>(comm->ar_stream)));
          SLIP_CUDA(pool.get(&ev));
          SLIP_CUDA(cudaEventRecord(ev, comm->ar_stream));
          SLIP_CUDA(cudaStreamWaitEvent(cs, ev, 0));
        }
      } else if (o.phase == SLIP_OPT) {
        ctx->opt_step += 1;
        SLIP_TRY(slip_optimizer_step(ctx, adam, ctx->opt_step, grad_scale, ctx->ws.nonfinite, stream));
      }
      if (timed) {
        cudaEvent_t te;
        SLIP_CUDA(tpool.get(&te));
        SLIP_CUDA(cudaEventRecord(te, cs));
      }
    }
    if (timed) timed_marks = marks;
    // join every side stream back into the compute stream
    for (auto& kv : comm->pair_stream) {
      cudaEvent_t e;
      SLIP_CUDA(pool.get(&e));
      SLIP_CUDA(cudaEventRecord(e, kv.second));
      SLIP_CUDA(cudaStreamWaitEvent(cs, e, 0));
    }
    {
      cudaEvent_t e;
      SLIP_CUDA(pool.get(&e));
      SLIP_CUDA(cudaEventRecord(e, comm->ar_stream));
      SLIP_CUDA(cudaStreamWaitEvent(cs, e, 0));
    }
    if (phase_run == 1) {
      SLIP_CUDA(cudaEventRecord(t1, cs));
      out->predicted_period = plan.period;
      out->n_ops = static_cast<int64_t>(seq.size()) / H;
      out->plan_hash = plan_hash(plan.ops.data(), static_cast<int64_t>(plan.ops.size()));
    }
  }
  SLIP_CUDA(cudaEventSynchronize(t1));
  float ms = 0.f;
  SLIP_CUDA(cudaEventElapsedTime(&ms, t0, t1));
  out->total_ms = ms;
  out->period_ms = ms / iterations;
  out->n_kernels = ctx->launches - launches0;
  for (const auto& mk : timed_marks) {
    float e = 0.f;
    SLIP_CUDA(cudaEventElapsedTime(&e, tpool.ev[mk.second], tpool.ev[mk.second + 1]));
    out->phase_ms[mk.first] += e;
    out->phase_ops[mk.first] += 1;
  }
  // losses of the micro-batches whose last stage ran here
  if (me_i + 1 == N) {
    std::vector<float> hl(static_cast<size_t>(DP) * m, 0.f);
    SLIP_CUDA(cudaMemcpy(hl.data(), d_losses, hl.size() * sizeof(float), cudaMemcpyDeviceToHost));
    std::vector<int> ex;
    assign(cl, ex);
    double sum = 0;
    int cnt = 0;
    for (int k = 0; k < DP; ++k)
      for (int j = 0; j < m; ++j) {
        const int li = k * m + j;
        if (ex[(static_cast<size_t>(N - 1) * m + j) * DP + k] != me_k) continue;
        sum += hl[li];
        ++cnt;
        if (io && io->loss_host) io->loss_host[li] = hl[li];
      }
    out->last_loss = cnt ? static_cast<float>(sum / cnt) : 0.f;
  }
  {
    int32_t nf = 0;
    SLIP_CUDA(cudaMemcpy(&nf, ctx->ws.nonfinite, sizeof nf, cudaMemcpyDeviceToHost));
    out->nonfinite = nf;
  }
  return SLIP_OK;
}
