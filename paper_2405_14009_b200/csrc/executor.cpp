// executor.cpp — slip_execute_schedule: interprets this rank's program (program.cpp) on
// the GPU.  Compute actions run on the caller's stream; every directed worker pair has
// its own NCCL communicator and stream (comm.cpp); the stage all-reduce has its own
// stream.  Cross-stream ordering uses CUDA events only — the host never blocks inside
// the loop — and receives are posted in the sender's order (check_fifo), so re-routed
// traffic (§3.1, ReRouteAct / ReRouteGrad line 554) cannot deadlock.
//
// Buffer protocol per slot: slot.x holds the stage input (RECV_X / LOAD_X); slot.dy holds
// the stage output that SEND_Y ships and, after it, the output gradient (RECV_DY / LOSS);
// slot.dx holds the input gradient B produces and SEND_DX ships.  Events: `freed` (W
// done) guards slot.x, `sent_y` guards slot.dy, `sent_dx` guards slot.dx.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "comm.h"
#include "common.h"
#include "kernels.cuh"
#include "program.h"
#include "stage.h"

using namespace slip;

namespace {

template <bool kTiming>
struct EventPool {
  std::vector<cudaEvent_t> ev;
  size_t next = 0;
  ~EventPool() {
    for (auto e : ev) cudaEventDestroy(e);
  }
  cudaError_t get(cudaEvent_t* out) {
    if (next == ev.size()) {
      cudaEvent_t e;
      cudaError_t r = kTiming ? cudaEventCreate(&e) : cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      if (r != cudaSuccess) return r;
      ev.push_back(e);
    }
    *out = ev[next++];
    return cudaSuccess;
  }
};

struct SlotEv {
  cudaEvent_t freed = nullptr;
  cudaEvent_t sent_y = nullptr;
  cudaEvent_t sent_dx = nullptr;
  cudaEvent_t f_done = nullptr;  // dual stream: the slot's forward finished
};

// map action kinds onto the report's phase slots
int phase_of(int kind) {
  switch (kind) {
    case SLIP_ACT_F: return SLIP_F;
    case SLIP_ACT_B: return SLIP_B;
    case SLIP_ACT_W: return SLIP_W;
    case SLIP_ACT_BC: return SLIP_BC;
    case SLIP_ACT_OPT: return SLIP_OPT;
    case SLIP_ACT_AR: return SLIP_AR;
    default: return -1;
  }
}

// last plan + rank programs per context and horizon slot (warm-up / timed)
struct ExecCache {
  bool valid = false;
  int N = 0, DP = 0, m = 0, me = -1;
  std::vector<uint8_t> live;
  slip_costs costs{};
  slip_plan_opts opts{};
  Plan plan;
  std::vector<std::vector<slip_action>> progs;
  int need = 0;
};
std::map<std::pair<const slip_ctx*, int>, ExecCache> exec_cache_;

// CUDA events of a context's calls, reused from call to call (every call ends synchronized,
// so all of them have completed): creating ~1000 events per call cost host time at the
// start of every step of the end-to-end loop, while the GPU idled
struct CallEvents {
  EventPool<false> pool;
  EventPool<true> tpool;
};
std::map<const slip_ctx*, CallEvents> call_events_;

}  // namespace

extern "C" slip_status slip_execute_schedule(slip_ctx* ctx, slip_comm* comm, const slip_cluster* cluster,
                                             const slip_costs* costs, const slip_plan_opts* opts,
                                             const slip_adam* adam, int32_t warmup, int32_t iterations,
                                             uint64_t seed, const slip_io* io, slip_stream stream,
                                             slip_report* out) {
  SLIP_CHECK(ctx && ctx->bound, SLIP_EINVAL, "execute: ctx not bound");
  SLIP_CHECK(comm && comm->ready, SLIP_EINVAL, "execute: comm not set up (slip_comm_setup)");
  // SLIP_NO_MERGE_W=1: one launch per W action (A/B measurements)
  static const bool merge_w_ = [] {
    const char* e = std::getenv("SLIP_NO_MERGE_W");
    return !(e && e[0] == '1');
  }();
  // forward actions on a second compute stream (slip_set_dual_stream; SLIP_DUAL_STREAM=1
  // sets the default), so the F of a later micro-batch fills the SMs the B / W kernels of
  // an earlier one leave idle (one-wave GEMMs, wave tails, small kernels)
  static const bool dual_env_ = [] {
    const char* e = std::getenv("SLIP_DUAL_STREAM");
    return e && e[0] == '1';
  }();
  const bool dual_ = ctx->dual_stream < 0 ? dual_env_ : ctx->dual_stream != 0;
  SLIP_CHECK(costs && opts && adam && out, SLIP_EINVAL, "execute: NULL argument");
  SLIP_CHECK(warmup >= 0 && iterations >= 1, SLIP_EINVAL, "execute: iterations must be >= 1");
  Cluster cl;
  SLIP_TRY(read_cluster(cluster, cl));
  SLIP_CHECK(cl.N == comm->cl.N && cl.DP == comm->cl.DP && cl.m == comm->cl.m && cl.live == comm->cl.live,
             SLIP_EINVAL, "execute: cluster differs from the one passed to slip_comm_setup");
  std::memset(out, 0, sizeof *out);
  const int N = cl.N, DP = cl.DP, m = cl.m;
  SLIP_CHECK(DP * m <= 1024, SLIP_EINVAL, "execute: DP * m must be <= 1024");
  const int me = comm->role, me_i = comm->my_stage, me_k = comm->my_pipe;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  if (!comm->my_live) return SLIP_OK;  // masked (failed) rank idles
  const Dims& D = ctx->dm;
  const size_t Th = static_cast<size_t>(D.T) * D.h;
  const size_t bytes = Th * sizeof(bf16);
  const float grad_scale = 1.0f / static_cast<float>(DP * m);
  float* d_losses = ctx->ws.losses;
  // DP = 2 all-reduce fused into AdamW (slip_comm_fuse_ar_adam); validated steps keep the
  // NCCL all-reduce (their rollback needs the summed gradient in place)
  const bool fused_ar = comm->fused_ar && comm->stage_comm && !ctx->validate;
  // AdamW of the 2-D weights in the epilogue of the iteration's last W (slip_set_fused_adamw):
  // only where that W's dW is already the final gradient — no all-reduce (DP = 1 or a
  // singleton group whose peer failed), no validation, no model ends
  const bool adamw_in_w = ctx->fuse_adamw && !comm->stage_comm && !ctx->validate && ctx->dm.ends == 0 &&
                          ctx->n_slots >= 2;
  SLIP_CHECK(!fused_ar || comm->fused_local == ctx->grad, SLIP_ESTATE,
             "execute: gradient buffer re-bound since slip_comm_fuse_ar_adam");

  // push mode (slip_comm_fuse_ar_push): this call's W launches also write the 2-D weight
  // gradients into the peer's receive buffer (the W tables carry that mirror)
  if (fused_ar && comm->push && ctx->w_mirror != comm->peer_recv) SLIP_TRY(slip::encode_w_tables(ctx, comm->peer_recv));
  struct MirrorOn {
    slip_ctx* c;
    ~MirrorOn() { c->w_mirror_on = false; }
  } mirror_guard{ctx};
  ctx->w_mirror_on = fused_ar && comm->push;
  CallEvents& ce = call_events_[ctx];
  EventPool<false>& pool = ce.pool;
  EventPool<true>& tpool = ce.tpool;
  pool.next = 0;
  tpool.next = 0;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  SLIP_CUDA(tpool.get(&t0));
  SLIP_CUDA(tpool.get(&t1));
  std::vector<std::pair<int, size_t>> marks;  // (phase, index of the begin event in tpool)
  std::vector<std::pair<size_t, int>> mark_extra;  // (mark, extra ops it covers): merged W's
  int w_extra = 0;
  std::vector<std::pair<slip_trace_rec, size_t>> tmarks;  // trace records, begin event index
  const bool tracing = ctx->trace_on;
  int64_t launches0 = ctx->launches;

  if (ctx->validate) SLIP_CUDA(cudaMemsetAsync(ctx->ws.vflags + 4, 0, 2 * sizeof(int32_t), cs));
  // host inputs (slip_io): copied on their own stream as soon as the slot is free, so the
  // copies of later micro-batches overlap the compute of earlier ones
  if (io && !ctx->h2d) SLIP_CUDA(cudaStreamCreateWithFlags(&ctx->h2d, cudaStreamNonBlocking));
  cudaStream_t hs = ctx->h2d;
  // (not in validated mode: a rollback rewrites the weights the forward of the next
  // iteration may be reading on the other stream)
  const bool dual = dual_ && !ctx->validate;
  // the backward-side actions then run on a high-priority stream of the context (the block
  // scheduler places their CTAs first: the backward chain is the pipeline's critical path),
  // the forward ones on a low-priority one; the caller's stream brackets both
  cudaStream_t cs_call = cs;
  if (dual) {
    if (!ctx->fwd || !ctx->bwd) {
      int least = 0, greatest = 0;
      SLIP_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
      if (!ctx->fwd) SLIP_CUDA(cudaStreamCreateWithPriority(&ctx->fwd, cudaStreamNonBlocking, least));
      if (!ctx->bwd) SLIP_CUDA(cudaStreamCreateWithPriority(&ctx->bwd, cudaStreamNonBlocking, greatest));
    }
    cudaEvent_t e;
    SLIP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    SLIP_CUDA(cudaEventRecord(e, cs_call));
    SLIP_CUDA(cudaStreamWaitEvent(ctx->bwd, e, 0));
    SLIP_CUDA(cudaEventDestroy(e));
    cs = ctx->bwd;
    stream = reinterpret_cast<slip_stream>(cs);
  }
  cudaStream_t fs = dual ? ctx->fwd : cs;  // stream of the forward actions
  for (int run = 0; run < 2; ++run) {
    const int H = run == 0 ? warmup : iterations;
    if (H == 0) continue;
    const bool timed = run == 1;
    slip_plan_opts po = *opts;
    po.horizon = H;
    // The plan and the rank programs depend only on (cluster, costs, options, horizon):
    // a repeated call (one call per step in e2e use) reuses them instead of re-planning
    // on the host while the GPU idles (~1 ms per rank program at N = 8).
    ExecCache& ec = exec_cache_[{ctx, run}];
    const bool hit = ec.valid && ec.N == cl.N && ec.DP == cl.DP && ec.m == cl.m && ec.live == cl.live &&
                     ec.me == me && std::memcmp(&ec.costs, costs, sizeof(slip_costs)) == 0 &&
                     std::memcmp(&ec.opts, &po, sizeof(slip_plan_opts)) == 0;
    if (!hit) {
      ec.valid = false;
      ec.plan = Plan();
      SLIP_TRY(slip::plan(cl, *costs, po, ec.plan));
      // programs of every rank (cheap): mine to run, all of them to check pair FIFO order
      ec.progs.assign(N * DP, {});
      ec.need = 0;
      for (int r = 0; r < N * DP; ++r) {
        int ns = 0;
        SLIP_TRY(build_program(cl, ec.plan, H, r, ec.progs[r], ns));
        if (r == me) ec.need = ns;
      }
      SLIP_CHECK(check_fifo(cl, ec.progs, me), SLIP_ESTATE, "execute: plan violates per-pair FIFO order");
      ec.N = cl.N;
      ec.DP = cl.DP;
      ec.m = cl.m;
      ec.live = cl.live;
      ec.me = me;
      ec.costs = *costs;
      ec.opts = po;
      ec.valid = true;
    }
    const Plan& plan = ec.plan;
    const std::vector<std::vector<slip_action>>& progs = ec.progs;
    const int need = ec.need;
    SLIP_CHECK(need <= ctx->n_slots, SLIP_EINVAL,
               ("execute: the plan needs " + std::to_string(need) + " slots, ctx has " +
                std::to_string(ctx->n_slots))
                   .c_str());
    std::vector<SlotEv> sev(ctx->n_slots);
    cudaEvent_t opt_done = nullptr;  // dual stream: the last OPT (the weights F reads)
    if (timed) {
      SLIP_CUDA(cudaEventRecord(t0, cs));
      launches0 = ctx->launches;
    }
    if (fs != cs) {  // the forward stream starts with the compute stream
      cudaEvent_t e;
      SLIP_CUDA(pool.get(&e));
      SLIP_CUDA(cudaEventRecord(e, cs));
      SLIP_CUDA(cudaStreamWaitEvent(fs, e, 0));
    }
    auto xfer_stream = [&](int src, int dst) { return comm->pair_stream.at({src, dst}); };
    auto xfer_comm = [&](int src, int dst) { return comm->pair_comm.at({src, dst}); };
    auto chain = [&](cudaStream_t from, cudaStream_t to) -> cudaError_t {
      cudaEvent_t e;
      cudaError_t r = pool.get(&e);
      if (r != cudaSuccess) return r;
      r = cudaEventRecord(e, from);
      if (r != cudaSuccess) return r;
      return cudaStreamWaitEvent(to, e, 0);
    };
    // validated mode: the rollback check of iteration t runs before this worker's first W / BC
    // of a later iteration (the last moment t's gradients are intact) or at the end
    struct Pending {
      int iter = -1;
      int64_t step = 0;
      cudaEvent_t flag_ready = nullptr;
    } pend;
    auto flush_rollback = [&](int before_iter) -> slip_status {
      if (pend.iter < 0 || pend.iter >= before_iter) return SLIP_OK;
      SLIP_CUDA(cudaStreamWaitEvent(cs, pend.flag_ready, 0));
      int32_t* vf = ctx->ws.vflags;
      SLIP_TRY(rollback_if(ctx, adam, pend.step, grad_scale, vf + 2 + (pend.iter & 1), vf + (pend.iter & 1), vf + 4,
                           cs));
      pend.iter = -1;
      return SLIP_OK;
    };
    // validated mode: the stages whose OPT the plan finishes before this stage's OPT starts
    // ("preceding stages") send their validation flag point to point
    // (designated sender: the lowest live pipeline of the stage); this stage steps only if
    // its own validation and theirs pass, the later stages' failures are rolled back
    const bool val_p2p = ctx->validate && comm->val_comm;
    std::vector<std::vector<std::vector<int>>> pre;  // [iter][stage] -> preceding stages
    auto sender_of = [&](int j) {
      for (int k = 0; k < DP; ++k)
        if (cl.is_live(j, k)) return rank_of(N, j, k);
      return -1;
    };
    if (val_p2p) {
      pre.assign(H, std::vector<std::vector<int>>(N));
      std::vector<int64_t> s0(static_cast<size_t>(H) * N, INT64_MAX), e1(static_cast<size_t>(H) * N, INT64_MIN);
      for (const slip_op& o : plan.ops)
        if (o.phase == SLIP_OPT && o.iter < H) {
          int64_t& a0 = s0[static_cast<size_t>(o.iter) * N + o.stage];
          int64_t& a1 = e1[static_cast<size_t>(o.iter) * N + o.stage];
          a0 = std::min(a0, o.start);
          a1 = std::max(a1, o.end);
        }
      for (int t = 0; t < H; ++t)
        for (int i = 0; i < N; ++i)
          for (int j = 0; j < N; ++j)
            if (j != i && e1[static_cast<size_t>(t) * N + j] != INT64_MIN &&
                s0[static_cast<size_t>(t) * N + i] != INT64_MAX &&
                e1[static_cast<size_t>(t) * N + j] <= s0[static_cast<size_t>(t) * N + i])
              pre[t][i].push_back(j);
    }
    int send_pos = kValSend, recv_pos = kValRecv;
    int w_adamw_iter = -1;  // iteration whose 2-D weights the last W's epilogue stepped
    const std::vector<slip_action>& prog = progs[me];
    size_t skip_to = 0;  // W actions already run by a merged W launch
    for (size_t ai = 0; ai < prog.size(); ++ai) {
      if (ai < skip_to) continue;
      const slip_action& a = prog[ai];
      const int ph = phase_of(a.kind);
      if (ctx->validate && (a.kind == SLIP_ACT_W || a.kind == SLIP_ACT_BC)) SLIP_TRY(flush_rollback(a.iter));
      // tracing: begin / end events on the stream the action runs on
      cudaStream_t ts = cs;
      if (a.kind == SLIP_ACT_RECV_X || a.kind == SLIP_ACT_RECV_DY) ts = xfer_stream(a.peer, me);
      if (a.kind == SLIP_ACT_SEND_Y || a.kind == SLIP_ACT_SEND_DX) ts = xfer_stream(me, a.peer);
      if (a.kind == SLIP_ACT_AR) ts = comm->ar_stream;
      if (io && io->x_host && a.kind == SLIP_ACT_LOAD_X) ts = hs;
      else if (a.kind == SLIP_ACT_LOAD_X || a.kind == SLIP_ACT_F) ts = fs;
      const bool tr = timed && tracing && !(a.kind == SLIP_ACT_AR && !comm->stage_comm);
      size_t tb_idx = 0;
      // called by every action after its stream waits: the phase timing (and the trace)
      // measure the operation itself, not the time it waited for a peer or a free slot
      bool marked = false, mark_done = false;
      auto trace_begin = [&]() -> cudaError_t {
        cudaError_t r = cudaSuccess;
        if (timed && ph >= 0) {
          marked = true;
          cudaEvent_t tb, te;
          r = tpool.get(&tb);
          if (r == cudaSuccess) r = tpool.get(&te);
          if (r == cudaSuccess) r = cudaEventRecord(tb, ts);
          marks.push_back({ph, tpool.next - 2});
        }
        if (!tr || r != cudaSuccess) return r;
        cudaEvent_t e0, e1;
        r = tpool.get(&e0);
        if (r == cudaSuccess) r = tpool.get(&e1);
        if (r == cudaSuccess) r = cudaEventRecord(e0, ts);
        tb_idx = tpool.next - 2;
        return r;
      };
      SlotBufs* sb = a.slot >= 0 ? &ctx->slots[a.slot] : nullptr;
      SlotEv* se = a.slot >= 0 ? &sev[a.slot] : nullptr;
      switch (a.kind) {
        case SLIP_ACT_LOAD_X: {
          if (io && io->x_host) {  // H2D on the copy stream once the slot is free, then join
            if (se->freed) SLIP_CUDA(cudaStreamWaitEvent(hs, se->freed, 0));
            SLIP_CUDA(trace_begin());
            if (ctx->dm.ends & 1)  // the stage input is T token ids (embedding end)
              SLIP_CUDA(cudaMemcpyAsync(sb->end.tokens, io->x_host[a.origin * m + a.mb], D.T * sizeof(int32_t),
                                        cudaMemcpyHostToDevice, hs));
            else
              SLIP_CUDA(cudaMemcpyAsync(sb->x, io->x_host[a.origin * m + a.mb], bytes, cudaMemcpyHostToDevice, hs));
            SLIP_CUDA(chain(hs, fs));
            break;
          }
          if (se->freed) SLIP_CUDA(cudaStreamWaitEvent(fs, se->freed, 0));
          SLIP_CUDA(trace_begin());
          if (ctx->dm.ends & 1) {  // the stage input is T token ids (embedding end)
            SLIP_CUDA(synth_tokens(sb->end.tokens, D.T, D.V, seed, a.origin, a.mb, fs));
            ctx->launches += 1;
          } else {
            SLIP_CUDA(synth_normal(sb->x, static_cast<int64_t>(Th), seed, a.origin, a.mb, fs));
            ctx->launches += 1;
          }
          break;
        }
        case SLIP_ACT_RECV_X: {
          cudaStream_t ps = xfer_stream(a.peer, me);
          if (se->freed) SLIP_CUDA(cudaStreamWaitEvent(ps, se->freed, 0));
          SLIP_CUDA(trace_begin());
          ncclResult_t r = ncclRecv(sb->x, Th, ncclBfloat16, 0, xfer_comm(a.peer, me), ps);
          if (r != ncclSuccess) return nccl_status(r, "ncclRecv activation");
          SLIP_CUDA(chain(ps, fs));
          break;
        }
        case SLIP_ACT_F:
          if (se->sent_y) SLIP_CUDA(cudaStreamWaitEvent(fs, se->sent_y, 0));
          if (dual) {  // the slot's stash is free (W done) and the weights are this iteration's
            if (se->freed) SLIP_CUDA(cudaStreamWaitEvent(fs, se->freed, 0));
            if (opt_done) SLIP_CUDA(cudaStreamWaitEvent(fs, opt_done, 0));
          }
          SLIP_CUDA(trace_begin());
          SLIP_TRY(slip_stage_forward(ctx, a.slot, (ctx->dm.ends & 1) ? static_cast<void*>(sb->end.tokens) : sb->x,
                                      sb->dy, reinterpret_cast<slip_stream>(fs)));
          if (dual) {  // B / LOSS of this slot (on cs) read the F-stash and the output
            SLIP_CUDA(pool.get(&se->f_done));
            SLIP_CUDA(cudaEventRecord(se->f_done, fs));
          }
          break;
        case SLIP_ACT_SEND_Y: {
          cudaStream_t ps = xfer_stream(me, a.peer);
          SLIP_CUDA(chain(fs, ps));
          SLIP_CUDA(trace_begin());
          ncclResult_t r = ncclSend(sb->dy, Th, ncclBfloat16, 1, xfer_comm(me, a.peer), ps);
          if (r != ncclSuccess) return nccl_status(r, "ncclSend activation");
          SLIP_CUDA(pool.get(&se->sent_y));
          SLIP_CUDA(cudaEventRecord(se->sent_y, ps));
          break;
        }
        case SLIP_ACT_LOSS: {
          bf16* target = ctx->ws.dy1;  // B's temporaries are free before the head runs
          if (dual && se->f_done) SLIP_CUDA(cudaStreamWaitEvent(cs, se->f_done, 0));
          SLIP_CUDA(trace_begin());
          if (ctx->dm.ends & 2) {  // LM head + cross-entropy on T int32 labels
            int32_t* labels = reinterpret_cast<int32_t*>(target);
            if (io && io->target_host) {
              SLIP_CUDA(cudaMemcpyAsync(labels, io->target_host[a.origin * m + a.mb], D.T * sizeof(int32_t),
                                        cudaMemcpyHostToDevice, cs));
            } else {
              SLIP_CUDA(synth_tokens(labels, D.T, D.V, seed + 1, a.origin, a.mb, cs));
              ctx->launches += 1;
            }
            SLIP_TRY(slip_loss_ce(ctx, a.slot, sb->dy, labels, sb->dy, d_losses + a.origin * m + a.mb, a.accumulate & 1,
                                  stream));
            break;
          }
          if (io && io->target_host) {
            // the target goes to slot.dx (free until this micro-batch's B writes its input
            // gradient there, after the head), copied on the copy stream ahead of time
            target = sb->dx;
            if (se->freed) SLIP_CUDA(cudaStreamWaitEvent(hs, se->freed, 0));
            if (se->sent_dx) SLIP_CUDA(cudaStreamWaitEvent(hs, se->sent_dx, 0));
            SLIP_CUDA(
                cudaMemcpyAsync(target, io->target_host[a.origin * m + a.mb], bytes, cudaMemcpyHostToDevice, hs));
            SLIP_CUDA(chain(hs, cs));
          } else {
            SLIP_CUDA(synth_normal(target, static_cast<int64_t>(Th), seed + 1, a.origin, a.mb, cs));
            ctx->launches += 1;
          }
          SLIP_TRY(slip_loss_mse(ctx, sb->dy, target, sb->dy, d_losses + a.origin * m + a.mb, stream));
          break;
        }
        case SLIP_ACT_RECV_DY: {
          cudaStream_t ps = xfer_stream(a.peer, me);
          if (se->sent_y) SLIP_CUDA(cudaStreamWaitEvent(ps, se->sent_y, 0));
          SLIP_CUDA(chain(cs, ps));  // slot.dy is no longer read by compute (F done)
          SLIP_CUDA(trace_begin());
          ncclResult_t r = ncclRecv(sb->dy, Th, ncclBfloat16, 0, xfer_comm(a.peer, me), ps);
          if (r != ncclSuccess) return nccl_status(r, "ncclRecv gradient");
          SLIP_CUDA(chain(ps, cs));
          break;
        }
        case SLIP_ACT_B:
        case SLIP_ACT_BC: {
          // slot.dx is the send buffer of the input gradient: the previous occupant's send must be done
          if (se->sent_dx) SLIP_CUDA(cudaStreamWaitEvent(cs, se->sent_dx, 0));
          if (dual && se->f_done) SLIP_CUDA(cudaStreamWaitEvent(cs, se->f_done, 0));
          SLIP_CUDA(trace_begin());
          void* dx = me_i > 0 ? static_cast<void*>(sb->dx) : nullptr;
          SLIP_TRY(slip_backward_input(ctx, a.slot, sb->dy, dx, a.accumulate & 1, stream));
          if (a.kind == SLIP_ACT_BC) {
            SLIP_TRY(slip_backward_weight(ctx, a.slot, (a.accumulate >> 1) & 1, stream));
            SLIP_CUDA(pool.get(&se->freed));
            SLIP_CUDA(cudaEventRecord(se->freed, cs));
            if (timed) out->w_gemm_launches += 1;  // one grouped launch of all 4L products
          }
          break;
        }
        case SLIP_ACT_SEND_DX: {
          cudaStream_t ps = xfer_stream(me, a.peer);
          SLIP_CUDA(chain(cs, ps));
          SLIP_CUDA(trace_begin());
          ncclResult_t r = ncclSend(sb->dx, Th, ncclBfloat16, 1, xfer_comm(me, a.peer), ps);
          if (r != ncclSuccess) return nccl_status(r, "ncclSend gradient");
          SLIP_CUDA(pool.get(&se->sent_dx));
          SLIP_CUDA(cudaEventRecord(se->sent_dx, ps));
          break;
        }
        case SLIP_ACT_W: {
          // W actions the program puts back to back (same iteration; e.g. the deferred W's of
          // the cool-down) run as ONE grouped launch over their slots (K = n T): each dW is
          // accumulated in TMEM and written once instead of read-modified-written per W
          size_t run = 1;
          if (merge_w_ && !ctx->validate && ctx->n_slots >= 2)
            while (ai + run < prog.size() && run < 8 && prog[ai + run].kind == SLIP_ACT_W &&
                   prog[ai + run].iter == a.iter)
              ++run;
          SLIP_CUDA(trace_begin());
          const bool last_w = ai + run < prog.size() && prog[ai + run].kind == SLIP_ACT_AR && prog[ai + run].iter == a.iter;
          if (adamw_in_w && last_w) {  // dW straight into AdamW (step = the coming OPT's)
            int slots[8];
            for (size_t j = 0; j < run; ++j) slots[j] = prog[ai + j].slot;
            const AdamEpi ad = adam_epilogue_args(ctx, adam, ctx->opt_step + 1, grad_scale);
            SLIP_TRY(weight_multi(ctx, slots, static_cast<int>(run), a.accumulate, cs, &ad));
            w_adamw_iter = a.iter;
          } else if (run == 1) {
            SLIP_TRY(slip_backward_weight(ctx, a.slot, a.accumulate, stream));
          } else {
            int slots[8];
            for (size_t j = 0; j < run; ++j) slots[j] = prog[ai + j].slot;
            SLIP_TRY(weight_multi(ctx, slots, static_cast<int>(run), a.accumulate, cs));
          }
          for (size_t j = 0; j < run; ++j) {
            SlotEv& sj = sev[prog[ai + j].slot];
            SLIP_CUDA(pool.get(&sj.freed));
            SLIP_CUDA(cudaEventRecord(sj.freed, cs));
          }
          if (timed) {
            out->w_gemm_launches += 1;  // one grouped launch of all 4L products (of `run` slots)
            w_extra = static_cast<int>(run) - 1;  // the phase mark stands for `run` W's
          }
          skip_to = ai + run;
          break;
        }
        case SLIP_ACT_AR:
          if (comm->stage_comm && !fused_ar) {
            SLIP_CUDA(chain(cs, comm->ar_stream));
            SLIP_CUDA(trace_begin());
            SLIP_TRY(slip_grad_allreduce(ctx, comm, reinterpret_cast<slip_stream>(comm->ar_stream)));
            SLIP_CUDA(chain(comm->ar_stream, cs));
          }
          break;
        case SLIP_ACT_OPT:
          ctx->opt_step += 1;
          // the stage all-reduce fused into AdamW over NVLink (DP = 2): both peers' W are
          // done before either reads (this barrier's wait for the peer stays outside the
          // OPT phase mark, as the NCCL all-reduce's does), and neither overwrites its
          // gradient (next iteration's first W) before the other has read it
          if (fused_ar) SLIP_CUDA(peer_barrier(comm->peer_flags, comm->flags, ++comm->epoch, cs));
          SLIP_CUDA(trace_begin());
          if (fused_ar) {
            SLIP_TRY(slip::optimizer_step_peer(ctx, adam, ctx->opt_step, grad_scale, ctx->ws.nonfinite, stream,
                                               comm->peer_grad, comm->push ? comm->my_recv : nullptr));
            // the OPT phase (a planner cost) ends with AdamW; the wait for the peer's AdamW
            // below is peer skew, not optimizer time
            if (marked) {
              SLIP_CUDA(cudaEventRecord(tpool.ev[marks.back().second + 1], ts));
              mark_done = true;
            }
            SLIP_CUDA(peer_barrier(comm->peer_flags, comm->flags, ++comm->epoch, cs));
          } else if (!ctx->validate && w_adamw_iter == a.iter) {  // the 2-D weights stepped in W
            SLIP_TRY(optimizer_step_vectors(ctx, adam, ctx->opt_step, grad_scale, ctx->ws.nonfinite, cs));
          } else if (!ctx->validate) {
            SLIP_TRY(slip_optimizer_step(ctx, adam, ctx->opt_step, grad_scale, ctx->ws.nonfinite, stream));
          } else {
            // local validation, step only if finite (no wait for other stages), then the
            // live-rank MAX of the flag on the all-reduce stream
            int32_t* own = ctx->ws.vflags + (a.iter & 1);
            int32_t* glob = ctx->ws.vflags + 2 + (a.iter & 1);
            int n_pre = 0;
            int32_t* pre_buf = nullptr;
            if (val_p2p && !pre[a.iter][me_i].empty()) {
              const std::vector<int>& P = pre[a.iter][me_i];
              n_pre = static_cast<int>(P.size());
              if (recv_pos + n_pre > kVflags) {  // ring wrap: the earlier readers (cs) first
                recv_pos = kValRecv;
                SLIP_CUDA(chain(cs, comm->val_stream));
              }
              pre_buf = ctx->ws.vflags + recv_pos;
              recv_pos += n_pre;
              SLIP_NCCL(ncclGroupStart());
              for (int q = 0; q < n_pre; ++q) {
                ncclResult_t r = ncclRecv(pre_buf + q, 1, ncclInt32, comm->val_rank[sender_of(P[q])], comm->val_comm,
                                          comm->val_stream);
                if (r != ncclSuccess) {
                  ncclGroupEnd();
                  return nccl_status(r, "ncclRecv(validation flag)");
                }
              }
              SLIP_NCCL(ncclGroupEnd());
              SLIP_CUDA(chain(comm->val_stream, cs));
            }
            SLIP_TRY(validated_step(ctx, adam, ctx->opt_step, grad_scale, own, ctx->fault_next_opt, cs, pre_buf,
                                    n_pre));
            ctx->fault_next_opt = 0;
            if (val_p2p && sender_of(me_i) == me) {  // my stage's flag to the stages it precedes
              std::vector<int> dst;
              for (int i = 0; i < N; ++i) {
                const std::vector<int>& P = pre[a.iter][i];
                if (i != me_i && std::find(P.begin(), P.end(), me_i) != P.end())
                  for (int k = 0; k < DP; ++k)
                    if (cl.is_live(i, k)) dst.push_back(rank_of(N, i, k));
              }
              if (!dst.empty()) {
                if (send_pos + 1 > kValRecv) {  // ring wrap: the earlier sends first
                  send_pos = kValSend;
                  SLIP_CUDA(chain(comm->val_stream, cs));
                }
                int32_t* sb = ctx->ws.vflags + send_pos++;
                SLIP_CUDA(cudaMemcpyAsync(sb, own, sizeof(int32_t), cudaMemcpyDeviceToDevice, cs));
                SLIP_CUDA(chain(cs, comm->val_stream));
                SLIP_NCCL(ncclGroupStart());
                for (int r : dst) {
                  ncclResult_t e = ncclSend(sb, 1, ncclInt32, comm->val_rank[r], comm->val_comm, comm->val_stream);
                  if (e != ncclSuccess) {
                    ncclGroupEnd();
                    return nccl_status(e, "ncclSend(validation flag)");
                  }
                }
                SLIP_NCCL(ncclGroupEnd());
              }
            }
            cudaEvent_t fe;
            if (comm->live_comm) {
              SLIP_CUDA(chain(cs, comm->ar_stream));
              ncclResult_t r = ncclAllReduce(own, glob, 1, ncclInt32, ncclMax, comm->live_comm, comm->ar_stream);
              if (r != ncclSuccess) return nccl_status(r, "ncclAllReduce(validation flag)");
              SLIP_CUDA(pool.get(&fe));
              SLIP_CUDA(cudaEventRecord(fe, comm->ar_stream));
            } else {
              SLIP_CUDA(cudaMemcpyAsync(glob, own, sizeof(int32_t), cudaMemcpyDeviceToDevice, cs));
              SLIP_CUDA(pool.get(&fe));
              SLIP_CUDA(cudaEventRecord(fe, cs));
            }
            pend.iter = a.iter;
            pend.step = ctx->opt_step;
            pend.flag_ready = fe;
          }
          if (dual) {
            SLIP_CUDA(pool.get(&opt_done));
            SLIP_CUDA(cudaEventRecord(opt_done, cs));
          }
          break;
        default:
          set_error("execute: unknown action");
          return SLIP_EINVAL;
      }
      if (marked && !mark_done) SLIP_CUDA(cudaEventRecord(tpool.ev[marks.back().second + 1], ts));
      if (marked && w_extra > 0) mark_extra.push_back({marks.size() - 1, w_extra});
      w_extra = 0;
      if (tr) {
        SLIP_CUDA(cudaEventRecord(tpool.ev[tb_idx + 1], ts));
        slip_trace_rec rec{a.kind, a.mb, a.origin, a.iter, a.peer, a.slot, 0.f, 0.f};
        tmarks.push_back({rec, tb_idx});
      }
    }
    if (ctx->validate) SLIP_TRY(flush_rollback(1 << 30));
    // join every side stream back into the compute stream
    if (fs != cs) SLIP_CUDA(chain(fs, cs));
    for (auto& kv : comm->pair_stream) SLIP_CUDA(chain(kv.second, cs));
    SLIP_CUDA(chain(comm->ar_stream, cs));
    if (comm->val_stream) SLIP_CUDA(chain(comm->val_stream, cs));
    if (hs) SLIP_CUDA(chain(hs, cs));
    if (timed) {
      SLIP_CUDA(cudaEventRecord(t1, cs));
      out->predicted_period = plan.period;
      out->n_ops = static_cast<int64_t>(progs[me].size());
      out->plan_hash = plan_hash(plan.ops.data(), static_cast<int64_t>(plan.ops.size()));
    }
  }
  if (cs != cs_call) {  // the caller's stream resumes after the backward-side stream
    cudaEvent_t e;
    SLIP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    SLIP_CUDA(cudaEventRecord(e, cs));
    SLIP_CUDA(cudaStreamWaitEvent(cs_call, e, 0));
    SLIP_CUDA(cudaEventDestroy(e));
  }
  SLIP_CUDA(cudaEventSynchronize(t1));
  float ms = 0.f;
  SLIP_CUDA(cudaEventElapsedTime(&ms, t0, t1));
  out->total_ms = ms;
  out->period_ms = ms / iterations;
  out->n_kernels = ctx->launches - launches0;
  if (tracing) {
    ctx->trace.clear();
    for (auto& tm : tmarks) {
      SLIP_CUDA(cudaEventElapsedTime(&tm.first.begin_ms, t0, tpool.ev[tm.second]));
      SLIP_CUDA(cudaEventElapsedTime(&tm.first.end_ms, t0, tpool.ev[tm.second + 1]));
      ctx->trace.push_back(tm.first);
    }
  }
  for (const auto& me : mark_extra) out->phase_ops[marks[me.first].first] += me.second;
  for (const auto& mk : marks) {
    float e = 0.f;
    SLIP_CUDA(cudaEventElapsedTime(&e, tpool.ev[mk.second], tpool.ev[mk.second + 1]));
    out->phase_ms[mk.first] += e;
    out->phase_ops[mk.first] += 1;
  }
  if (me_i + 1 == N) {  // losses of the micro-batches whose last stage ran here
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
  int32_t nf = 0;
  SLIP_CUDA(cudaMemcpy(&nf, ctx->ws.nonfinite, sizeof nf, cudaMemcpyDeviceToHost));
  out->nonfinite = nf;
  if (ctx->validate) {
    int32_t rs[2] = {0, 0};  // rollbacks, skipped steps
    SLIP_CUDA(cudaMemcpy(rs, ctx->ws.vflags + 4, sizeof rs, cudaMemcpyDeviceToHost));
    out->rollbacks = rs[0];
    out->skipped = rs[1];
    // a rolled-back or skipped step does not count towards AdamW's bias correction next call
    ctx->opt_step -= rs[0] + rs[1];
  }
  return SLIP_OK;
}

namespace slip {
// the executor's per-context caches (plans, rank programs, events), dropped with the context
void executor_forget(const slip_ctx* ctx) {
  call_events_.erase(ctx);
  for (int run = 0; run < 2; ++run) exec_cache_.erase({ctx, run});
}
}  // namespace slip

extern "C" slip_status slip_set_dual_stream(slip_ctx* ctx, int32_t enable) {
  SLIP_CHECK(ctx, SLIP_EINVAL, "set_dual_stream: ctx is NULL");
  ctx->dual_stream = enable != 0 ? 1 : 0;
  return SLIP_OK;
}

extern "C" slip_status slip_set_trace(slip_ctx* ctx, int32_t enable) {
  SLIP_CHECK(ctx, SLIP_EINVAL, "set_trace: ctx is NULL");
  ctx->trace_on = enable != 0;  // the last traced run's records stay readable
  return SLIP_OK;
}

extern "C" slip_status slip_get_trace(slip_ctx* ctx, slip_trace_rec* out, int64_t cap, int64_t* n) {
  SLIP_CHECK(ctx && n, SLIP_EINVAL, "get_trace: NULL argument");
  *n = static_cast<int64_t>(ctx->trace.size());
  if (out && cap > 0) std::copy(ctx->trace.begin(), ctx->trace.begin() + std::min<int64_t>(cap, *n), out);
  return SLIP_OK;
}
