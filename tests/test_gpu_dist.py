"""Multi-GPU executor checks (skipped unless >= 2 GPUs): launches
tests/dist_check.py under torchrun (127.0.0.1 rendezvous)."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _run(n, dp, pp, *extra):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + n + pp + 7 * len(extra)),
           os.path.join(HERE, "dist_check.py"), "--dp", str(dp), "--pp", str(pp), *extra]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
    return r.stdout


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_dp2_pp1_reroute():
    out = _run(2, 2, 1)
    assert '"ok": true' in out


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_dp1_pp2_pipeline():
    out = _run(2, 1, 2)
    assert '"ok": true' in out


@pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs 4 GPUs")
def test_dp2_pp2_reroute():
    out = _run(4, 2, 2)
    assert '"ok": true' in out


@pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs 4 GPUs")
def test_dp2_pp2_normalization_swap():
    """A failure at stage 0 migrated to the last stage by a P2P state copy; the GPU
    that takes over the role continues training identically (dist_check --migrate)."""
    out = _run(4, 2, 2, "--migrate")
    assert '"scenario": "migrate", "ok": true' in out


@pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs 4 GPUs")
def test_dp2_pp2_validation_rollback():
    """Stage 0 fails validation in iteration 2: it skips its step, stage 1 (which
    stepped on its own validation) rolls back (dist_check --validate)."""
    out = _run(4, 2, 2, "--validate")
    assert '"scenario": "validate"' in out and '"ok": false' not in out


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_dp1_pp2_validation_preceding_stage():
    """DP1 x PP2 on 2 GPUs: a fault at the stage that steps first is seen by the later
    stage through the point-to-point validation flag (it skips instead of rolling back)."""
    out = _run(2, 1, 2, "--validate")
    assert '"scenario": "validate"' in out and '"ok": false' not in out
    assert '"via_preceding": true' in out  # the point-to-point flag path was exercised


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_dp2_fused_allreduce_adam():
    """DP=2 all-reduce fused into AdamW over NVLink: bit-identical to NCCL + AdamW."""
    out = _run(2, 2, 1, "--fused-ar")
    assert '"scenario": "fused_ar"' in out and '"ok": false' not in out


@pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs 4 GPUs")
def test_dp2_pp2_fused_allreduce_adam():
    out = _run(4, 2, 2, "--fused-ar")
    assert '"scenario": "fused_ar"' in out and '"ok": false' not in out


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_dp2_pp1_reroute_gpt_ends():
    """GPT ends (token + position embedding, final LN + LM head + cross-entropy) on the
    single stage, DP = 2: re-routing leaves the CE losses bit-identical."""
    out = _run(2, 2, 1, "--gpt-ends")
    assert '"ok": true' in out and '"ok": false' not in out


@pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs 4 GPUs")
def test_dp2_pp2_reroute_gpt_ends():
    """Embedding on stage 0, LM head + CE on stage 1, DP2 x PP2 with re-routing."""
    out = _run(4, 2, 2, "--gpt-ends")
    assert '"ok": true' in out and '"ok": false' not in out


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_dp2_pp1_reroute_three_iterations_fused_allreduce():
    """Three iterations per run with the fused DP = 2 all-reduce + AdamW (the bench's
    default): the replicas stay byte-identical step after step, fault-free and re-routed."""
    out = _run(2, 2, 1, "--iters", "3", "--fuse-ar-main")
    assert '"ok": true' in out and '"ok": false' not in out


@pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs 4 GPUs")
def test_dp2_pp2_reroute_three_iterations_fused_allreduce():
    """DP2 x PP2, three iterations per run, fused all-reduce where a stage has two live
    peers and plain AdamW where its peer failed: replicas byte-identical after the steps,
    losses within 1e-3 and the stage gradient within 1e-2 of the fault-free run."""
    out = _run(4, 2, 2, "--iters", "3", "--fuse-ar-main")
    assert '"ok": true' in out and '"ok": false' not in out


@pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs 4 GPUs")
def test_dp4_pp1_reroute_three_iterations():
    """Four data-parallel replicas of one stage (NCCL all-reduce over the live peers),
    a failed worker (two placements) re-routed to the three survivors, three iterations per run."""
    out = _run(4, 4, 1, "--iters", "3")
    assert '"ok": true' in out and '"ok": false' not in out


@pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs 4 GPUs")
def test_dp1_pp4_pipeline_gpt_ends_three_iterations():
    """A four-stage pipeline (the N = 8 default's depth) with the GPT ends, three iterations."""
    out = _run(4, 1, 4, "--gpt-ends", "--iters", "3")
    assert '"ok": true' in out and '"ok": false' not in out


@pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs 4 GPUs")
def test_dp2_pp2_normalization_swap_gpt_ends():
    """The normalization swap when the roles moved hold different stage models (embedding
    on stage 0, LM head on stage 1): the GPU taking over binds its new role's model, then
    receives the state (slip_migrate_state checks that both sides agree on the size)."""
    out = _run(4, 2, 2, "--gpt-ends", "--migrate")
    assert '"ok": true' in out and '"ok": false' not in out


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_dp2_fused_allreduce_push_into_w():
    """slip_comm_fuse_ar_push: each peer's W launches also write their dW tiles into the
    other's receive buffer (TMA over NVLink); AdamW reads them locally.  Master, m, v, the
    bf16 weights and the losses equal the NCCL all-reduce + AdamW bit for bit, and the
    re-route scenarios keep the replicas byte-identical over three iterations."""
    out = _run(2, 2, 1, "--fused-ar", "--push")
    assert '"ok": true' in out and '"ok": false' not in out
    out = _run(2, 2, 1, "--iters", "3", "--fuse-ar-main", "--push")
    assert '"ok": true' in out and '"ok": false' not in out


@pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs 4 GPUs")
def test_dp2_pp2_fused_allreduce_push_into_w():
    """Push mode with two stages (several W launches per iteration: the mirror adds with
    TMA reduce-add into the peer's buffer) and a failed worker (a singleton stage)."""
    out = _run(4, 2, 2, "--fused-ar", "--push")
    assert '"ok": true' in out and '"ok": false' not in out


@pytest.mark.skipif(torch.cuda.device_count() < 4, reason="needs 4 GPUs")
def test_dp2_pp2_reroute_ragged_shape():
    """A ragged stage (h 640, d = 80, s = 200) through re-routing with the fused all-reduce
    and two iterations: partial GEMM / attention tiles in every P2P-fed stage."""
    out = _run(4, 2, 2, "--ragged", "--iters", "2", "--fuse-ar-main")
    assert '"ok": true' in out and '"ok": false' not in out
