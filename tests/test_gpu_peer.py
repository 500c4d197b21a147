"""The fused DP = 2 all-reduce + AdamW (slip_optimizer_step_peer, the compute half of
slip_comm_fuse_ar_adam, SURVEY §8(e) option (i); the all-reduce of PAPER.md line 561 and
the optimizer step of line 583) in ONE process driving two GPUs with peer access: the
step that reads g_own + g_peer over NVLink must equal slip_optimizer_step on the summed
gradient bit for bit (the same fp32 addition, the same update), and the peer buffer must
be left untouched."""
import ctypes as C

import pytest
import torch

import slipdata as sd

pytestmark = pytest.mark.gpu


def _need_two():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")


@pytest.mark.parametrize("name", ["c1", "d80"])
def test_optimizer_step_peer_equals_step_on_summed_gradient(name):
    _need_two()
    from cuda.bindings import runtime as cudart
    from paper_2405_14009_b200 import runtime as rt
    from paper_2405_14009_b200._binding import slip_adam
    cfg, L = {"c1": (sd.C1_TINY, 1),
              "d80": (sd.ModelCfg(hidden=640, heads=8, ffn=2560, seq=200, micro_batch=1, layers=2), 2)}[name]
    torch.cuda.set_device(0)
    err = cudart.cudaDeviceEnablePeerAccess(1, 0)[0]
    assert err in (cudart.cudaError_t.cudaSuccess, cudart.cudaError_t.cudaErrorPeerAccessAlreadyEnabled), err
    master = torch.from_numpy(sd.pack_stage(sd.stage_params(cfg, 0, L, total_layers=max(L, 2)))).float()
    n = master.numel()
    g0 = torch.randn(n, generator=torch.Generator().manual_seed(1)) * 1e-2
    g1 = torch.randn(n, generator=torch.Generator().manual_seed(2)) * 1e-2
    adam = slip_adam(1e-3, 0.9, 0.95, 1e-8, 0.1)
    out = []
    for fused in (False, True):
        st = rt.Stage(cfg, L, n_slots=1)
        st.load_master(master.cuda(0))
        peer = g1.to("cuda:1")
        flag = torch.zeros(1, dtype=torch.int32, device="cuda:0")
        s = rt._stream()
        for k in (1, 2):  # two steps: the moments carry over
            if fused:
                st.grad.copy_(g0.cuda(0))
                torch.cuda.synchronize(1)
                rt.call("slip_optimizer_step_peer", st.ctx, C.byref(adam), k, 0.5, C.c_void_p(flag.data_ptr()),
                        C.c_void_p(peer.data_ptr()), s)
            else:
                st.grad.copy_((g0 + g1).cuda(0))
                rt.call("slip_optimizer_step", st.ctx, C.byref(adam), k, 0.5, C.c_void_p(flag.data_ptr()), s)
        torch.cuda.synchronize(0)
        assert int(flag.item()) == 0
        if fused:
            assert torch.equal(peer.cpu(), g1)
        out.append([st.master.clone(), st.adam_m.clone(), st.adam_v.clone(), st.w.clone()])
        st.close()
    for a, b, what in zip(out[0], out[1], ("master", "m", "v", "w")):
        assert torch.equal(a, b), what
