"""Multi-process host logic of the N > 1 path on CPU (torch.distributed gloo,
world_size 2): every process builds the rank programs (slip_rank_program, the
executor's action lists) for its share of the ranks, the programs are exchanged
with all_gather_object, and each process checks

  * all processes computed the identical plan (hash) — the planner is replicated,
  * every directed pair is FIFO (the receiver posts receives in send order),
  * the ops executed by the live ranks partition all (stage, micro-batch) work,
  * a model of the executor's stream / event protocol (compute stream, one stream
    per directed pair with rendezvous send/recv, the stage all-reduce as a
    collective over live peers) runs to completion: no deadlock — both with the
    NCCL all-reduce and with the DP = 2 all-reduce fused into AdamW
    (slip_comm_fuse_ar_adam), whose OPT is a flag barrier with the peer, AdamW, and
    a second barrier, all on the compute stream.
"""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

CASES = [
    (2, 2, 3, []), (2, 2, 3, [(1, 1)]), (2, 2, 3, [(0, 0)]),
    (4, 2, 3, []), (4, 2, 3, [(3, 1)]), (4, 2, 3, [(3, 1), (2, 0)]), (4, 2, 3, [(0, 1)]),
    (4, 2, 2, [(1, 0)]), (4, 2, 1, [(2, 1)]), (2, 2, 8, [(1, 0)]), (4, 2, 16, [(3, 1)]),
    (4, 3, 6, [(2, 1)]), (3, 3, 4, [(1, 0), (2, 2), (0, 1)]), (4, 2, 8, [(1, 1)]),
]
KINDS = ("LOAD_X", "RECV_X", "F", "SEND_Y", "LOSS", "RECV_DY", "B", "SEND_DX", "W", "BC", "AR", "OPT")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def simulate(progs, N, DP, live, fused=False):
    """Executor stream/event model; returns True if every action completes.  fused:
    stages with exactly 2 live workers skip the AR collective and run OPT as
    barrier -> AdamW -> barrier with the peer on the compute stream."""
    nodes = []  # dict(deps=set, rv=key or None)
    rv_groups = {}

    def add(deps, rv=None):
        nodes.append({"deps": set(d for d in deps if d is not None), "rv": rv})
        if rv is not None:
            rv_groups.setdefault(rv, []).append(len(nodes) - 1)
        return len(nodes) - 1

    for r, prog in enumerate(progs):
        tail = {}  # stream -> last node
        chan = {}  # (src, dst, kind) -> count
        ar_count = 0
        opt_count = 0
        pair_fused = fused and sum(1 for k in range(DP) if live[r % N][k]) == 2
        slot = {}  # slot -> dict(freed, sent_y, sent_dx)
        pending_cs_dep = None
        for a in prog:
            kind, it, mb, origin, peer, s, acc = a
            k = KINDS[kind]
            sv = slot.setdefault(s, {"freed": None, "sent_y": None, "sent_dx": None})
            cs = tail.get("cs")
            if k == "LOAD_X":
                n = add([cs, sv["freed"]])
                tail["cs"] = n
            elif k in ("RECV_X", "RECV_DY"):
                st = ("pair", peer, r)
                q = chan.get((peer, r, k), 0)
                chan[(peer, r, k)] = q + 1
                deps = [tail.get(st)]
                deps += [sv["freed"]] if k == "RECV_X" else [sv["sent_y"], cs]
                n = add(deps, rv=(peer, r, "act" if k == "RECV_X" else "grad", q))
                tail[st] = n
                pending_cs_dep = n
            elif k in ("SEND_Y", "SEND_DX"):
                st = ("pair", r, peer)
                q = chan.get((r, peer, k), 0)
                chan[(r, peer, k)] = q + 1
                n = add([tail.get(st), cs], rv=(r, peer, "act" if k == "SEND_Y" else "grad", q))
                tail[st] = n
                sv["sent_y" if k == "SEND_Y" else "sent_dx"] = n
            elif k == "AR" and pair_fused:
                continue  # the exchange happens inside OPT
            elif k == "OPT" and pair_fused:
                stage = r % N
                b1 = add([cs, pending_cs_dep], rv=("bar", stage, opt_count, 0))
                adam = add([b1])
                b2 = add([adam], rv=("bar", stage, opt_count, 1))
                opt_count += 1
                pending_cs_dep = None
                tail["cs"] = b2
            elif k == "AR":
                stage = r % N
                n = add([tail.get("ar"), cs], rv=("ar", stage, ar_count))
                ar_count += 1
                tail["ar"] = n
                pending_cs_dep = n
            else:  # compute on cs: F, LOSS, B, BC, W, OPT
                deps = [cs, pending_cs_dep]
                if k == "F":
                    deps.append(sv["sent_y"])
                if k in ("B", "BC"):
                    deps.append(sv["sent_dx"])  # slot.dx is the previous occupant's send buffer
                n = add(deps)
                pending_cs_dep = None
                tail["cs"] = n
                if k in ("W", "BC"):
                    sv["freed"] = n
    # singleton all-reduce groups need no partner
    for key, members in rv_groups.items():
        if key[0] == "ar":
            n_live = sum(1 for k in range(DP) if live[key[1]][k])
            if n_live == 1 or len(members) == 1:
                for i in members:
                    nodes[i]["rv"] = None
    done = [False] * len(nodes)
    changed = True
    while changed:
        changed = False
        for i, nd in enumerate(nodes):
            if done[i] or not all(done[d] for d in nd["deps"]):
                continue
            if nd["rv"] is None:
                done[i] = changed = True
                continue
            grp = rv_groups[nd["rv"]]
            if len(grp) >= 2 and all(all(done[d] for d in nodes[g]["deps"]) for g in grp):
                for g in grp:
                    done[g] = True
                changed = True
    return all(done)


def _worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2405_14009_b200 import runtime as rt
    ok = []
    for (N, DP, m, failed) in CASES:
        live = [[1] * DP for _ in range(N)]
        for (i, k) in failed:
            live[i][k] = 0
        costs = rt.make_costs(t_f=3, t_b=4, t_w=2, t_comm=1, t_ar=2, t_opt=1)
        H = 2
        plan = rt.plan_schedule(N, DP, m, live, costs, True, True, H)
        mine = {r: rt.rank_program(N, DP, m, live, costs, r, True, True, H)[0]
                for r in range(N * DP) if r % world == rank}
        gathered = [None] * world
        dist.all_gather_object(gathered, (plan.hash, mine))
        hashes = {g[0] for g in gathered}
        progs = {}
        for g in gathered:
            progs.update(g[1])
        progs = [progs[r] for r in range(N * DP)]
        # FIFO per directed pair
        snd, rcv = {}, {}
        for r, p in enumerate(progs):
            for a in p:
                k = KINDS[a[0]]
                if k in ("SEND_Y", "SEND_DX"):
                    snd.setdefault((r, a[4], k == "SEND_DX"), []).append(a[1:4])
                if k in ("RECV_X", "RECV_DY"):
                    rcv.setdefault((a[4], r, k == "RECV_DY"), []).append(a[1:4])
        # work partition: every (iter, stage, mb, origin) F / B / W exactly once on live ranks
        work = sorted((r % N, a[1], a[2], a[3], KINDS[a[0]]) for r, p in enumerate(progs) for a in p
                      if KINDS[a[0]] in ("F", "B", "W"))
        want = sorted((i, t, j, k, ph) for i in range(N) for t in range(H) for j in range(m) for k in range(DP)
                      for ph in ("F", "B", "W"))
        dead_idle = all(not progs[k * N + i] for i in range(N) for k in range(DP) if not live[i][k])
        ok.append((len(hashes) == 1, snd == rcv, work == want, dead_idle, simulate(progs, N, DP, live),
                   simulate(progs, N, DP, live, fused=True)))
    results[rank] = ok
    dist.destroy_process_group()


def test_rank_programs_gloo_world2():
    pytest.importorskip("paper_2405_14009_b200")
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    for r in range(world):
        for case, flags in zip(CASES, results[r]):
            assert all(flags), (case, flags)
