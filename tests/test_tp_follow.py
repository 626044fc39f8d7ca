"""NX_TP_NCCL on the device clock: rank 0's engine forwards every launch to the
followers (nx_engine_set_launch_observer), which replay them with
device.tp_follow. The NCCL path itself needs >= 2 GPUs; here the plumbing is
checked on CPU: the observer's batches are exactly the engine's launches, and
a world-size-2 gloo job (the bench's transport) delivers them to a follower
that issues the same batches in the same per-lane order."""
import json
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _engine(nx):
    tiny = nx.derive(256, 1024, 2, 4, 2)
    trace = nx.workload_trace("mixed", 2.5, 24, 3)
    return nx.Engine(nx.sim_config(tiny, nx.gpu_preset("desk"))), trace


def test_observer_batches_are_the_engine_launches(nx):
    eng, trace = _engine(nx)
    seen = []
    eng.set_launch_observer(seen.append)
    eng.submit_trace(trace)
    eng.run()
    launches = [l.split("\t") for l in eng.event_log().splitlines() if l.split("\t")[2] == "launch"]
    assert len(seen) == len(launches) > 10
    for b, l in zip(seen, launches):
        assert b["lane"] == (1 if l[1] == "decode" else 0)
        if l[1] == "prefill":
            assert b["sm_pct"] == int(l[4])
        # members in log order with the logged token counts; pages cover the
        # positions the launch writes
        assert [m["n"] for m in b["members"]] == [int(m.split(":")[1]) for m in l[3].split(",")]
        for m in b["members"]:
            assert 16 * len(m["pages"]) >= m["start"] + m["n"]
        # no device bound: the engine holds no token ids
        assert all(m["tokens"] == [] for m in b["members"])


def test_observer_errors_surface(nx):
    eng, trace = _engine(nx)

    def boom(_b):
        raise KeyError("x")

    eng.set_launch_observer(boom)
    eng.submit_trace(trace)
    with pytest.raises(RuntimeError, match="launch observer failed"):
        eng.run()


class _FakeShard:
    """Stands in for a follower's Device: records launches, enforces that a
    lane is relaunched only after its previous batch was waited for."""

    def __init__(self):
        self.log, self.pending = [], set()

    def launch(self, members, lane=0, sm_pct=100):
        assert lane not in self.pending
        self.pending.add(lane)
        self.log.append(dict(lane=lane, sm_pct=sm_pct, members=members))

    def wait(self, lane):
        self.pending.remove(lane)
        return [], 0.0


def _worker(rank, world, port, out_dir):
    import paper_2507_06608_b200 as nx
    from paper_2507_06608_b200 import device as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if rank == 0:
            eng, trace = _engine(nx)
            sent = []

            def forward(b):
                sent.append(b)
                dist.broadcast_object_list([b], src=0)

            eng.set_launch_observer(forward)
            eng.submit_trace(trace)
            eng.run()
            dist.broadcast_object_list([None], src=0)
            json.dump(sent, open(os.path.join(out_dir, "rank0.json"), "w"))
        else:
            shard = _FakeShard()

            def recv():
                box = [None]
                dist.broadcast_object_list(box, src=0)
                return box[0]

            n = D.tp_follow(shard, recv)
            assert n == len(shard.log) and not shard.pending
            json.dump(shard.log, open(os.path.join(out_dir, f"rank{rank}.json"), "w"))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_follower_replays_rank0_launches_gloo(tmp_path):
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    sent = json.load(open(tmp_path / "rank0.json"))
    got = json.load(open(tmp_path / "rank1.json"))
    assert len(sent) > 10 and got == sent
