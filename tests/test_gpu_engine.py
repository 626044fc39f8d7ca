"""The step executor driving the real device.

* virtual clock + device: scheduling (event/decision logs) byte-identical to
  the compiled reference on C1, while every batch really runs on the two
  green-context partitions and produces greedy tokens; tokens are checked
  against the fp32 oracle under teacher forcing (margin rule of
  test_gpu_model.py).
* device clock: latencies are measured; feeding them to the pinned Python
  port (oracle/engine_port.py) reproduces the run's logs exactly (replay
  parity), and block tables match the page-model oracle.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LOGIT_TOL = 3e-2


@pytest.fixture(scope="module")
def tiny_dev():
    from paper_2507_06608_b200 import device as D
    # desk GpuSpec capacity = 4 GiB / 2048 B = 2M tokens -> 131072 pages (+slack)
    return D.Device(D.arch_preset("tiny"), num_pages=(4 << 30) // 2048 // 16 + 4096, seed=5)


def _teacher_forced_check(ref, tokens, prompt_len, max_checked=64):
    seq = np.array(tokens)
    logits = ref.logits(seq[:-1])[prompt_len - 1:]
    gen = seq[prompt_len:]
    checked = mism = 0
    for row, tok in list(zip(logits, gen))[:max_checked]:
        top2 = np.sort(row)[-2:]
        if top2[1] - top2[0] > 4 * LOGIT_TOL * np.abs(row).max():
            checked += 1
            mism += int(tok != int(np.argmax(row)))
    return checked, mism


def test_c1_virtual_clock_with_device(nx, tiny_dev):
    from oracle import reference
    from oracle.llama_fp32 import LlamaFP32
    tiny = nx.derive(256, 1024, 2, 4, 2)
    trace = nx.workload_trace("mixed", 2.5, 64, 1)
    cfg = nx.sim_config(tiny, nx.gpu_preset("desk"))
    eng = nx.Engine(cfg, device=tiny_dev)
    eng.submit_trace(trace)
    eng.run()
    if reference.available():
        r = reference.run(cfg, trace)
        assert eng.event_log() == r["event_log"]
        assert eng.decision_log() == r["decision_log"]
    import hashlib
    assert hashlib.sha256(eng.event_log().encode()).hexdigest()[:16] == "9ef62d973e3f23f9"
    reqs = eng.requests()
    assert all(q.finish_s >= 0 for q in reqs)
    ref = LlamaFP32(tiny_dev)
    # teacher-forced greedy parity on a spread of requests (short and long prompts)
    picks = sorted(reqs, key=lambda q: q.prompt_len)
    picks = picks[:4] + picks[len(picks) // 2: len(picks) // 2 + 2] + picks[-2:]
    total_checked = total_mism = 0
    for q in picks:
        toks = eng.tokens(q.id)
        assert len(toks) == q.prompt_len + q.output_len
        c, m = _teacher_forced_check(ref, toks, q.prompt_len)
        total_checked += c
        total_mism += m
    assert total_checked > 50
    assert total_mism == 0


def test_device_clock_replay_parity(nx, tiny_dev):
    from oracle.engine_port import run_port
    from oracle.kvpages_model import replay_pages
    tiny = nx.derive(256, 1024, 2, 4, 2)
    trace = nx.workload_trace("sharegpt", 50.0, 40, 2)
    cfg = nx.sim_config(tiny, nx.gpu_preset("desk"), clock_mode=nx.NX_CLOCK_DEVICE)
    eng = nx.Engine(cfg, device=tiny_dev)
    eng.submit_trace(trace)
    eng.run()
    lat = eng.launch_latencies()
    assert len(lat) > 10 and all(x > 0 for x in lat)
    dev_ms = eng.launch_device_ms()
    assert all(d > 0 for d in dev_ms)
    # replay through the pinned Python port and through the product's replay clock
    replay_cfg = nx.sim_config(tiny, nx.gpu_preset("desk"), clock_mode=nx.NX_CLOCK_REPLAY)
    ev, dec = run_port(replay_cfg, trace, replay=lat)
    assert ev == eng.event_log()
    assert dec == eng.decision_log()
    e2 = nx.Engine(replay_cfg)
    e2.set_replay_latencies(lat)
    e2.submit_trace(trace)
    e2.run()
    assert e2.event_log() == eng.event_log()
    n_pages = tiny_dev.cfg.num_pages
    log, live = replay_pages(eng.event_log(), {r.id: r.prompt_len for r in trace}, 16, n_pages)
    assert eng.page_log() == log and not live


def test_static_and_monolithic_engines_on_device(nx, tiny_dev):
    from oracle import reference
    tiny = nx.derive(256, 1024, 2, 4, 2)
    trace = nx.workload_trace("mixed", 2.5, 24, 3)
    for kind in (nx.NX_ENGINE_STATIC, nx.NX_ENGINE_MONOLITHIC):
        cfg = nx.sim_config(tiny, nx.gpu_preset("desk"), kind=kind)
        eng = nx.Engine(cfg, device=tiny_dev)
        eng.submit_trace(trace)
        eng.run()
        if reference.available():
            assert eng.event_log() == reference.run(cfg, trace)["event_log"]
        for q in eng.requests():
            assert len(eng.tokens(q.id)) == q.prompt_len + q.output_len


def test_launch_observer_replays_on_a_second_device(nx, tiny_dev):
    """The NX_TP_NCCL leader / follower protocol on one GPU: rank 0's engine
    forwards every launch (with the token ids it holds once a device is bound)
    and a second device with the same weights replays them with
    device.tp_follow; every token the follower samples is the token the
    engine appended for that member."""
    from paper_2507_06608_b200 import device as D
    tiny = nx.derive(256, 1024, 2, 4, 2)
    trace = nx.workload_trace("sharegpt", 50.0, 24, 9)
    cfg = nx.sim_config(tiny, nx.gpu_preset("desk"))
    eng = nx.Engine(cfg, device=tiny_dev)
    sent = []
    eng.set_launch_observer(sent.append)
    eng.submit_trace(trace)
    eng.run()
    launches = [l.split("\t") for l in eng.event_log().splitlines() if l.split("\t")[2] == "launch"]
    assert len(sent) == len(launches) > 10
    follower = D.Device(D.arch_preset("tiny"), num_pages=tiny_dev.cfg.num_pages, seed=5)
    try:
        fifo, produced = {}, {}
        launch0, wait0 = follower.launch, follower.wait
        order = []

        def launch_tracked(members, lane=0, sm_pct=100):
            order.append(lane)
            fifo.setdefault(lane, []).append(len(order) - 1)
            launch0(members, lane=lane, sm_pct=sm_pct)

        def wait(lane):
            toks, ms = wait0(lane)
            produced[fifo[lane].pop(0)] = toks
            return toks, ms

        follower.launch, follower.wait = launch_tracked, wait
        it = iter(sent + [None])
        assert D.tp_follow(follower, lambda: next(it)) == len(sent)
        checked = 0
        for k, (b, l) in enumerate(zip(sent, launches)):
            ids = [int(m.split(":")[0]) for m in l[3].split(",")]
            toks = iter(produced[k])
            for rid, m in zip(ids, b["members"]):
                assert len(m["tokens"]) == m["n"]
                if m["sample"]:
                    assert next(toks) == eng.tokens(rid)[m["start"] + m["n"]]
                    checked += 1
        assert checked > 50
    finally:
        follower.close()
