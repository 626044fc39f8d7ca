"""Bit-exact parity of the product's host path against the compiled reference.

Decisions, SM splits and logs must be byte-identical (SURVEY §8(c) "Parity
targets"): randomized operator/cost-model/controller/scheduler checks plus
whole-engine event and decision logs on several fixtures.
"""
import ctypes as C
import hashlib
import random

import pytest

from paper_2507_06608_b200 import _abi
from oracle.kvpages_model import replay_pages


def _ref_ops(ref, fn, *args):
    out = (_abi.OpWorkload * 8)()
    n = C.c_size_t()
    assert fn(*args, out, C.byref(n)) == 0
    return list(out[: n.value])


def _ops_equal(a, b):
    assert len(a) == len(b)
    for x, y in zip(a, b):
        assert (x.kind, x.is_attention) == (y.kind, y.is_attention)
        assert (x.flops, x.mem_bytes, x.kv_bytes) == (y.flops, y.mem_bytes, y.kv_bytes)


def _bd_equal(a, b):
    assert (a.total_s, a.attn_mem_time_s, a.n_ops) == (b.total_s, b.attn_mem_time_s, b.n_ops)
    for i in range(a.n_ops):
        x, y = a.per_op[i], b.per_op[i]
        assert (x.kind, x.memory_bound, x.compute_s, x.mem_s) == (y.kind, y.memory_bound, y.compute_s, y.mem_s)


MODELS = [(256, 1024, 2, 4, 2), (4096, 14336, 32, 32, 2), (5120, 13824, 48, 40, 2), (2048, 8192, 36, 16, 2),
          (2, 8, 1, 1, 2), (8192, 28672, 80, 64, 2)]


@pytest.mark.parametrize("dims", MODELS)
def test_opmodel_and_costmodel_randomized(nx, ref, dims):
    L = ref.lib()
    rng = random.Random(hash(dims) & 0xFFFF)
    m = nx.derive(*dims)
    mr = L.nxref_model_derive(*dims)
    assert bytes(m) == bytes(mr)
    gpus = [nx.gpu_preset(n) for n in ("desk", "desk-contention", "l20like")]
    gpus.append(nx.gpu_spec(148, 1.6595e15, 6.5562e12, 100 << 30))
    prof = nx.lib().nx_kernel_profile_default()
    for _ in range(60):
        chunks = []
        for _ in range(rng.randint(1, 6)):
            t = rng.randint(1, 2048)
            chunks.append((t, t + rng.randint(0, 16000)))
        lens = [rng.randint(1, 20000) for _ in range(rng.randint(1, 64))]
        tok = (C.c_int64 * len(chunks))(*[c[0] for c in chunks])
        ctx = (C.c_int64 * len(chunks))(*[c[1] for c in chunks])
        dl = (C.c_int64 * len(lens))(*lens)
        pa = nx.prefill_batch_workloads(m, chunks)
        _ops_equal(pa, _ref_ops(ref, L.nxref_prefill_batch_workloads, C.byref(mr), tok, ctx, len(chunks)))
        da = nx.decode_op_workloads(m, lens)
        _ops_equal(da, _ref_ops(ref, L.nxref_decode_op_workloads, C.byref(mr), dl, len(lens)))
        ma = nx.mixed_batch_workloads(m, chunks, lens)
        _ops_equal(ma, _ref_ops(ref, L.nxref_mixed_batch_workloads, C.byref(mr), tok, ctx, len(chunks), dl,
                                len(lens)))
        g = rng.choice(gpus)
        for share_pct in (1, rng.randint(2, 98), 99, 100):
            share = share_pct / 100.0
            for ops in (pa, da, ma):
                arr = (_abi.OpWorkload * len(ops))(*ops)
                b1 = nx.phase_latency_isolated(ops, share, g, prof)
                b2 = _abi.Breakdown()
                assert L.nxref_phase_latency_isolated(arr, len(ops), share, C.byref(g), C.byref(prof),
                                                      C.byref(b2)) == 0
                _bd_equal(b1, b2)
            pbd = nx.phase_latency_isolated(pa, 1 - share + 0.01 if share < 0.99 else 0.5, g, prof)
            c1 = nx.decode_latency_contended(da, share, pbd, pa, g, prof)
            c2 = _abi.Breakdown()
            parr = (_abi.OpWorkload * len(pa))(*pa)
            darr = (_abi.OpWorkload * len(da))(*da)
            assert L.nxref_decode_latency_contended(darr, len(da), share, C.byref(pbd), parr, len(pa), C.byref(g),
                                                    C.byref(prof), C.byref(c2)) == 0
            _bd_equal(c1, c2)


def test_controller_sequences_match(nx, ref):
    """A long scripted sequence of decide() calls on both controllers."""
    L = ref.lib()
    rng = random.Random(7)
    cfg = nx.lib().nx_controller_config_default()
    init = _abi.PartitionState(50, 50, 50)
    mine = nx.PartitionController(init, cfg)
    h = C.c_void_p()
    L.nxref_controller_create(C.byref(init), C.byref(cfg), C.byref(h))
    from paper_2507_06608_b200 import _Phase
    for step in range(3000):
        a, b = rng.uniform(0.1, 3), rng.uniform(0.1, 3)
        sat_p, sat_d = rng.randint(10, 90), rng.randint(10, 90)
        pf = lambda p, a=a, s=sat_p: a * 100.0 / min(p, s)  # noqa: E731
        df = lambda p, b=b, s=sat_d: b * 100.0 / min(p, s) + (0.3 if p < 20 else 0)  # noqa: E731
        pre = (rng.random() > 0.1, pf)
        dec = (rng.random() > 0.1, df)
        cap = 1 << 30
        used = rng.randint(0, cap)
        d1 = mine.decide(used, cap, pre, dec)
        p, d = _Phase(*pre), _Phase(*dec)
        d2 = _abi.Decision()
        assert L.nxref_controller_decide(h, used, cap, C.byref(p.pm), C.byref(d.pm), C.byref(d2)) == 0
        assert bytes(d1) == bytes(d2), step
    L.nxref_controller_destroy(h)


def test_schedulers_randomized(nx, ref):
    L = ref.lib()
    rng = random.Random(11)
    for trial in range(300):
        n = rng.randint(0, 80)
        queue = [(i, rng.randint(1, 9000), round(rng.uniform(0, 50), rng.choice([0, 1, 3]))) for i in
                 rng.sample(range(10000), n)]
        active = [(i, round(rng.uniform(0, 50), rng.choice([0, 1, 3]))) for i in rng.sample(range(10000), rng.randint(0, 100))]
        budget = rng.choice([1, 7, 512, 2048, 4096])
        gamma = rng.choice([0.0, 15.0, 1e6])
        now = rng.uniform(0, 60)
        skip = rng.random() < 0.3
        q = (_abi.PrefillEntry * max(1, n))(*[_abi.PrefillEntry(*e) for e in queue])
        a = (_abi.DecodeCandidate * max(1, len(active)))(*[_abi.DecodeCandidate(*e) for e in active])

        def ref_plan(fn, *args):
            out = (_abi.BatchMember * 4096)()
            k, tot = C.c_size_t(), C.c_int64()
            assert fn(*args, out, 4096, C.byref(k), C.byref(tot)) == 0
            return [(x.id, x.tokens) for x in out[: k.value]], tot.value

        assert nx.spf_schedule(queue, budget, gamma, now, skip) == ref_plan(L.nxref_spf_schedule, q, n, budget,
                                                                           gamma, now, int(skip))
        assert nx.fcfs_prefill_schedule(queue, budget) == ref_plan(L.nxref_fcfs_prefill_schedule, q, n, budget)
        mb = rng.choice([1, 8, 64, 256])
        assert nx.fcfs_decode_schedule(active, mb) == ref_plan(L.nxref_fcfs_decode_schedule, a, len(active), mb)
        ch = rng.choice([1, 100, 2048])
        assert nx.chunked_mixed_schedule(queue, active, budget, mb, ch) == ref_plan(
            L.nxref_chunked_mixed_schedule, q, n, a, len(active), budget, mb, ch)


@pytest.mark.parametrize("preset,rate,count,seed", [("mixed", 2.5, 64, 1), ("sharegpt", 20.0, 300, 3),
                                                    ("long-data", 1.5, 40, 2), ("arxiv", 4.0, 50, 5)])
def test_traces_identical(nx, ref, preset, rate, count, seed):
    a = nx.workload_trace(preset, rate, count, seed)
    b = ref.workload_trace(preset, rate, count, seed)
    assert nx.trace_text(a) == ref.trace_text(b)
    assert nx.trace_text(nx.parse_trace(nx.trace_text(a))) == nx.trace_text(a)


def test_c1_trace_fingerprint(nx):
    """the C1 trace file hashes to 456b6f50a9c1f2aa."""
    t = nx.trace_text(nx.workload_trace("mixed", 2.5, 64, 1))
    assert hashlib.sha256(t.encode()).hexdigest()[:16] == "456b6f50a9c1f2aa"


def _fixtures(nx):
    tiny = nx.derive(256, 1024, 2, 4, 2)
    b200 = nx.gpu_spec(148, 1.6595e15, 6.5562e12, 100 << 30)
    tight = nx.gpu_preset("desk-tight")
    tight.kv_capacity_bytes = 64 << 20
    fx = {
        "c1-nexus": (tiny, nx.gpu_preset("desk"), dict(kind=nx.NX_ENGINE_NEXUS), ("mixed", 2.5, 64, 1)),
        "c1-static": (tiny, nx.gpu_preset("desk"), dict(kind=nx.NX_ENGINE_STATIC), ("mixed", 2.5, 64, 1)),
        "c1-static30": (tiny, nx.gpu_preset("desk"), dict(kind=nx.NX_ENGINE_STATIC, static_r_p=30),
                        ("mixed", 2.5, 64, 1)),
        "c1-mono": (tiny, nx.gpu_preset("desk"), dict(kind=nx.NX_ENGINE_MONOLITHIC), ("mixed", 2.5, 64, 1)),
        "c1-fcfs": (tiny, nx.gpu_preset("desk"), dict(prefill_policy=nx.NX_PREFILL_FCFS), ("mixed", 2.5, 64, 1)),
        "c1-b200": (tiny, b200, dict(), ("mixed", 2.5, 64, 1)),
        "contention": (nx.model_preset("tiny"), nx.gpu_preset("desk-contention"), dict(), ("long-data", 2.5, 80, 1)),
        "8b-sharegpt": (nx.model_preset("8b"), nx.gpu_spec(148, 2.25e15, 8e12, 150 << 30), dict(),
                        ("sharegpt", 20.0, 400, 1)),
        "3b-l20": (nx.model_preset("3b"), nx.gpu_preset("l20like"), dict(), ("arxiv", 1.0, 60, 4)),
        "timeout": (tiny, nx.gpu_preset("desk"), dict(timeout_sim_s=5.0), ("mixed", 2.5, 64, 1)),
        "max-events": (tiny, nx.gpu_preset("desk"), dict(max_events=777), ("mixed", 2.5, 64, 1)),
    }
    return fx, tight


FIXTURES = ["c1-nexus", "c1-static", "c1-static30", "c1-mono", "c1-fcfs", "c1-b200", "contention", "8b-sharegpt",
            "3b-l20", "timeout", "max-events"]


@pytest.mark.parametrize("name", FIXTURES)
def test_engine_logs_byte_identical(nx, ref, name):
    fx, _ = _fixtures(nx)
    model, gpu, kw, (preset, rate, count, seed) = fx[name]
    cfg = nx.sim_config(model, gpu, **kw)
    trace = nx.workload_trace(preset, rate, count, seed)
    mine = nx.run(cfg, trace)
    theirs = ref.run(cfg, trace)
    assert mine.event_log == theirs["event_log"]
    assert mine.decision_log == theirs["decision_log"]
    assert mine.summary_json == theirs["summary_json"]
    assert mine.timed_out == theirs["timed_out"]
    assert mine.sim_end_s == theirs["sim_end_s"]


def test_c1_fingerprints(nx):
    """SURVEY Appendix B log hashes (nexus / static / monolithic on desk)."""
    tiny = nx.derive(256, 1024, 2, 4, 2)
    trace = nx.workload_trace("mixed", 2.5, 64, 1)
    want = {nx.NX_ENGINE_NEXUS: ("9ef62d973e3f23f9", 17366), nx.NX_ENGINE_STATIC: ("d0489a18f928b7c9", 17932),
            nx.NX_ENGINE_MONOLITHIC: ("4c99c2d3e6f1dbad", 17644)}
    for kind, (h, n) in want.items():
        r = nx.run(nx.sim_config(tiny, nx.gpu_preset("desk"), kind=kind), trace)
        assert hashlib.sha256(r.event_log.encode()).hexdigest()[:16] == h
        assert len(r.event_log.splitlines()) == n


def test_decode_prioritized_fixture(nx, ref):
    """SURVEY Appendix B decode-mode fixture: in=64/out=4000, 64 MiB cap."""
    _, tight = _fixtures(nx)
    tiny = nx.derive(256, 1024, 2, 4, 2)
    trace = [nx.Request(i, t.arrival_s, 64, 4000) for i, t in enumerate(nx.workload_trace("sharegpt", 20.0, 200, 1))]
    cfg = nx.sim_config(tiny, tight)
    mine = nx.run(cfg, trace)
    theirs = ref.run(cfg, trace)
    assert mine.event_log == theirs["event_log"]
    assert mine.decision_log == theirs["decision_log"]
    modes = [l.split("\t")[2] for l in mine.decision_log.splitlines()[1:]]
    assert modes.count("decode") > 1000


def test_replay_clock_reproduces_virtual_run(nx):
    """Replay mode fed a run's own launch latencies reproduces its logs."""
    tiny = nx.derive(256, 1024, 2, 4, 2)
    trace = nx.workload_trace("mixed", 2.5, 64, 1)
    e1 = nx.Engine(nx.sim_config(tiny, nx.gpu_preset("desk")))
    e1.submit_trace(trace)
    e1.run()
    lat = e1.launch_latencies()
    e2 = nx.Engine(nx.sim_config(tiny, nx.gpu_preset("desk"), clock_mode=nx.NX_CLOCK_REPLAY))
    e2.set_replay_latencies(lat)
    e2.submit_trace(trace)
    e2.run()
    assert e2.event_log() == e1.event_log()
    assert e2.decision_log() == e1.decision_log()


def test_replay_with_perturbed_latencies_matches_port(nx):
    """Replay with arbitrary latencies: engine == oracle port (oracle/engine_port.py)."""
    from oracle.engine_port import run_port
    tiny = nx.derive(256, 1024, 2, 4, 2)
    trace = nx.workload_trace("mixed", 4.0, 40, 9)
    rng = random.Random(3)
    lat = [rng.uniform(1e-4, 5e-2) for _ in range(20000)]
    cfg = nx.sim_config(tiny, nx.gpu_preset("desk"), clock_mode=nx.NX_CLOCK_REPLAY)
    e = nx.Engine(cfg)
    e.set_replay_latencies(lat)
    e.submit_trace(trace)
    e.run()
    ev, dec = run_port(cfg, trace, replay=lat)
    assert e.event_log() == ev
    assert e.decision_log() == dec


def test_block_tables_match_page_model(nx):
    tiny = nx.derive(256, 1024, 2, 4, 2)
    trace = nx.workload_trace("mixed", 2.5, 64, 1)
    e = nx.Engine(nx.sim_config(tiny, nx.gpu_preset("desk")))
    e.configure_pages(16, 40000)
    e.submit_trace(trace)
    for _ in range(6000):  # stop mid-run so live tables exist
        e.step()
    log, live = replay_pages(e.event_log(), {r.id: r.prompt_len for r in trace}, 16, 40000)
    assert e.page_log() == log
    for rid, pages in live.items():
        assert e.block_table(rid) == pages
    e.run()
    log, live = replay_pages(e.event_log(), {r.id: r.prompt_len for r in trace}, 16, 40000)
    assert e.page_log() == log and not live


def test_engine_rejects_bad_traces(nx):
    tiny = nx.derive(256, 1024, 2, 4, 2)
    e = nx.Engine(nx.sim_config(tiny, nx.gpu_preset("desk")))
    e.submit(nx.Request(1, 1.0, 10, 10))
    with pytest.raises(ValueError):
        e.submit(nx.Request(2, 0.5, 10, 10))  # unsorted
    with pytest.raises(ValueError):
        e.submit(nx.Request(1, 2.0, 10, 10))  # duplicate
    with pytest.raises(ValueError):
        e.submit(nx.Request(3, 2.0, 0, 10))  # empty prompt
    with pytest.raises(ValueError):
        e.submit(nx.Request(4, 2.0, 10 ** 9, 10))  # footprint > capacity
    with pytest.raises(ValueError):
        nx.Engine(nx.sim_config(tiny, nx.gpu_preset("desk"), kind=nx.NX_ENGINE_STATIC, static_r_p=0))


def test_empty_trace(nx, ref):
    tiny = nx.derive(256, 1024, 2, 4, 2)
    cfg = nx.sim_config(tiny, nx.gpu_preset("desk"))
    mine = nx.run(cfg, [])
    theirs = ref.run(cfg, [])
    assert mine.event_log == theirs["event_log"] == ""


def test_cost_ext_disabled_is_reference_and_port_mirrors_enabled(nx, ref):
    """The flagged bandwidth extension: off == reference exactly; on, the
    product engine and the Python port still agree byte for byte."""
    from oracle.engine_port import run_port
    m = nx.model_preset("8b")
    g = nx.gpu_spec(148, 1.3e15, 5.5e12, 150 << 30)
    trace = nx.workload_trace("sharegpt", 25.0, 150, 4)
    off = nx.sim_config(m, g)
    assert nx.run(off, trace).event_log == ref.run(off, trace)["event_log"]
    on = nx.sim_config(m, g, bw_sat=[0.55, 0.7, 0.6, 0.55, 0.55])
    r = nx.run(on, trace)
    ev, dec = run_port(on, trace)
    assert r.event_log == ev and r.decision_log == dec
    # the extension changes the split: decode gets far more than 1-8 % of SMs
    applied = [int(l.split("\t")[4]) for l in r.decision_log.splitlines()[1:]]
    assert min(applied) < 90
    # standalone cost queries honour nx_set_cost_ext
    ops = nx.decode_op_workloads(m, [600] * 64)
    prof = nx.lib().nx_kernel_profile_default()
    base = nx.phase_latency_isolated(ops, 0.2, g, prof).total_s
    nx.set_cost_ext([0.6] * 5)
    try:
        slow = nx.phase_latency_isolated(ops, 0.2, g, prof).total_s
    finally:
        nx.set_cost_ext(None)
    assert slow > 2.5 * base


@pytest.mark.parametrize("name", FIXTURES)
def test_engine_logs_match_committed_golden(nx, name):
    """Same check without the reference library: committed sha256 fingerprints
    of the reference's logs (tests/golden/make_golden.py)."""
    import json
    import os
    golden = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))[name]
    fx, _ = _fixtures(nx)
    model, gpu, kw, (preset, rate, count, seed) = fx[name]
    trace = nx.workload_trace(preset, rate, count, seed)
    assert hashlib.sha256(nx.trace_text(trace).encode()).hexdigest() == golden["trace_sha256"]
    r = nx.run(nx.sim_config(model, gpu, **kw), trace)
    assert hashlib.sha256(r.event_log.encode()).hexdigest() == golden["event_log_sha256"]
    assert hashlib.sha256(r.decision_log.encode()).hexdigest() == golden["decision_log_sha256"]
    assert hashlib.sha256(r.summary_json.encode()).hexdigest() == golden["summary_sha256"]
    assert r.timed_out == golden["timed_out"] and r.sim_end_s == golden["sim_end_s"]


def test_c1_trace_file_golden(nx):
    import os
    text = open(os.path.join(os.path.dirname(__file__), "golden", "c1_mixed_64_2.5rps_seed1.trace")).read()
    assert nx.trace_text(nx.workload_trace("mixed", 2.5, 64, 1)) == text
    assert nx.trace_text(nx.parse_trace(text)) == text


def test_contention_ext_engine_matches_port(nx):
    """The flagged measured-contention term (nx_cost_ext.contention): the
    co-located decode prediction becomes isolated x (c0 + c1 p + c2 p^2);
    the product engine and the Python port agree byte for byte, and the term
    changes the predicted timeline versus the bandwidth-only extension."""
    from oracle.engine_port import run_port
    m = nx.model_preset("8b")
    g = nx.gpu_spec(148, 1.3e15, 5.5e12, 150 << 30)
    trace = nx.workload_trace("sharegpt", 40.0, 200, 7)
    bw = [0.45] * 5
    plain = nx.sim_config(m, g, bw_sat=bw)
    cont = nx.sim_config(m, g, bw_sat=bw, contention=[1.05, 0.3, -0.1])
    r = nx.run(cont, trace)
    ev, dec = run_port(cont, trace)
    assert r.event_log == ev and r.decision_log == dec
    assert r.event_log != nx.run(plain, trace).event_log
    ops = nx.decode_op_workloads(m, [600] * 64)
    pops = nx.prefill_batch_workloads(m, [(512, 512)] * 4)
    prof = nx.lib().nx_kernel_profile_default()
    nx.set_cost_ext(bw, [1.05, 0.3, -0.1])
    try:
        iso = nx.phase_latency_isolated(ops, 0.25, g, prof).total_s
        pbd = nx.phase_latency_isolated(pops, 0.75, g, prof)
        co = nx.decode_latency_contended(ops, 0.25, pbd, pops, g, prof).total_s
    finally:
        nx.set_cost_ext(None)
    assert abs(co / iso - (1.05 + 0.3 * 0.75 - 0.1 * 0.75 ** 2)) < 1e-12


def test_decode_target_ext_engine_matches_port(nx):
    """The flagged decode-step target (nx_cost_ext.decode_target_s): in
    prefill-priority mode a prefill share also fits when the co-located decode
    step stays within the target. Product and port agree byte for byte, with
    and without the contention factor; the target moves the split toward
    prefill versus the reference rule; a zero target is the reference."""
    from oracle.engine_port import run_port
    m = nx.model_preset("8b")
    g = nx.gpu_spec(148, 1.3e15, 5.5e12, 150 << 30)
    trace = nx.workload_trace("sharegpt", 40.0, 200, 7)
    bw = [0.45] * 5
    plain = nx.sim_config(m, g, bw_sat=bw)
    assert nx.run(nx.sim_config(m, g, bw_sat=bw, decode_target_s=0.0), trace).event_log == nx.run(plain, trace).event_log
    for cont in (None, [1.05, 0.3, -0.1]):
        cfg = nx.sim_config(m, g, bw_sat=bw, contention=cont, decode_target_s=0.03)
        r = nx.run(cfg, trace)
        ev, dec = run_port(cfg, trace)
        assert r.event_log == ev and r.decision_log == dec

        def mean_rp(log):
            rows = [ln.split("\t") for ln in log.splitlines() if ln and not ln.startswith("#")]
            return sum(int(x[4]) for x in rows) / len(rows)

        base = nx.run(nx.sim_config(m, g, bw_sat=bw, contention=cont), trace)
        assert mean_rp(r.decision_log) > mean_rp(base.decision_log)
    with pytest.raises(ValueError):
        nx.sim_config(m, g, decode_target_s=0.03)
