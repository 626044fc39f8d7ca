"""SPEC.md known-answer examples, run against BOTH the compiled reference
oracle and the product library. Passing on the reference pins the oracle
(SURVEY §4 / §8(c)); passing on the product checks the restatement.
"""
import ctypes as C
import math

import pytest

from paper_2507_06608_b200 import _abi


class RefFacade:
    """Reference calls shaped like the product's Python API."""

    def __init__(self, ref):
        self.r = ref
        self.L = ref.lib()

    def derive(self, *a):
        return self.L.nxref_model_derive(*a)

    def compute_latency(self, flops, share, curve, peak):
        out = C.c_double()
        if self.L.nxref_compute_latency(flops, share, curve, peak, C.byref(out)):
            raise ValueError(self.L.nxref_last_error().decode())
        return out.value

    def effective_decode_bandwidth(self, *a):
        out = C.c_double()
        if self.L.nxref_effective_decode_bandwidth(*a, C.byref(out)):
            raise ValueError("bad")
        return out.value

    def _ops(self, fn, *args):
        out = (_abi.OpWorkload * 8)()
        n = C.c_size_t()
        if fn(*args, out, C.byref(n)):
            raise ValueError(self.L.nxref_last_error().decode())
        return list(out[: n.value])

    def prefill_batch_workloads(self, m, chunks):
        tok = (C.c_int64 * len(chunks))(*[c[0] for c in chunks])
        ctx = (C.c_int64 * len(chunks))(*[c[1] for c in chunks])
        return self._ops(self.L.nxref_prefill_batch_workloads, C.byref(m), tok, ctx, len(chunks))

    def decode_op_workloads(self, m, lens):
        arr = (C.c_int64 * max(1, len(lens)))(*lens)
        return self._ops(self.L.nxref_decode_op_workloads, C.byref(m), arr, len(lens))

    def select_mode(self, u, c, f):
        v = self.L.nxref_select_mode(u, c, f)
        if v < 0:
            raise ValueError("bad")
        return v

    def spf_schedule(self, queue, budget, gamma, now, skip=False):
        q = (_abi.PrefillEntry * len(queue))(*[_abi.PrefillEntry(*e) for e in queue])
        out = (_abi.BatchMember * 64)()
        n, tot = C.c_size_t(), C.c_int64()
        self.L.nxref_spf_schedule(q, len(queue), budget, gamma, now, int(skip), out, 64, C.byref(n), C.byref(tot))
        return [(m.id, m.tokens) for m in out[: n.value]], tot.value

    def fcfs_decode_schedule(self, active, maxb):
        a = (_abi.DecodeCandidate * len(active))(*[_abi.DecodeCandidate(*e) for e in active])
        out = (_abi.BatchMember * 64)()
        n, tot = C.c_size_t(), C.c_int64()
        self.L.nxref_fcfs_decode_schedule(a, len(active), maxb, out, 64, C.byref(n), C.byref(tot))
        return [(m.id, m.tokens) for m in out[: n.value]], tot.value

    def chunked_mixed_schedule(self, queue, active, budget, maxb, chunk):
        q = (_abi.PrefillEntry * max(1, len(queue)))(*[_abi.PrefillEntry(*e) for e in queue])
        a = (_abi.DecodeCandidate * max(1, len(active)))(*[_abi.DecodeCandidate(*e) for e in active])
        out = (_abi.BatchMember * 64)()
        n, tot = C.c_size_t(), C.c_int64()
        self.L.nxref_chunked_mixed_schedule(q, len(queue), a, len(active), budget, maxb, chunk, out, 64,
                                            C.byref(n), C.byref(tot))
        return [(m.id, m.tokens) for m in out[: n.value]], tot.value

    def adjust_partition(self, target, cur, pre, dec, cfg):
        from paper_2507_06608_b200 import _Phase
        p, d = _Phase(*pre), _Phase(*dec)
        out = _abi.AdjustOutcome()
        self.L.nxref_adjust_partition(target, C.byref(cur), C.byref(p.pm), C.byref(d.pm), C.byref(cfg),
                                      C.byref(out))
        return out


@pytest.fixture(params=["reference", "product"])
def api(request, nx):
    if request.param == "product":
        return nx
    from oracle import reference as r
    if not r.available():
        pytest.skip("reference oracle not built")
    return RefFacade(r)


def test_compute_latency_known_answers(api):
    # c=6e11, C=1e12, r_sat=0.6, lambda=0.2.
    curve = _abi.SaturationCurve(0.6, 0.2)
    assert api.compute_latency(6e11, 0.3, curve, 1e12) == pytest.approx(2.0, rel=1e-15)
    assert api.compute_latency(6e11, 0.6, curve, 1e12) == pytest.approx(1.0, rel=1e-15)
    assert api.compute_latency(6e11, 0.8, curve, 1e12) == pytest.approx(1.04, rel=1e-15)
    with pytest.raises(ValueError):
        api.compute_latency(1.0, 0.0, curve, 1e12)


def test_effective_decode_bandwidth_known_answers(api):
    # SPEC.md:197-199.
    assert api.effective_decode_bandwidth(0.5, 1.0, 1.0, 3.0, 100.0) == pytest.approx(37.5)
    assert api.effective_decode_bandwidth(0.3, 5.0, 0.0, 0.0, 100.0) == pytest.approx(100.0)
    assert api.effective_decode_bandwidth(0.0, 2.0, 7.0, 2.0, 100.0) == pytest.approx(50.0)
    with pytest.raises(ValueError):
        api.effective_decode_bandwidth(0.5, 0.0, 1.0, 1.0, 100.0)


def test_opcost_known_answers(api):
    # d=2, d_ff=8, 1 layer.
    m = api.derive(2, 8, 1, 1, 2)
    ops = api.prefill_batch_workloads(m, [(1, 1)])
    assert [o.kind for o in ops] == [0, 1, 3, 4]
    assert ops[0].flops == 24 and ops[1].flops == 8
    dec = api.decode_op_workloads(m, [1])
    assert dec[1].flops == 8 and dec[1].kind == _abi.NX_OP_ATTN_DECODE
    # kv bytes per token = 2*1*2*2 = 8; [100, 300] -> 400*8
    dec2 = api.decode_op_workloads(m, [100, 300])
    assert dec2[1].kv_bytes == 400 * 8
    with pytest.raises(ValueError):
        api.decode_op_workloads(m, [])


def test_select_mode_known_answers(api):
    # SPEC.md:262-264.
    assert api.select_mode(80, 100, 0.7) == _abi.NX_MODE_DECODE
    assert api.select_mode(0, 100, 0.7) == _abi.NX_MODE_PREFILL
    assert api.select_mode(70, 100, 0.7) == _abi.NX_MODE_PREFILL
    with pytest.raises(ValueError):
        api.select_mode(101, 100, 0.7)


def test_spf_known_answers(api):
    # A(100,0), B(10,0), C(2000, age 10), gamma=15 -> B, A, C.
    q = [(0, 100, 10.0), (1, 10, 10.0), (2, 2000, 0.0)]
    members, total = api.spf_schedule(q, 10_000, 15.0, 10.0)
    assert [m[0] for m in members] == [1, 0, 2]
    members, total = api.spf_schedule(q, 120, 15.0, 10.0)
    assert members == [(1, 10), (0, 100)] and total == 110
    # Oversized head takes a budget-sized chunk.
    members, total = api.spf_schedule([(7, 5000, 0.0)], 2048, 15.0, 0.0)
    assert members == [(7, 2048)] and total == 2048


def test_fcfs_decode_known_answers(api):
    # SPEC.md:337-339.
    act = [(i, float(10 - i)) for i in range(10)]
    members, total = api.fcfs_decode_schedule(act[:3], 8)
    assert total == 3
    members, total = api.fcfs_decode_schedule(act, 8)
    assert [m[0] for m in members] == [9, 8, 7, 6, 5, 4, 3, 2]
    members, _ = api.fcfs_decode_schedule([(5, 1.0), (2, 1.0), (9, 0.5)], 8)
    assert [m[0] for m in members] == [9, 2, 5]


def test_chunked_mixed_known_answers(api):
    # 4 decodes + one 2048-token chunk, budget 2052.
    members, total = api.chunked_mixed_schedule([(10, 5000, 0.0)], [(i, 1.0) for i in range(4)], 2052, 64,
                                                2048)
    assert total == 2052 and members[-1] == (10, 2048)
    members, total = api.chunked_mixed_schedule([], [(i, 1.0) for i in range(4)], 2052, 64, 2048)
    assert total == 4


def test_adjust_partition_known_answers(api, nx):
    # decode constraint holds for all R_p <= 63 and fails at 64.
    cfg = nx.lib().nx_controller_config_default()
    cur = _abi.PartitionState(50, 50, 50)
    dec_lat = lambda pct: 1.0 if pct >= 37 else 10.0  # noqa: E731
    out = api.adjust_partition(_abi.NX_PHASE_PREFILL, cur, (True, lambda p: 1.0), (True, dec_lat), cfg)
    assert (out.r_p, out.r_d, out.infeasible) == (63, 37, 0)
    # Exhaustive oracle: the answer is the largest feasible share.
    feasible = [r for r in range(1, 100) if dec_lat(100 - r) <= cfg.beta * dec_lat(100)]
    assert out.r_p == max(feasible)
    # Other phase empty -> 99 with zero queries.
    out = api.adjust_partition(_abi.NX_PHASE_PREFILL, cur, (True, lambda p: 1.0), (False, None), cfg)
    assert (out.r_p, out.queries) == (99, 0)
    # Infeasible everywhere -> (1, infeasible).
    out = api.adjust_partition(_abi.NX_PHASE_DECODE, cur, (True, lambda p: 5.0 if p < 100 else 1.0),
                               (True, lambda p: 1.0), cfg)
    assert out.r_d == 1 and out.infeasible == 1


def test_validate_config_known_answers(nx):
    m = nx.derive(256, 1024, 2, 4, 2)
    g = nx.gpu_preset("desk")
    c = nx.lib().nx_controller_config_default()
    p = nx.lib().nx_kernel_profile_default()
    assert nx.validate_config(m, g, c, p) == []
    c.alpha = 1.0
    assert any("controller.alpha" in e for e in nx.validate_config(m, g, c, p))
    c.alpha = 1.3
    p.ffn.r_sat = 0.0
    assert any("profile.ffn.r_sat" in e for e in nx.validate_config(m, g, c, p))
