"""ORACLE / TEST INFRASTRUCTURE ONLY — pure-Python restatement of the
reference's intra-GPU engine (nexussim IntraGpuSim) with a pluggable latency
source.

Why it exists: the compiled reference (oracle/_ref) can only *predict*
latencies. Device-clock runs of the product are checked by "replay parity":
this port, fed the per-launch latencies the device measured, must reproduce
the device run's event and decision logs byte for byte. The port itself is
pinned by tests/test_oracle_port.py, which requires byte-identical logs with
the compiled reference in virtual-clock mode.

Every function cites the reference lines it restates. Python floats are IEEE
doubles and Python never fuses multiply-add, so keeping the reference's
operand order keeps results bit-identical.
"""
from __future__ import annotations

import math

INF = float("inf")
QKV, ATTN_PREFILL, ATTN_DECODE, OUT_PROJ, FFN = range(5)


# ---- opcost.cpp ------------------------------------------------------------

def _dense_bytes(m):  # split_dense_weights, opcost.cpp:56-67
    d, dff = float(m.hidden_dim), float(m.ffn_dim)
    qkv, out, ffn = 3.0 * d * d, d * d, 2.0 * d * dff
    tot = qkv + out + ffn
    b = float(m.num_layers) * float(m.weight_bytes_per_layer_dense)
    return b * (qkv / tot), b * (out / tot), b * (ffn / tot)


def _attn_w(m):  # opcost.cpp:69-72
    return float(m.num_layers) * float(m.weight_bytes_per_layer_attn)


def _dense(m, n, first):  # append_dense_ops, opcost.cpp:74-87
    d, dff, L = float(m.hidden_dim), float(m.ffn_dim), float(m.num_layers)
    wq, wo, wf = _dense_bytes(m)
    if first:
        return [(QKV, 6.0 * n * d * d * L, wq, 0.0, False)]
    return [(OUT_PROJ, 2.0 * n * d * d * L, wo, 0.0, False), (FFN, 4.0 * n * d * dff * L, wf, 0.0, False)]


def prefill_ops(m, chunks):  # prefill_batch_workloads, opcost.cpp:99-126
    n = fl = kv = 0.0
    d, L = float(m.hidden_dim), float(m.num_layers)
    for tok, ctx in chunks:
        n += float(tok)
        fl += 4.0 * float(tok) * float(ctx) * d * L
        kv += float(ctx) * float(m.kv_bytes_per_token)
    return _dense(m, n, True) + [(ATTN_PREFILL, fl, kv + _attn_w(m), kv, True)] + _dense(m, n, False)


def decode_ops(m, lens):  # decode_op_workloads, opcost.cpp:128-148
    fl = kv = 0.0
    d, L = float(m.hidden_dim), float(m.num_layers)
    for c in lens:
        fl += 4.0 * float(c) * d * L
        kv += float(c) * float(m.kv_bytes_per_token)
    n = float(len(lens))
    return _dense(m, n, True) + [(ATTN_DECODE, fl, kv + _attn_w(m), kv, True)] + _dense(m, n, False)


def mixed_ops(m, chunks, lens):  # mixed_batch_workloads, opcost.cpp:150-189
    if not chunks:
        return decode_ops(m, lens)
    if not lens:
        return prefill_ops(m, chunks)
    d, L = float(m.hidden_dim), float(m.num_layers)
    n = float(len(lens))
    pf = pk = 0.0
    for tok, ctx in chunks:
        n += float(tok)
        pf += 4.0 * float(tok) * float(ctx) * d * L
        pk += float(ctx) * float(m.kv_bytes_per_token)
    df = dk = 0.0
    for c in lens:
        df += 4.0 * float(c) * d * L
        dk += float(c) * float(m.kv_bytes_per_token)
    aw = _attn_w(m)
    return (_dense(m, n, True) + [(ATTN_PREFILL, pf, pk + aw, pk, True), (ATTN_DECODE, df, dk + aw, dk, True)]
            + _dense(m, n, False))


# ---- costmodel.cpp ---------------------------------------------------------

def _curve(prof, kind):
    return (prof.qkv_proj, prof.attn_prefill, prof.attn_decode, prof.attn_out_proj, prof.ffn)[kind]


def compute_latency(flops, share, c, peak):  # costmodel.cpp:8-14
    if share <= c.r_sat:
        return flops / (share * peak)
    return flops / (c.r_sat * peak) * (1.0 + c.lambda_ * (share - c.r_sat))


def breakdown(ops, share, gpu, prof, dbw=0.0, ext=None):  # costmodel.cpp:18-41
    """ext: per-op bw_sat list (the product's flagged nx_cost_ext), or None."""
    total = attn = 0.0
    for kind, fl, mem, kv, is_attn in ops:
        bw = dbw if (kind == ATTN_DECODE and dbw > 0) else gpu.peak_bandwidth
        if ext is not None and share < ext[kind]:
            bw = bw * (share / ext[kind])
        comp = compute_latency(fl, share, _curve(prof, kind), gpu.peak_compute)
        ms = mem / bw
        t = ms if comp < ms else comp
        total += t
        if is_attn and ms > comp:
            attn += t
    return total, attn


def contended(dops, share, pbd, pops, gpu, prof, ext=None, cont=None):  # costmodel.cpp:66-96
    if cont is not None:  # the product's flagged measured-slowdown form (model_cost.cpp decode_contended)
        t, a = breakdown(dops, share, gpu, prof, 0.0, ext)
        pp = 1.0 - share
        f = cont[0] + cont[1] * pp + cont[2] * pp * pp
        return t * f, a * f
    p = 0.0 if pbd[0] <= 0 else pbd[1] / pbd[0]
    m_p1 = m_p2 = m_d = 0.0
    for kind, fl, mem, kv, is_attn in pops:
        if is_attn:
            m_p1 += kv
        else:
            m_p2 += mem
    for kind, fl, mem, kv, is_attn in dops:
        if kind == ATTN_DECODE:
            m_d += kv
    B = gpu.peak_bandwidth
    bw = (m_d / (m_d + m_p1) * p * B + m_d / (m_d + m_p2) * (1.0 - p) * B) if m_d > 0 else B
    return breakdown(dops, share, gpu, prof, bw, ext)


# ---- schedulers.cpp --------------------------------------------------------

def _fill(ordered, budget):  # fill_prefill_budget, schedulers.cpp:13-32
    members, total = [], 0
    for rid, rem, _ in ordered:
        if total + rem <= budget:
            members.append((rid, rem))
            total += rem
        elif not members:
            members.append((rid, budget))
            total = budget
        else:
            break
    return members


def spf(queue, budget, gamma, now):  # schedulers.cpp:43-64
    keyed = sorted(((float(rem) - gamma * (now - arr), arr, rid, rem) for rid, rem, arr in queue))
    return _fill([(rid, rem, arr) for _, arr, rid, rem in keyed], budget)


def fcfs_prefill(queue, budget):  # schedulers.cpp:66-75
    return _fill(sorted(queue, key=lambda e: (e[2], e[0])), budget)


def fcfs_decode(cands, max_batch):  # schedulers.cpp:77-88
    return [(rid, 1) for _, rid in sorted((a, r) for r, a in cands)[:max(max_batch, 0)]]


def chunked_mixed(queue, cands, budget, max_batch, chunk):  # schedulers.cpp:90-125
    dec = sorted((a, r) for r, a in cands)
    take = min(len(dec), max(max_batch, 0), budget)
    members = [(rid, 1) for _, rid in dec[:take]]
    left = budget - take
    for rid, rem, arr in sorted(queue, key=lambda e: (e[2], e[0])):
        if left <= 0:
            break
        t = min(rem, chunk, left)
        if t <= 0:
            continue
        members.append((rid, t))
        left -= t
    return members


# ---- optimizer.cpp ---------------------------------------------------------

class Controller:
    def __init__(self, r_p, ctrl, target=None):
        """target: (decode_target_s, contention coefficients or None) of the
        product's flagged nx_cost_ext.decode_target_s, or None = reference."""
        self.r_p, self.r_d, self.last = r_p, 100 - r_p, r_p
        self.c = ctrl
        self.target = target

    def _adjust(self, target_prefill, other):  # adjust_partition, optimizer.cpp:22-61
        active, lat = other
        share_of = lambda s: s if target_prefill else 100 - s  # noqa: E731
        if not active:
            return share_of(99), False, 0
        slack = self.c.beta if target_prefill else self.c.alpha
        q = 1
        bound = slack * lat(100)
        tgt = self.target if target_prefill else None

        def fits(s):
            t = lat(100 - s)
            if not (t > bound):
                return True
            if tgt is None:
                return False
            p = s / 100.0
            f = 1.0 if tgt[1] is None else tgt[1][0] + tgt[1][1] * p + tgt[1][2] * p * p
            return not (t * f > tgt[0])

        s = min(max(self.r_p if target_prefill else self.r_d, 1), 99)
        while True:
            q += 1
            if fits(s):
                break
            if s == 1:
                return share_of(1), True, q
            s -= 1
        while s < 99:
            q += 1
            if not fits(s + 1):
                break
            s += 1
        return share_of(s), False, q

    def decide(self, used, cap, pre, dec):  # optimizer.cpp:63-99
        mode = "decode" if float(used) > self.c.kv_switch_fraction * float(cap) else "prefill"
        target_prefill = mode == "prefill"
        if not (pre if target_prefill else dec)[0]:
            return mode, self.r_p, self.r_p, False, 0
        cand, infeasible, q = self._adjust(target_prefill, dec if target_prefill else pre)
        if abs(cand - self.last) < self.c.delta_pp:
            return mode, cand, self.r_p, False, q
        self.r_p, self.r_d, self.last = cand, 100 - cand, cand
        return mode, cand, cand, True, q


# ---- simulator.cpp IntraGpuSim ----------------------------------------------

def _g(x):
    return "%.17g" % x


class _Lane:
    def __init__(self):
        self.busy, self.done_at, self.lat, self.r_p = False, 0.0, 0.0, 0
        self.dec, self.pre, self.ops, self.bd = [], [], [], (0.0, 0.0)


def run_port(cfg, trace, replay=None):
    """Runs the engine; returns (event_log, decision_log). `replay` replaces
    the cost-model latency of the k-th launch by replay[k]."""
    m, gpu, ctrl, prof, eng = cfg.model, cfg.gpu, cfg.ctrl, cfg.profile, cfg.engine
    ext = list(cfg.ext.bw_sat) if cfg.ext.enabled else None
    cont = list(cfg.ext.contention_c) if cfg.ext.enabled and cfg.ext.contention else None
    kind = eng.kind  # 0 nexus, 1 monolithic, 2 static
    dynamic, mono = kind == 0, kind == 1
    tgt = ((cfg.ext.decode_target_s, cont) if cfg.ext.enabled and cfg.ext.decode_target_s > 0 else None)
    ctl = Controller(eng.static_r_p if kind == 2 else 50, ctrl, tgt)
    kvb = m.kv_bytes_per_token
    R = {r.id: dict(id=r.id, arr=r.arrival_s, P=r.prompt_len, O=r.output_len, pf=0, dc=0, adm=False, fl=False)
         for r in trace}
    order = [r.id for r in trace]
    active, nxt = [], 0
    st = dict(clock=0.0, used=0, res=0, launches=0, events=0)
    ev, dec_log = [], ["# time_s\tkv_frac\tmode\tcandidate_r_p\tapplied_r_p\tswitched\tqueries\n"]
    P, D = _Lane(), _Lane()

    def log(lane, kindname, members, r_p, lat):
        mem = "-" if not members else ",".join(f"{i}:{t}:{e}" for i, t, e in members)
        ev.append(f"{_g(st['clock'])}\t{lane}\t{kindname}\t{mem}\t{r_p}\t{st['used']}\t{_g(lat)}\n")

    def cur_rp():
        return 100 if mono else ctl.r_p

    def pq():
        return [(i, R[i]["P"] - R[i]["pf"], R[i]["arr"]) for i in active
                if not R[i]["fl"] and R[i]["P"] - R[i]["pf"] > 0]

    def dq():
        return [(i, R[i]["arr"]) for i in active
                if not R[i]["fl"] and R[i]["pf"] == R[i]["P"] and R[i]["dc"] < R[i]["O"]]

    def admit(members, commit):  # filter_admissible, :223-244
        kept, res = [], st["res"]
        for rid, tok in members:
            r = R[rid]
            if not (r["pf"] < r["P"]) or r["adm"]:
                kept.append((rid, tok))
                continue
            need = (r["P"] + r["O"]) * kvb
            if res + need > gpu.kv_capacity_bytes:
                break
            res += need
            if commit:
                r["adm"] = True
                st["res"] = res
            kept.append((rid, tok))
        return kept

    def plan_prefill(q):
        return fcfs_prefill(q, ctrl.token_budget) if eng.prefill_policy == 1 else spf(
            q, ctrl.token_budget, ctrl.gamma, st["clock"])

    chunks = lambda ms: [(t, R[i]["pf"] + t) for i, t in ms]  # noqa: E731
    ctxs = lambda ms: [R[i]["P"] + R[i]["dc"] for i, _ in ms]  # noqa: E731

    def provisional_prefill():
        q = pq()
        if not q:
            return []
        kept = admit(plan_prefill(q), False)
        return prefill_ops(m, chunks(kept)) if kept else []

    def provisional_decode():
        q = dq()
        if not q:
            return []
        ms = fcfs_decode(q, ctrl.max_decode_batch)
        return decode_ops(m, ctxs(ms)) if ms else []

    def decide(launching_prefill, ops):  # controller_decide, :290-324
        pre = P.ops if P.busy else (ops if launching_prefill else provisional_prefill())
        dco = D.ops if D.busy else (provisional_decode() if launching_prefill else ops)
        pm = (bool(pre), lambda s: breakdown(pre, s / 100.0, gpu, prof, 0.0, ext)[0])
        dm = (bool(dco), lambda s: breakdown(dco, s / 100.0, gpu, prof, 0.0, ext)[0])
        mode, cand, applied, sw, q = ctl.decide(st["used"], gpu.kv_capacity_bytes, pm, dm)
        dec_log.append(f"{_g(st['clock'])}\t{_g(float(st['used']) / float(gpu.kv_capacity_bytes))}\t{mode}\t"
                       f"{cand}\t{applied}\t{int(sw)}\t{q}\n")
        return applied

    def begin(lane, lane_name, predicted):
        lat = replay[st["launches"]] if replay is not None else predicted
        st["launches"] += 1
        lane.busy, lane.lat, lane.done_at = True, lat, st["clock"] + lat
        for i, _ in lane.dec + lane.pre:
            R[i]["fl"] = True
        log(lane_name, "launch", [(i, t, 0) for i, t in lane.dec + lane.pre], lane.r_p, lat)

    def launch_decode():
        q = dq()
        if not q:
            return
        ms = fcfs_decode(q, ctrl.max_decode_batch)
        if not ms:
            return
        ops = decode_ops(m, ctxs(ms))
        r_p = decide(False, ops) if dynamic else ctl.r_p
        share = (100 - r_p) / 100.0
        D.bd = (contended(ops, share, P.bd, P.ops, gpu, prof, ext, cont) if P.busy
                else breakdown(ops, share, gpu, prof, 0.0, ext))
        D.dec, D.pre, D.ops, D.r_p = ms, [], ops, r_p
        begin(D, "decode", D.bd[0])

    def launch_prefill():
        q = pq()
        if not q:
            return
        kept = admit(plan_prefill(q), True)
        if not kept:
            return
        ops = prefill_ops(m, chunks(kept))
        r_p = decide(True, ops) if dynamic else ctl.r_p
        P.bd = breakdown(ops, r_p / 100.0, gpu, prof, 0.0, ext)
        P.pre, P.dec, P.ops, P.r_p = kept, [], ops, r_p
        begin(P, "prefill", P.bd[0])

    def launch_mixed():
        q, c = pq(), dq()
        if not q and not c:
            return
        ms = chunked_mixed(q, c, ctrl.token_budget, ctrl.max_decode_batch, ctrl.chunk_size)
        if not ms:
            return
        d = [x for x in ms if R[x[0]]["pf"] == R[x[0]]["P"]]
        p = admit([x for x in ms if R[x[0]]["pf"] != R[x[0]]["P"]], True)
        if not d and not p:
            return
        ops = mixed_ops(m, chunks(p), ctxs(d))
        P.bd = breakdown(ops, 1.0, gpu, prof, 0.0, ext)
        P.dec, P.pre, P.ops, P.r_p = d, p, ops, 100
        begin(P, "mixed", P.bd[0])

    def finish(rid, r_p):  # :483-492
        r = R[rid]
        r["done"] = True
        st["used"] -= (r["P"] + r["dc"]) * kvb
        st["res"] -= (r["P"] + r["O"]) * kvb
        r["adm"] = False
        active.remove(rid)
        log("-", "finish", [(rid, 0, 0)], r_p, 0.0)

    def complete(lane, name):  # :443-481
        evm, fin = [], []
        for rid, tok in lane.dec:
            r = R[rid]
            r["fl"] = False
            r["dc"] += 1
            st["used"] += kvb
            evm.append((rid, tok, 1))
            if r["dc"] == r["O"]:
                fin.append(rid)
        for rid, tok in lane.pre:
            r = R[rid]
            r["fl"] = False
            r["pf"] += tok
            st["used"] += tok * kvb
            e = 0
            if r["pf"] == r["P"]:
                e = 1
                r["dc"] = 1
                st["used"] += kvb
                if r["O"] == 1:
                    fin.append(rid)
            evm.append((rid, tok, e))
        lane.busy = False
        lane.dec, lane.pre = [], []
        log(name, "complete", evm, lane.r_p, lane.lat)
        for rid in fin:
            finish(rid, lane.r_p)

    while True:  # IntraGpuSim::run, :150-179
        if mono:
            if not P.busy:
                launch_mixed()
        else:
            if not D.busy:
                launch_decode()
            if not P.busy:
                launch_prefill()
        tp = P.done_at if P.busy else INF
        td = D.done_at if D.busy else INF
        ta = R[order[nxt]]["arr"] if nxt < len(order) else INF
        t = min(tp, td, ta)
        if t == INF:
            break
        if t > eng.timeout_sim_s:
            log("-", "timeout", [], cur_rp(), 0.0)
            break
        st["events"] += 1
        if st["events"] > eng.max_events:
            log("-", "timeout", [], cur_rp(), 0.0)
            break
        st["clock"] = t
        if P.busy and P.done_at == t:
            complete(P, "mixed" if mono else "prefill")
        elif D.busy and D.done_at == t:
            complete(D, "decode")
        else:
            rid = order[nxt]
            nxt += 1
            active.append(rid)
            log("-", "arrival", [(rid, 0, 0)], cur_rp(), 0.0)
    return "".join(ev), "".join(dec_log)
