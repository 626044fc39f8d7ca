"""Forward parity at the geometries the bench publishes (VERDICT r1 "close the
parity gaps"): two-layer models with the exact per-layer shapes of

  * Llama-3.1-8B   (d 4096, 32 q / 8 kv heads -> G = 4, ffn 14336, theta 5e5),
  * Qwen2.5-14B    (d 5120, 40 q / 8 kv heads -> G = 5, QKV bias, theta 1e6,
                    RMSNorm eps 1e-6),
  * Llama-3.1-70B  (d 8192, 64 q / 8 kv heads -> G = 8, ffn 28672),

presets from device.ARCH_PRESETS (reference model presets presets.cpp:13-19),
vocab reduced to 8192 so the fp32 oracle stays small (the lm_head kernel path
is the same one: vocab rows are 128-row packed tiles either way).

Each geometry runs the two kernel paths the bench uses:
  * prefill: one 2048-token chunk of four 512-token prompts on the CTA-pair
    tcgen05 GEMMs (gemm_tc2, RoPE + paged-KV epilogue) and the prefill
    attention, on the 116-SM prefill layout (share 79);
  * decode: a 64-row decode batch (ragged contexts) on the 32-SM decode layout
    through gemm_decode + the fold kernels + split-KV decode attention.
Logits of every sampled row are compared with oracle/llama_fp32.py on the same
bf16 weights; tolerance as tests/test_gpu_model.py (3e-2 * max|ref| per row,
greedy token equal where the fp32 top-2 margin exceeds 4x that bound).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LOGIT_TOL = 3e-2
GEOMETRIES = ["llama3-8b", "qwen2.5-14b", "llama3-70b"]


def _check(dev_logits, ref_logits, dev_tokens):
    assert len(dev_logits) == len(ref_logits) == len(dev_tokens)
    for row, ref, tok in zip(dev_logits, ref_logits, dev_tokens):
        err = np.abs(row - ref).max()
        assert err <= LOGIT_TOL * np.abs(ref).max(), (err, np.abs(ref).max())
        top2 = np.sort(ref)[-2:]
        if top2[1] - top2[0] > 4 * LOGIT_TOL * np.abs(ref).max():
            assert tok == int(np.argmax(ref))


@pytest.fixture(scope="module", params=GEOMETRIES)
def geo(request):
    from paper_2507_06608_b200 import device as D
    from oracle.llama_fp32 import LlamaFP32
    a = D.arch_preset(request.param, n_layers=2, vocab=8192)
    dev = D.Device(a, num_pages=4096, seed=21, max_prefill_tokens=2048 + 128, max_decode_batch=128)
    yield request.param, dev, LlamaFP32(dev)
    dev.close()


def test_prefill_2048_chunk_pair_gemm(geo):
    name, dev, ref = geo
    rng = np.random.default_rng(31)
    prompts = [rng.integers(0, dev.arch.vocab, 512).tolist() for _ in range(4)]
    members = [dict(tokens=p, start=0, pages=list(range(40 * i, 40 * i + 32))[::-1])
               for i, p in enumerate(prompts)]
    out, logits, _ = dev.forward(members, lane=0, sm_pct=79, want_logits=True)
    want = np.stack([ref.logits(np.array(p))[-1] for p in prompts])
    _check(logits, want, out)


def test_prefix_chunk_then_64_row_decode(geo):
    """A second prefill chunk over a paged prefix, then one 64-row decode
    batch with ragged contexts (17..400 tokens) on the decode layout."""
    name, dev, ref = geo
    rng = np.random.default_rng(32)
    long_prompt = rng.integers(0, dev.arch.vocab, 700).tolist()
    lp_pages = list(range(3000, 3000 + 48))
    dev.forward([dict(tokens=long_prompt[:512], start=0, pages=lp_pages, sample=False)], lane=0, sm_pct=79)
    out, logits, _ = dev.forward([dict(tokens=long_prompt[512:], start=512, pages=lp_pages)], lane=0,
                                 sm_pct=79, want_logits=True)
    _check(logits, ref.logits(np.array(long_prompt))[-1:], out)

    lens = [int(x) for x in rng.integers(17, 400, 63)]
    prompts = [rng.integers(0, dev.arch.vocab, n).tolist() for n in lens]
    page_sets = [list(range(200 + 40 * i, 200 + 40 * i + 26)) for i in range(63)]
    # prefill them in token-budgeted batches (the decode rows need a KV prefix)
    batch, used = [], 0
    for p, pg in zip(prompts, page_sets):
        if used + len(p) > 2048:
            dev.forward(batch, lane=0, sm_pct=79)
            batch, used = [], 0
        batch.append(dict(tokens=p, start=0, pages=pg, sample=False))
        used += len(p)
    if batch:
        dev.forward(batch, lane=0, sm_pct=79)
    seqs = [p + [int(rng.integers(0, dev.arch.vocab))] for p in prompts] + [long_prompt + [out[0]]]
    pages = page_sets + [lp_pages]
    dmem = [dict(tokens=[s[-1]], start=len(s) - 1, pages=pg) for s, pg in zip(seqs, pages)]
    out2, logits2, _ = dev.forward(dmem, lane=1, sm_pct=21, want_logits=True)
    want2 = np.stack([ref.logits(np.array(s))[-1] for s in seqs])
    _check(logits2, want2, out2)


def test_long_among_short_decode_full_gpu():
    """one 9.6K-token context among 100 short ones on the
    full 148-SM GPU, 8B geometry (8 kv heads). The split-KV partials are
    indexed (item, unit)-compactly, so the workspace bound no longer scales
    with n_items x the worst item's piece count and the launch must succeed.
    The 100 short rows share one prompt and next token (each still owns its
    own pages and decode item), so one oracle recompute checks them all."""
    from paper_2507_06608_b200 import device as D
    from oracle.llama_fp32 import LlamaFP32
    a = D.arch_preset("llama3-8b", n_layers=1, vocab=2048)
    dev = D.Device(a, num_pages=8192, seed=23, max_prefill_tokens=2048 + 128, max_decode_batch=128)
    try:
        ref = LlamaFP32(dev)
        rng = np.random.default_rng(33)
        short = rng.integers(0, a.vocab, 600).tolist()
        long_p = rng.integers(0, a.vocab, 9600).tolist()
        short_pages = [list(range(40 * i, 40 * i + 38)) for i in range(100)]
        long_pages = list(range(4200, 4200 + 601))
        for c0 in range(0, 9600, 2048):
            dev.forward([dict(tokens=long_p[c0:c0 + 2048], start=c0, pages=long_pages, sample=False)],
                        lane=0, sm_pct=100)
        for i in range(0, 100, 3):
            dev.forward([dict(tokens=short, start=0, pages=short_pages[j], sample=False)
                         for j in range(i, min(100, i + 3))], lane=0, sm_pct=100)
        nxt = 7
        dmem = [dict(tokens=[nxt], start=600, pages=pg) for pg in short_pages]
        dmem.append(dict(tokens=[nxt], start=9600, pages=long_pages))
        out, logits, _ = dev.forward(dmem, lane=1, sm_pct=100, want_logits=True)
        want_s = ref.logits(np.array(short + [nxt]))[-1]
        want_l = ref.logits(np.array(long_p + [nxt]))[-1]
        _check(logits, np.stack([want_s] * 100 + [want_l]), out)
    finally:
        dev.close()


def test_8b_device_clock_replay_parity(nx):
    """Full Llama-3.1-8B geometry (32 layers, random bf16 weights) served on
    the device clock with the bench's configuration (calibrated profile,
    share-limited bandwidth extension, beta 2, gamma 5000, max decode batch
    128) for 120 ShareGPT-shaped requests at 64 rps; the measured per-launch
    latencies replayed through the pinned Python port (oracle/engine_port.py,
    itself byte-pinned to the compiled reference) reproduce the run's event
    and decision logs byte for byte, and the block tables match the page
    model."""
    import json
    import os
    from paper_2507_06608_b200 import device as D
    from oracle.engine_port import run_port
    from oracle.kvpages_model import replay_pages
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    base = os.path.join(repo, "profiles", "b200_llama3_8b")
    cal = json.load(open(base + ".json"))
    prof, _ = nx.parse_kernel_profile(open(base + ".calib").read())
    num_pages = 40000
    dev = D.Device(D.arch_preset("llama3-8b"), num_pages=num_pages, max_prefill_tokens=2048 + 128,
                   max_decode_batch=128, seed=3)
    try:
        m = nx.derive(4096, 14336, 32, 32, 2)
        g = nx.gpu_spec(148, cal["gpu_spec"]["peak_compute"], cal["gpu_spec"]["peak_bandwidth"],
                        (num_pages - 4096) * 16 * 2 * 32 * 4096 * 2)
        ctrl = nx.lib().nx_controller_config_default()
        ctrl.max_decode_batch, ctrl.beta, ctrl.gamma = 128, 2.0, 5000.0
        trace = nx.workload_trace("sharegpt", 64.0, 120, 11)
        kw = dict(ctrl=ctrl, profile=prof, bw_sat=cal["bw_sat"])
        cfg = nx.sim_config(m, g, clock_mode=nx.NX_CLOCK_DEVICE, **kw)
        eng = nx.Engine(cfg, device=dev)
        eng.submit_trace(trace)
        eng.run()
        lat = eng.launch_latencies()
        assert len(lat) > 100 and all(x > 0 for x in lat)
        rcfg = nx.sim_config(m, g, clock_mode=nx.NX_CLOCK_REPLAY, **kw)
        ev, dec = run_port(rcfg, trace, replay=lat)
        assert ev == eng.event_log()
        assert dec == eng.decision_log()
        log, live = replay_pages(eng.event_log(), {r.id: r.prompt_len for r in trace}, 16, num_pages)
        assert eng.page_log() == log and not live
        for q in eng.requests():
            assert len(eng.tokens(q.id)) == q.prompt_len + q.output_len
    finally:
        dev.close()
