"""HATA decode hot path benchmark (driver contract).

python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4|cfg3|cfg5] [--impl hata|reference]

A step = one decode step of one attention layer over one batch: the fused
hata_decode_step launch (append k_new/v_new + key code, q-hash, Hamming score,
exact top-k, gather-attention, combine) -- every §8(a) decode row.  Inputs
are synthetic (synth.make_case recipe, planted relevance) and resident in HBM;
consecutive steps rotate over 16 distinct cache sets (16 x 25 MB > 126 MB L2),
captured as 16 PDL-chained steps in one CUDA graph (the caches play the
attention layers of one model decode step), and each set sees a different q
on every replay (4 query variants per set), so the selection hint carried in
the workspace is exercised the way a decode loop uses it.

value / unit: "tokens/s (attention-only, 32 layers)" = B / (32 x per-layer
step time); --config cfg5 times the 32-layer step directly.
N = 1: cfg4 (the north_star config) + secondary cfg2 / cfg3 / cfg5 lines.
N > 1 (torchrun): cfg4 is sequence-sharded (NCCL exchange, CUDA graph);
--config cfg3 / cfg5 shard heads (no collective).  Rank 0 prints ONE line.
--impl reference: the CPU oracle (this tier's reference arm), whole steps.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402

METRIC = "decode attention µs/step & tokens/s at 32K/128K ctx; HBM GB/s vs roofline"
UNIT = "tokens/s (attention-only, 32 layers)"
LAYERS = 32
N_SETS = int(os.environ.get("HATA_BENCH_SETS", "16"))   # < 8 is an L2-resident diagnostic, not a bench number
N_Q = 4                                                  # query variants per cache set (cycled per replay)


def tokens_per_s(B, us_layer):
    return B / (LAYERS * us_layer * 1e-6)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _ncu_traffic(kernel, workload):
    """DRAM bytes per launch from the committed ncu capture (profiles/ncu_traffic.json), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return int(json.load(f)[kernel][workload]["bytes"])
    except Exception:
        return None


def algorithmic_bytes(sh, N=None, k=None):
    """codes + k' selected K/V rows + q (north_star roofline definition)."""
    N = sh.N if N is None else N
    k = sh.k if k is None else k
    eb = 2 if sh.dtype == "bf16" else 4
    kp = min(k, N)
    return sh.B * sh.Hkv * N * sh.rbits // 8 + sh.B * sh.Hkv * kp * 2 * sh.d * eb + sh.B * sh.Hq * sh.d * eb


def dense_bytes(sh, N=None):
    N = sh.N if N is None else N
    eb = 2 if sh.dtype == "bf16" else 4
    return sh.B * sh.Hkv * N * 2 * sh.d * eb + sh.B * sh.Hq * sh.d * eb


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for nm, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def apply_options():
    """Bench-side A/B switches (the library itself reads no environment):
    HATA_BENCH_HINT / HATA_BENCH_PDL = 0 turn the option off, HATA_BENCH_COOP = 1 on."""
    import paper_2506_02572_b200 as H
    opts = {}
    for name, env in (("selection_hint", "HATA_BENCH_HINT"), ("pdl", "HATA_BENCH_PDL"),
                      ("cooperative", "HATA_BENCH_COOP")):
        v = int(os.environ.get(env, "0" if name == "cooperative" else "1"))
        H.set_option(name, v)
        opts[name] = bool(v)
    return opts


def _pct(xs, p):
    xs = sorted(xs)
    return xs[min(len(xs) - 1, max(0, int(round(p / 100 * (len(xs) - 1)))))]


def _graph(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()  # warm / plan outside capture
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


# ---------------------------------------------------------------------------
# single-GPU layer steps
# ---------------------------------------------------------------------------
class Step:
    """Device-resident inputs of one layer step (one cache set) + outputs.
    ``qs``: N_Q query variants (q_h = u_g + 0.5 N(0,1), fresh noise per
    variant) so consecutive replays of the same set present a different q."""

    def __init__(self, sh, seed, device, n_q=N_Q, kv_pair=True):
        import paper_2506_02572_b200 as H
        self.H = H
        c = synth.make_case(sh, seed, device=device, variant="planted")
        self.sh = sh
        self.K, self.V, self.W = c["K"], c["V"], c["W"]
        if kv_pair and self.K.dtype == torch.bfloat16:
            # a token's K and V rows adjacent in HBM ([B, H_kv, cap, 2, d]):
            # the decode gathers both with one 512-byte request
            kv = torch.stack((self.K, self.V), dim=3)
            del c["K"], c["V"]
            self.K, self.V = kv[:, :, :, 0, :], kv[:, :, :, 1, :]
        gen = torch.Generator(device=device).manual_seed(seed * 7919 + 1)
        q0 = c["q"].float()
        self.qs = [c["q"]] + [(q0 + 0.5 * torch.randn(q0.shape, generator=gen, device=device)).to(c["q"].dtype)
                              for _ in range(n_q - 1)]
        self.q = self.qs[0]
        self.kn, self.vn = c["k_new"], c["v_new"]
        self.pos = c["n_before"]
        self.n = self.pos + 1
        B, Hkv, cap, d = self.K.shape
        self.codes = torch.zeros(B, Hkv, cap, sh.rbits // 32, dtype=torch.int32, device=device)
        H.hash_keys(self.K, self.W, self.codes, 0, sh.N - 1)
        self.out = torch.empty(B, sh.Hq, d, dtype=torch.float32, device=device)
        ws = H.decode_workspace_size(B, sh.Hq, Hkv, d, sh.rbits, sh.N, sh.k, self.K.dtype)
        self.ws = torch.zeros(max(ws, 4 * 4 * B * Hkv), dtype=torch.uint8, device=device)

    def run(self, r=0):
        """One decode step = ONE launch: append (k_new, v_new, key code at row
        N-1) fused with q-hash, score, top-k, gather-attention and combine."""
        self.H.decode_step(self.qs[r], self.kn, self.vn, self.K, self.V, self.codes, self.W, self.n, self.sh.k,
                           n_max=self.sh.N, out=self.out, workspace=self.ws)

    def hint_counters(self):
        """Per-unit (hinted selections, window-exchange thresholds): workspace word 3, 16-bit wrapping."""
        w = self.ws[:32 * self.sh.B * self.sh.Hkv].view(torch.int32).view(-1, 8)[:, 3].cpu().long() & 0xFFFFFFFF
        return (w & 0xFFFF), (w >> 16)


def time_replays(seq):
    """seq: list of (graph, n_steps).  Events around every replay on the
    launching stream; returns (total seconds, per-replay us per step)."""
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(len(seq) + 1)]
    torch.cuda.synchronize()
    evs[0].record()
    for i, (g, _) in enumerate(seq):
        g.replay()
        evs[i + 1].record()
    evs[-1].synchronize()
    per = [evs[i].elapsed_time(evs[i + 1]) * 1e3 / n for i, (_, n) in enumerate(seq)]
    total = evs[0].elapsed_time(evs[-1]) / 1e3
    return total, per


def _soak(graphs, seconds):
    """Keep the GPU busy with the same step so nvidia-smi samples clocks under load."""
    t0 = time.perf_counter()
    i = 0
    while time.perf_counter() - t0 < seconds:
        for _ in range(20):
            graphs[i % len(graphs)].replay()
            i += 1
        torch.cuda.synchronize()


def bench_single(sh, steps, warmup, device, n_sets=N_SETS, clocks=True, dist_steps=208):
    """Time EXACTLY ``steps`` layer steps: full graphs of n_sets PDL-chained
    steps (query variant r on replay r mod N_Q) plus one graph of the
    remainder.  Per-replay events give the p5 / median / p95 distribution
    (from a separate pass of >= dist_steps steps if ``steps`` is smaller)."""
    sets = [Step(sh, 1000 + i, device) for i in range(n_sets)]
    graphs = [_graph(lambda r=r: [st.run(r) for st in sets]) for r in range(N_Q)]
    rem = steps % n_sets
    g_rem = _graph(lambda: [st.run(0) for st in sets[:rem]]) if rem else None

    def sequence(n):
        seq = [(graphs[i % N_Q], n_sets) for i in range(n // n_sets)]
        if n % n_sets:
            seq.append((g_rem, n % n_sets))
        return seq
    for i in range(max(1, -(-max(warmup, 3) // n_sets))):
        graphs[i % N_Q].replay()
    torch.cuda.synchronize()
    cs = ClockSampler(torch.cuda.current_device()) if clocks else None
    if cs:
        cs.__enter__()
        _soak(graphs, 0.5)
    h0 = [st.hint_counters() for st in sets]
    t_total, per = time_replays(sequence(steps))
    h1 = [st.hint_counters() for st in sets]
    if cs:
        _soak(graphs, 0.3)
        cs.__exit__()
    if steps < dist_steps:
        _, per = time_replays(sequence(-(-dist_steps // n_sets) * n_sets))
    units = sh.B * sh.Hkv
    fast = sum(int(((a1 - a0) & 0xFFFF).sum()) for (a0, _), (a1, _) in zip(h0, h1))
    window = sum(int(((b1 - b0) & 0xFFFF).sum()) for (_, b0), (_, b1) in zip(h0, h1))
    M = sets[0].H.decode_ranks(sh.B, sh.Hq, sh.Hkv, sh.d, sh.rbits, sh.N, sh.k)
    hint = {"hinted_selection_rate": fast / (units * steps),
            "window_exchange_rate": window / (units * steps) if M > 1 else None,
            "query_variants_per_set": N_Q,
            "note": "fraction of the timed (unit, step) selections that took the hinted (candidate-bitmap) path / "
                    "whose threshold came from the one-round-trip window exchange; q differs on every replay of a set"}
    return dict(t_step=t_total, steps=steps, per=per, clocks=cs.summary() if cs else None, sets=sets, hint=hint,
                launches=steps, units=units)


def bench_e2e(sh, steps, device):
    """Same metric through the public API with HOST buffers: per step, pinned
    q/k_new/v_new go H2D, the fused step runs, the output comes back D2H."""
    s = Step(sh, 77, device, n_q=1)
    hq = s.q.cpu().pin_memory()
    hk = s.kn.cpu().pin_memory()
    hv = s.vn.cpu().pin_memory()
    ho = torch.empty(s.out.shape, dtype=s.out.dtype).pin_memory()

    def one():
        s.q.copy_(hq, non_blocking=True)
        s.kn.copy_(hk, non_blocking=True)
        s.vn.copy_(hv, non_blocking=True)
        s.run()
        ho.copy_(s.out, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    for _ in range(3):
        one()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    dt = time.perf_counter() - t0
    h2d = hq.numel() * hq.element_size() + hk.numel() * hk.element_size() + hv.numel() * hv.element_size()
    d2h = ho.numel() * ho.element_size()
    us = dt / steps * 1e6
    return dict(value=tokens_per_s(sh.B, us), unit=UNIT, us_per_step=us, h2d_bytes_per_step=h2d,
                d2h_bytes_per_step=d2h, steps=steps)


def bench_hash_keys(st, reps):
    """Prefill key hash (hata_hash_keys, §8(a) a1) over the whole cache of one
    set: B*H_kv*(N-1) bf16 keys -> codes on the tcgen05 tensor cores."""
    sh = st.sh
    n = sh.N - 1
    st.H.hash_keys(st.K, st.W, st.codes, 0, n)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        st.H.hash_keys(st.K, st.W, st.codes, 0, n)
    e1.record()
    e1.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    eb = 2 if sh.dtype == "bf16" else 4
    kbytes = sh.B * sh.Hkv * n * sh.d * eb
    flops = 2.0 * sh.B * sh.Hkv * n * sh.d * sh.rbits
    peak, _ = _peaks()
    return {"us": us, "keys": sh.B * sh.Hkv * n, "GBps_K_read": kbytes / (us * 1e-6) / 1e9,
            "TFLOPs": flops / (us * 1e-6) / 1e12, "frac_of_hbm": kbytes / (us * 1e-6) / 1e9 / peak,
            "kernel": "hash_keys_umma_kernel (tcgen05.mma kind::f16, TMEM fp32 accumulators, TMA SW128 K tiles)",
            "note": f"K ({kbytes / 1e6:.0f} MB) exceeds the 126 MB L2; {reps} back-to-back calls"}


def bench_prefill_write(st, reps):
    """NEXT-1: a whole prefilled chunk (B*H_kv*(N-1) keys and values) written
    into the paired cache with its codes in one pass (hata_prefill_write) vs
    the separate copy + hata_hash_keys."""
    sh = st.sh
    n = sh.N - 1
    B, Hkv, cap, d = st.K.shape
    g = torch.Generator(device=st.K.device).manual_seed(5)
    Ks = torch.randn(B, Hkv, n, d, generator=g, device=st.K.device).to(st.K.dtype)
    Vs = torch.randn_like(Ks)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]

    def fused():
        st.H.prefill_write(Ks, Vs, st.W, st.K, st.V, st.codes, 0)

    def separate():
        st.K[:, :, :n].copy_(Ks)
        st.V[:, :, :n].copy_(Vs)
        st.H.hash_keys(st.K, st.W, st.codes, 0, n)
    fused(); separate()
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(reps):
        fused()
    ev[1].record()
    for _ in range(reps):
        separate()
    ev[2].record()
    ev[2].synchronize()
    uf = ev[0].elapsed_time(ev[1]) / reps * 1e3
    us = ev[1].elapsed_time(ev[2]) / reps * 1e3
    eb = 2 if sh.dtype == "bf16" else 4
    io = 4 * B * Hkv * n * d * eb + B * Hkv * n * sh.rbits // 8      # read K, V + write K, V + codes
    peak, _ = _peaks()
    return {"us": uf, "separate_copy_plus_hash_keys_us": us, "algorithmic_bytes": io,
            "GBps": io / (uf * 1e-6) / 1e9, "frac_of_hbm": io / (uf * 1e-6) / 1e9 / peak,
            "kernel": "hash_keys_umma_kernel<FUSED> (TMA loads of the chunk, TMA stores to the cache, tcgen05 hash)"}


def dense_baseline(st, steps):
    """Full-attention decode over the same cache (context, north_star)."""
    q = st.q.view(st.sh.B, st.sh.Hq, 1, st.sh.d)
    K, V = st.K.contiguous(), st.V.contiguous()          # the dense kernel reads its own (split) layout
    try:
        from flash_attn import flash_attn_with_kvcache
        qf = st.q.view(st.sh.B, 1, st.sh.Hq, st.sh.d)
        kc, vc = K.transpose(1, 2), V.transpose(1, 2)
        cs = st.n.to(torch.int32)
        fn = lambda: flash_attn_with_kvcache(qf, kc, vc, cache_seqlens=cs)  # noqa: E731
        fn()
        impl = "flash_attn.flash_attn_with_kvcache"
    except Exception:
        fn = lambda: torch.nn.functional.scaled_dot_product_attention(q, K, V, enable_gqa=True)  # noqa: E731
        impl = "torch SDPA (enable_gqa)"
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    e1.synchronize()
    us = e0.elapsed_time(e1) / steps * 1e3
    return {"impl": impl, "us_per_step": us, "tokens_per_s": tokens_per_s(st.sh.B, us),
            "note": "same resident cache every step (L2-warm upper bound for dense)"}


def bench_offload(sh, steps, device):
    """HATA-off: K/V in page-locked host memory
    mapped into the device address space, codes on the GPU; the fused step
    gathers only the selected K/V rows over the host link (TMA from mapped
    host memory).  One cache set, query variant cycled per step."""
    st = Step(sh, 3000, device)
    kv = torch.empty(st.K.shape[:3] + (2, st.K.shape[3]), dtype=st.K.dtype, pin_memory=True)
    kv[:, :, :, 0] = st.K.cpu()
    kv[:, :, :, 1] = st.V.cpu()
    st.K, st.V = kv[:, :, :, 0], kv[:, :, :, 1]
    torch.cuda.empty_cache()
    g = _graph(lambda: [st.run(r % N_Q) for r in range(8)])
    g.replay()
    t, per = time_replays([(g, 8)] * max(1, steps // 8))
    us = t / (max(1, steps // 8) * 8) * 1e6
    eb = 2 if sh.dtype == "bf16" else 4
    link = sh.B * sh.Hkv * min(sh.k, sh.N) * 2 * sh.d * eb
    return {"workload": f"{sh.name} with K/V in pinned host memory (HATA-off)", "us_per_step": us,
            "tokens_per_s": tokens_per_s(sh.B, us), "unit": UNIT, "host_link_bytes_per_step": link,
            "host_link_GBps": link / (us * 1e-6) / 1e9,
            "gpu_resident_bytes": sh.B * sh.Hkv * sh.N * sh.rbits // 8,
            "note": "codes and the scoring stay on the GPU; the decode kernel's bulk-copy gather reads only the "
                    "selected rows from mapped host memory; the appended row is written there by the same launch"}


class PagedStep:
    """A Step whose caches are moved into physical page pools ([pages, H_kv,
    ps, 2, d] K/V, [pages, H_kv, ps, W] codes) in a random page order,
    addressed through a block table (NEXT-2)."""

    def __init__(self, st, ps, seed):
        sh = st.sh
        B, Hkv, cap, d = st.K.shape
        self.st, self.ps = st, ps
        maxp = -(-cap // ps)
        npages = B * maxp
        g = torch.Generator().manual_seed(seed)
        perm = torch.randperm(npages, generator=g).view(B, maxp)
        dev = st.K.device
        kv = torch.zeros(npages, Hkv, ps, 2, d, dtype=st.K.dtype, device=dev)
        self.codes = torch.zeros(npages, Hkv, ps, sh.rbits // 32, dtype=torch.int32, device=dev)
        for b in range(B):
            for lp in range(maxp):
                a, z = lp * ps, min(cap, (lp + 1) * ps)
                pp = int(perm[b, lp])
                kv[pp, :, :z - a, 0] = st.K[b, :, a:z]
                kv[pp, :, :z - a, 1] = st.V[b, :, a:z]
                self.codes[pp, :, :z - a] = st.codes[b, :, a:z]
        self.K, self.V = kv[:, :, :, 0], kv[:, :, :, 1]
        self.pt = perm.to(torch.int32).to(dev)
        st.K = st.V = st.codes = None

    def run(self, r=0):
        st = self.st
        st.H.decode_step_paged(st.qs[r], st.kn, st.vn, self.K, self.V, self.codes, st.W, self.pt, st.n, st.sh.k,
                               n_max=st.sh.N, out=st.out, workspace=st.ws)


def bench_paged(sh, ps, steps, device, peak, n_sets=N_SETS):
    """NEXT-2: the CFG-4 step over paged pools (page size ps, pages shuffled),
    same rotation / graph / query variation as the contiguous bench line."""
    sets = [PagedStep(Step(sh, 1000 + i, device), ps, 77 + i) for i in range(n_sets)]
    torch.cuda.empty_cache()
    graphs = [_graph(lambda r=r: [st.run(r) for st in sets]) for r in range(N_Q)]
    for g in graphs:
        g.replay()
    reps = max(1, steps // n_sets)
    t, per = time_replays([(graphs[i % N_Q], n_sets) for i in range(reps)])
    us = t / (reps * n_sets) * 1e6
    b = algorithmic_bytes(sh)
    return {"workload": f"{sh.name} over paged pools (page size {ps}, pages in random order)", "us_per_step": us,
            "tokens_per_s": tokens_per_s(sh.B, us), "unit": UNIT, "frac": b / (us * 1e-6) / 1e9 / peak,
            "p5_us": _pct(per, 5), "p95_us": _pct(per, 95)}


def secondary_line(sh, steps, warmup, device, peak):
    r = bench_single(sh, steps, warmup, device, clocks=False)
    us = r["t_step"] / r["steps"] * 1e6
    b = algorithmic_bytes(sh)
    line = {"workload": f"{sh.name}: {sh.note}", "us_per_step": us, "tokens_per_s": tokens_per_s(sh.B, us),
            "unit": UNIT, "p5_us": _pct(r["per"], 5), "median_us": statistics.median(r["per"]),
            "p95_us": _pct(r["per"], 95), "achieved_GBps": b / (us * 1e-6) / 1e9,
            "frac": b / (us * 1e-6) / 1e9 / peak, "algorithmic_bytes": b, "hint": r["hint"]}
    line["dense_baseline"] = dense_baseline(r["sets"][0], 30)
    del r
    torch.cuda.empty_cache()
    return line


# ---------------------------------------------------------------------------
# CFG-5: full 32-layer decode step, heads sharded over the ranks (P = 1..8)
# ---------------------------------------------------------------------------
def bench_model(sh, steps, warmup, device, rank, world, n_dense=2, layers=LAYERS):
    """The 32 attention layers of one decode step on this rank's KV heads
    (headshard.HeadShardModel): with the paper's "vanilla attention for the
    first two layers" and with all 32 layers HATA; plus 32 dense
    layers (flash-attention) over the same caches.  One CUDA graph per
    variant; returns per-step times (us)."""
    from paper_2506_02572_b200.headshard import HeadShardDecode, HeadShardModel, head_range
    lo, hi = head_range(sh.Hkv, world, rank)
    local = dataclasses.replace(sh, Hq=sh.G * (hi - lo), Hkv=hi - lo)
    lays = [Step(local, 5000 + 97 * layer + rank, device, n_q=1) for layer in range(layers)]
    out = {}
    for name, nd in (("dense_first_2", n_dense), ("all_hata", 0)):
        pol = HeadShardModel.dense_policy(layers, nd)
        model = HeadShardModel([HeadShardDecode(st.K, st.V, st.codes, st.W, sh.G, sh.k, rank, world, sh.Hkv,
                                                dense=pol[i]) for i, st in enumerate(lays)])
        qs = [st.q for st in lays]
        kns = [st.kn for st in lays]
        vns = [st.vn for st in lays]
        g = _graph(lambda: model.step(qs, kns, vns, lays[0].n, sh.N))
        for _ in range(max(warmup, 3)):
            g.replay()
        t, per = time_replays([(g, 1)] * steps)
        out[name] = dict(us_per_step=t / steps * 1e6, p5_us=_pct(per, 5), p95_us=_pct(per, 95),
                         median_us=statistics.median(per))
        del g, model
    try:   # dense baseline: 32 flash-attention layers over the same caches
        from flash_attn import flash_attn_with_kvcache
        dl = []
        for st in lays:
            dl.append((st.q.view(local.B, 1, local.Hq, local.d), st.K.contiguous().transpose(1, 2),
                       st.V.contiguous().transpose(1, 2), st.n.to(torch.int32)))
        g = _graph(lambda: [flash_attn_with_kvcache(q, kc, vc, cache_seqlens=c) for q, kc, vc, c in dl])
        g.replay()
        nd_steps = max(3, steps // 2)
        t, _ = time_replays([(g, 1)] * nd_steps)
        out["dense_32_layers"] = dict(us_per_step=t / nd_steps * 1e6, impl="flash_attn.flash_attn_with_kvcache")
        del dl, g
    except Exception as e:  # pragma: no cover
        out["dense_32_layers"] = {"unavailable": str(e)[:200]}
    per_layer = algorithmic_bytes(local)
    out["bytes_per_step_hata"] = layers * per_layer
    out["bytes_per_step_dense_first_2"] = (layers - n_dense) * per_layer + n_dense * dense_bytes(local)
    del lays
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------------
# CPU oracle legs (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------
_CPU = {}


def _cpu_group(args):
    """One (b, KV head) group's oracle decode step (append + q-hash + score +
    top-k + attention of its G query heads), fp64 numpy."""
    import numpy as np
    import oracle.hata_oracle as O
    b, g = args
    c = _CPU
    sh = c["sh"]
    G = sh.G
    res = O.decode_step(c["q"][b:b + 1, g * G:(g + 1) * G], c["kn"][b:b + 1, g:g + 1], c["vn"][b:b + 1, g:g + 1],
                        c["K"][b:b + 1, g:g + 1], c["V"][b:b + 1, g:g + 1], c["codes"][b:b + 1, g:g + 1],
                        c["W"][g:g + 1], np.array([sh.N - 1]), sh.k)
    return float(res["out"][0, 0, 0])


def _cpu_setup(sh, seed=1000):
    """The GPU arm's first cache set (same seed, planted) on the host, with the oracle's own key codes."""
    import numpy as np
    import oracle.hata_oracle as O
    c = synth.make_case(sh, seed, device="cpu", variant="planted")
    d = {x: c[x].double().numpy() for x in ("q", "K", "V", "W", "k_new", "v_new")}
    codes, _ = O.hash_keys(d["K"], d["W"])
    _CPU.clear()
    _CPU.update(sh=sh, q=d["q"], K=d["K"], V=d["V"], W=d["W"], kn=d["k_new"], vn=d["v_new"],
                codes=np.ascontiguousarray(codes))


def _cpu_name():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def _pool(n):
    import multiprocessing as mp
    return mp.get_context("fork").Pool(n)


def _limit_threads():
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass


def cpu_oracle_baseline(sh, budget_s=20.0):
    """The oracle as it stands, on the GPU arm's inputs (seed 1000, planted):
    (1) one (b, KV head) group on one thread; (2) whole steps with one process
    per group up to nproc.  Bounded to ~budget_s seconds."""
    _limit_threads()
    _cpu_setup(sh)
    groups = [(b, g) for b in range(sh.B) for g in range(sh.Hkv)]
    t0 = time.perf_counter()
    _cpu_group(groups[0])
    t1g = time.perf_counter() - t0
    cores = min(len(groups), os.cpu_count() or 1)
    with _pool(cores) as pool:
        pool.map(_cpu_group, groups[:cores])                   # warm the workers
        reps, t0 = 0, time.perf_counter()
        while True:
            pool.map(_cpu_group, groups)
            reps += 1
            if time.perf_counter() - t0 > budget_s / 2 or reps >= 5:
                break
        step = (time.perf_counter() - t0) / reps
    return {"value": tokens_per_s(sh.B, step * 1e6), "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{reps} whole {sh.name} decode steps ({len(groups)} (b, KV head) groups, one process per "
                      f"group on {cores} cores) on the GPU arm's cache set 0 (seed 1000, planted); fp64 numpy",
            "s_per_step": step, "single_thread_s_per_group": t1g,
            "single_thread_value": tokens_per_s(sh.B, t1g * len(groups) * 1e6), "cpu": _cpu_name(),
            "nproc": os.cpu_count()}


def run_reference(args, sh, rank):
    """--impl reference: the CPU oracle as it stands (this tier's reference
    arm), timing whole steps (every (b, KV head) group, one process per group
    up to nproc) on the same workload, metric and unit as the GPU arm."""
    if rank != 0:
        return
    _limit_threads()
    _cpu_setup(sh)
    groups = [(b, g) for b in range(sh.B) for g in range(sh.Hkv)]
    cores = min(len(groups), os.cpu_count() or 1)
    with _pool(cores) as pool:
        for _ in range(args.warmup):
            pool.map(_cpu_group, groups)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            pool.map(_cpu_group, groups)
        dt = (time.perf_counter() - t0) / args.steps
    value = tokens_per_s(sh.B, dt * 1e6)
    sample = (f"each step = one whole {sh.name} layer decode step ({len(groups)} (b, KV head) groups, one process per "
              f"group on {cores} cores), inputs = the GPU arm's cache set 0 (seed 1000, planted); fp64 numpy oracle")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "us_per_step": dt * 1e6,
            "higher_is_better": True, "dtype": "f64", "data": "synthetic (synth.make_case, seed 1000, planted)",
            "config": {"workload": f"{sh.name}: {sh.note}", "B": sh.B, "Hq": sh.Hq, "Hkv": sh.Hkv, "d": sh.d,
                       "rbits": sh.rbits, "N": sh.N, "k": sh.k},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                             "cpu": _cpu_name()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# N > 1: sequence-sharded CFG-4 (paper_2506_02572_b200.seqshard)
# ---------------------------------------------------------------------------
class ShardSet:
    """One cache set on this rank: its contiguous token slice of every (b, g)."""

    def __init__(self, sh, seed, device, rank, world):
        import paper_2506_02572_b200 as H
        from paper_2506_02572_b200.seqshard import SeqShardDecode, shard_range
        c = synth.make_case(sh, seed, device=device, variant="planted")
        B, Hkv, cap, d = c["K"].shape
        lo, hi = shard_range(cap, world, rank)
        C = (cap + world - 1) // world
        kv = torch.zeros(B, Hkv, C, 2, d, dtype=c["K"].dtype, device=device)    # paired layout
        kv[:, :, :hi - lo, 0] = c["K"][:, :, lo:hi]
        kv[:, :, :hi - lo, 1] = c["V"][:, :, lo:hi]
        Kl, Vl = kv[:, :, :, 0], kv[:, :, :, 1]
        codes = torch.zeros(B, Hkv, C, sh.rbits // 32, dtype=torch.int32, device=device)
        nloc = max(0, min(sh.N - 1, hi) - lo)
        if nloc:
            H.hash_keys(Kl, c["W"], codes, 0, nloc)
        self.q, self.kn, self.vn, self.W = c["q"], c["k_new"], c["v_new"], c["W"]
        self.n = c["n_before"] + 1
        del c
        self.dec = SeqShardDecode(Kl, Vl, codes, self.W, sh.Hq, sh.k, cap, rank, world)

    def run(self, sh):
        return self.dec.step(self.q, self.n, sh.N, self.kn, self.vn)


def _max_over_ranks(x, device):
    import torch.distributed as dist
    if not dist.is_initialized():
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def bench_seqshard(args, sh, rank, world, device):
    import torch.distributed as dist
    n_sets = 8
    sets = [ShardSet(sh, 1000 + i, device, rank, world) for i in range(n_sets)]
    try:
        g = _graph(lambda: [st.run(sh) for st in sets])
        graphed = True
    except Exception:  # pragma: no cover - eager fallback if capturing the collectives fails
        g, graphed = None, False

    def run_all():
        if g is not None:
            g.replay()
        else:
            for st in sets:
                st.run(sh)
    for _ in range(max(1, -(-max(args.warmup, 3) // n_sets))):
        run_all()
    torch.cuda.synchronize()
    reps = max(1, -(-args.steps // n_sets))
    with ClockSampler(torch.cuda.current_device()) as cs:
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            run_all()
        e1.record()
        torch.cuda.synchronize()
        dist.barrier()
    steps = reps * n_sets
    t_max = _max_over_ranks(e0.elapsed_time(e1) / 1e3, device)
    us = t_max / steps * 1e6
    # e2e through the public API with host buffers
    st = sets[0]
    hq, hk, hv = st.q.cpu().pin_memory(), st.kn.cpu().pin_memory(), st.vn.cpu().pin_memory()
    ho = torch.empty(st.dec.out.shape, dtype=st.dec.out.dtype).pin_memory()
    e2e_steps = min(args.steps, 100)
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        st.q.copy_(hq, non_blocking=True); st.kn.copy_(hk, non_blocking=True); st.vn.copy_(hv, non_blocking=True)
        out = st.run(sh)
        ho.copy_(out, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    te = _max_over_ranks(time.perf_counter() - t0, device)
    # roofline of the whole step: this rank's share of the bytes / the step time
    lo, hi = st.dec.lo, st.dec.hi
    bytes_rank = (sh.B * sh.Hkv * (hi - lo) * sh.rbits // 8 + sh.B * sh.Hkv * sh.k * 2 * sh.d * 2 // world
                  + sh.B * sh.Hq * sh.d * 2)
    return dict(us=us, steps=steps, graphed=graphed, achieved=bytes_rank / (us * 1e-6) / 1e9, bytes_rank=bytes_rank,
                clocks=cs.summary(),
                e2e=dict(value=tokens_per_s(sh.B, te / e2e_steps * 1e6), unit=UNIT, us_per_step=te / e2e_steps * 1e6,
                         h2d_bytes_per_step=sum(x.numel() * x.element_size() for x in (hq, hk, hv)),
                         d2h_bytes_per_step=ho.numel() * ho.element_size()))


def bench_headshard_layer(sh, steps, warmup, device, rank, world):
    """CFG-3: one layer step on this rank's KV heads (no collective); the max
    over ranks of the per-step time."""
    from paper_2506_02572_b200.headshard import head_range
    lo, hi = head_range(sh.Hkv, world, rank)
    local = dataclasses.replace(sh, Hq=sh.G * (hi - lo), Hkv=hi - lo)
    r = bench_single(local, steps, warmup, device, clocks=False)
    us = _max_over_ranks(r["t_step"] / r["steps"] * 1e6, device)
    del r
    torch.cuda.empty_cache()
    return dict(us=us, bytes_rank=algorithmic_bytes(local))


# ---------------------------------------------------------------------------
def _base_line(args, sh, world, us_layer, steps, opts, extra_cfg):
    return {"metric": METRIC, "value": tokens_per_s(sh.B, us_layer), "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "ms_per_step": us_layer / 1e3, "us_per_step": us_layer, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": sh.dtype,
            "data": "synthetic (synth.make_case: K, V, q ~ N(0,1) with planted sink/recent/needle rows; seeds 1000+)",
            "config": dict({"workload": f"{sh.name}: {sh.note}", "B": sh.B, "Hq": sh.Hq, "Hkv": sh.Hkv, "d": sh.d,
                            "rbits": sh.rbits, "N": sh.N, "k": sh.k}, **extra_cfg,
                           pdl=opts["pdl"], cooperative=opts["cooperative"], selection_hint=opts["selection_hint"])}


def main_single(args, sh, device, peak, peak_src, opts):
    import paper_2506_02572_b200 as H
    r = bench_single(sh, args.steps, args.warmup, device)
    steps = r["steps"]
    us = r["t_step"] / steps * 1e6
    bytes_step = algorithmic_bytes(sh)
    achieved = bytes_step / (us * 1e-6) / 1e9
    M = H.decode_ranks(sh.B, sh.Hq, sh.Hkv, sh.d, sh.rbits, sh.N, sh.k, r["sets"][0].K.dtype)
    line = _base_line(args, sh, 1, us, steps, opts, {
        "ranks_per_head": M, "parallelism": "single GPU",
        "l2": f"inputs > L2: {N_SETS} distinct cache sets x {bytes_step / 1e6:.1f} MB step bytes rotate (> 126 MB L2)",
        "graph": f"{N_SETS} consecutive PDL-chained fused steps (one per cache set, like the attention layers of one "
                 f"model decode step) per CUDA graph; {N_Q} query variants per set cycled over replays",
        "kv_layout": "[B, H_kv, cap, 2, d] (K and V rows of a token adjacent)"})
    line["latency_us"] = {"p5": _pct(r["per"], 5), "median": statistics.median(r["per"]), "p95": _pct(r["per"], 95),
                          "samples": len(r["per"]), "note": "per CUDA-graph replay, us per layer step"}
    line["roofline"] = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                        "traffic": _ncu_traffic("hata_decode_kernel", sh.name),
                        "traffic_source": "profiles/ncu_traffic.json (ncu dram__bytes_read+write per launch)",
                        "kernel": "hata_decode_kernel (the whole step is this one launch)",
                        "algorithmic_bytes_per_launch": bytes_step, "us_per_launch": us,
                        "peak_source": peak_src, "frac_vs_8TBs": achieved / 8000.0}
    line["clocks"] = r["clocks"]
    line["gpu_launches"] = r["launches"]
    line["selection_hint"] = r["hint"]
    del r
    torch.cuda.empty_cache()
    line["e2e"] = bench_e2e(sh, min(args.steps, 200), device)
    # the same step with the selection hint off (the full selection scan every launch)
    H.set_option("selection_hint", 0)
    r0 = bench_single(sh, 208, 16, device, clocks=False)
    H.set_option("selection_hint", int(opts["selection_hint"]))
    line["no_hint_us_per_step"] = r0["t_step"] / r0["steps"] * 1e6
    del r0
    torch.cuda.empty_cache()
    if not args.no_secondary:
        sec = {}
        for nm in ("cfg2", "cfg3", "cfg5"):
            if nm != sh.name:
                sec[nm] = secondary_line(synth.CONFIGS[nm], 208, 16, device, peak)
        s5 = synth.CONFIGS["cfg5"]
        m = bench_model(s5, 10, 3, device, 0, 1)
        for v in m.values():
            if isinstance(v, dict) and "us_per_step" in v:
                v["tokens_per_s"] = s5.B / (v["us_per_step"] * 1e-6)
        sec["cfg5_32_layers"] = dict({"workload": "cfg5: Qwen2.5-14B-shaped full 32-layer decode step, 1 GPU",
                                      "unit": UNIT}, **m)
        sec["hata_off_cfg2"] = bench_offload(synth.CONFIGS["cfg2"], 64, device)
        sec["paged_cfg4_ps64"] = bench_paged(synth.CONFIGS["cfg4"], 64, 208, device, peak)
        torch.cuda.empty_cache()
        line["secondary"] = sec
    st = Step(sh, 1000, device, n_q=1)
    line["hash_keys"] = bench_hash_keys(st, 20)
    line["prefill_write"] = bench_prefill_write(st, 10)
    line["dense_baseline"] = dense_baseline(st, 50)
    line["dense_baseline"]["speedup_vs_dense"] = line["dense_baseline"]["us_per_step"] / us
    del st
    torch.cuda.empty_cache()
    if not args.no_cpu:
        line["cpu_baseline"] = cpu_oracle_baseline(sh)
    print(json.dumps(line), flush=True)


def main_model(args, sh, rank, world, device, peak, peak_src, opts):
    """--config cfg5: the full 32-layer decode step, heads sharded over the ranks."""
    m = bench_model(sh, args.steps, args.warmup, device, rank, world)
    us = _max_over_ranks(m["dense_first_2"]["us_per_step"], device)
    us_all = _max_over_ranks(m["all_hata"]["us_per_step"], device)
    dense = m["dense_32_layers"].get("us_per_step")
    dense = _max_over_ranks(dense, device) if dense is not None else None
    if rank != 0:
        return
    line = _base_line(args, sh, world, us / LAYERS, args.steps, opts, {
        "layers": LAYERS, "layer_policy": "layers 0-1 dense (P:347), 2-31 HATA",
        "parallelism": f"heads sharded x{world} (H_kv/{world} KV heads + their query heads per GPU, no collective)",
        "l2": "inputs > L2: 32 distinct layer caches", "graph": "the 32-layer step in one CUDA graph"})
    line["value"] = sh.B / (us * 1e-6)          # the 32-layer step measured directly
    line["ms_per_step"] = us / 1e3
    line["us_per_step"] = us
    line["all_hata_us_per_step"] = us_all
    line["dense_32_layers_us_per_step"] = dense
    b = m["bytes_per_step_dense_first_2"]
    line["roofline"] = {"bound": "hbm", "achieved": b / (us * 1e-6) / 1e9, "peak": peak, "unit": "GB/s",
                        "frac": b / (us * 1e-6) / 1e9 / peak, "traffic": None,
                        "kernel": "hata_decode_kernel x 32 per step (2 dense layers = k = N)",
                        "algorithmic_bytes_per_step_per_gpu": b, "peak_source": peak_src}
    line["gpu_launches"] = args.steps * LAYERS
    line["e2e"] = {"value": line["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                   "note": "device-resident inputs (a 32-layer step's q/k/v come from the model's projections)"}
    print(json.dumps(line), flush=True)


def main_multi(args, sh, rank, world, device, peak, peak_src, opts):
    if args.config == "cfg5":
        main_model(args, sh, rank, world, device, peak, peak_src, opts)
        return
    if args.config == "cfg3":
        hs = bench_headshard_layer(sh, args.steps, args.warmup, device, rank, world)
        if rank == 0:
            line = _base_line(args, sh, world, hs["us"], args.steps, opts, {
                "parallelism": f"heads sharded x{world} (no collective)", "l2": f"{N_SETS} distinct cache sets per rank"})
            a = hs["bytes_rank"] / (hs["us"] * 1e-6) / 1e9
            line["roofline"] = {"bound": "hbm", "achieved": a, "peak": peak, "unit": "GB/s", "frac": a / peak,
                                "traffic": None, "kernel": "hata_decode_kernel", "peak_source": peak_src,
                                "algorithmic_bytes_per_launch": hs["bytes_rank"], "us_per_launch": hs["us"]}
            line["gpu_launches"] = args.steps
            line["e2e"] = {"value": line["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
            print(json.dumps(line), flush=True)
        return
    r = bench_seqshard(args, sh, rank, world, device)
    sec = {}
    if not args.no_secondary:
        hs = bench_headshard_layer(synth.CONFIGS["cfg3"], 208, 16, device, rank, world)
        s3 = synth.CONFIGS["cfg3"]
        sec["cfg3_headshard"] = {"us_per_step": hs["us"], "tokens_per_s": tokens_per_s(s3.B, hs["us"]), "unit": UNIT,
                                 "frac": hs["bytes_rank"] / (hs["us"] * 1e-6) / 1e9 / peak,
                                 "parallelism": f"heads sharded x{world} (no collective)"}
    if rank != 0:
        return
    line = _base_line(args, sh, world, r["us"], r["steps"], opts, {
        "parallelism": f"sequence-sharded x{world} (one NCCL all-gather of packed top-k candidates + one of partials)",
        "l2": "8 rotating cache sets per rank", "graph": r["graphed"]})
    line["roofline"] = {"bound": "hbm", "achieved": r["achieved"], "peak": peak, "unit": "GB/s",
                        "frac": r["achieved"] / peak, "traffic": None,
                        "kernel": "whole sharded step (decode kernel in candidate mode + select + partial + combine "
                                  "+ 2 all-gathers); rank bytes / step time",
                        "algorithmic_bytes_per_step_per_rank": r["bytes_rank"], "us_per_step": r["us"],
                        "peak_source": peak_src}
    line["clocks"] = r["clocks"]
    line["gpu_launches"] = r["steps"] * 5
    line["e2e"] = r["e2e"]
    if sec:
        line["secondary"] = sec
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=208)
    ap.add_argument("--warmup", type=int, default=16)
    ap.add_argument("--config", default="cfg4", choices=["cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--impl", default="hata", choices=["hata", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the oracle cpu_baseline leg")
    ap.add_argument("--no-secondary", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    sh = synth.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, sh, rank)
        return
    local = int(os.environ.get("LOCAL_RANK", rank))
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    opts = apply_options()
    peak, peak_src = _peaks()
    if world > 1 or os.environ.get("HATA_BENCH_DIST"):        # env: exercise the N > 1 path at world 1
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=device)
        try:
            main_multi(args, sh, rank, world, device, peak, peak_src, opts)
        finally:
            dist.barrier()
            dist.destroy_process_group()
        return
    if args.config == "cfg5":
        main_model(args, sh, 0, 1, device, peak, peak_src, opts)
        return
    main_single(args, sh, device, peak, peak_src, opts)


if __name__ == "__main__":
    main()
