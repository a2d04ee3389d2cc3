#!/usr/bin/env python
"""Benchmark of the B200 UNIQUE sparse decode step (BASELINE.json metric).

Workload: BASELINE.json configs[2] -- Llama-3.1-8B attention shape, global batch 32,
128K context, 32 q / 8 kv heads, d=128, page 16, k = 2048 tokens (128 pages), bf16 KV pool,
exact f32 page stats (+ their bf16 mirror for bounded scoring).  One step = one decode token
per sequence through the full hot path: append the new K/V row (K1b, tail-page stats
recomputed exactly) -> lam*||q|| -> score every page (K2b, bounded over the bf16 mirror) ->
select the top-k pages (K3, exact keys resolved where the bounds straddle the cut) ->
split-KV sparse attention over them (K4), replayed as a CUDA graph.

Multi-GPU (`--gpus N`; self-launches N ranks under torch.distributed.run when WORLD_SIZE is
unset): the 256 (sequence, kv-head) units of the global batch are split over the ranks
(paper_2605_27740_b200/shard.py: whole sequences per rank), every rank holding only its
units' KV pages and stats -- "scaling": "strong", no data-path collective.  The optional
NCCL output all-gather is timed beside the line, and a weak-scaling measurement (32
sequences per rank) is reported in "weak".  The workload is generated per unit from the
global seed, so every N sees identical data.

Prints ONE JSON line on rank 0.  `--impl reference` times the reference's CPU path (its own
compiled kernels from oracle/_ref, else the bit-identical oracle port) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "sparse decode attn tokens/s @128K ctx (batch 32, k=2048 tokens, 32q/8kv d128 page16)"
UNIT = "tokens/s"
SEED = 1234


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--batch", type=int, default=32, help="global batch (sequences)")
    ap.add_argument("--ctx", type=int, default=131072)
    ap.add_argument("--q-heads", type=int, default=32)
    ap.add_argument("--kv-heads", type=int, default=8)
    ap.add_argument("--head-dim", type=int, default=128)
    ap.add_argument("--page", type=int, default=16)
    ap.add_argument("--budget", type=int, default=2048, help="token budget k*S")
    ap.add_argument("--stats-dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--no-mirror", action="store_true", help="exact f32-means scoring (no bounds)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline sample budget")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--no-weak", action="store_true", help="skip the weak-scaling leg (N > 1)")
    ap.add_argument("--no-parity", action="store_true", help="skip the in-bench oracle check")
    ap.add_argument("--dump-out", default=None,
                    help="save the gathered outputs of one eager step (tests: N ranks == 1 rank)")
    ap.add_argument("--profile", action="store_true",
                    help="few eager steps, no graph/cpu/dense (for ncu launch lists)")
    return ap.parse_args(argv)


# ---------------------------------------------------------------------------
# clocks sampler (NVML) during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        0x0000000000000002: "applications_clocks_setting",
        0x0000000000000004: "sw_power_cap",
        0x0000000000000008: "hw_slowdown",
        0x0000000000000020: "sw_thermal_slowdown",
        0x0000000000000040: "hw_thermal_slowdown",
        0x0000000000000080: "hw_power_brake_slowdown",
    }

    def __init__(self, index: int):
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # pragma: no cover - no NVML
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        return {
            "sm_mhz": statistics.median(self.samples) if self.samples else None,
            "sm_max_mhz": self.max_mhz,
            "reasons": sorted(self.reasons),
            "samples": len(self.samples),
        }


def host_cores() -> int:
    """Every host core this process may run on (torchrun exports OMP_NUM_THREADS=1; the
    CPU baseline sets its OpenMP team explicitly to this)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


# ---------------------------------------------------------------------------
# algorithmic bytes
# ---------------------------------------------------------------------------
def step_bytes(U, G, D, P, kp, S, e_kv, e_stats, N_tok):
    """SURVEY 8(d) per step; e_stats = the page-mean element size read by the scorer."""
    score = U * (P * D * e_stats + 4 * P + G * D * e_kv + 2 * P)
    topk = U * (2 * P + 8 * kp)  # keys read + page-table entries read + ids written
    T = kp * S
    attn = U * (2 * T * D * e_kv + G * D * e_kv + 4 * kp) + U * G * D * 4
    append = U * (S * D * e_kv + 3 * D * e_kv + 4)
    dense = 2 * U * N_tok * D * e_kv + U * G * D * 4
    return dict(score=score, topk=topk, attend=attn, append=append, dense=dense)


def bounded_score_moved(U, G, D, P):
    """Bytes the bounded scorer actually moves: bf16 mirror, std + err, q, norms, two keys."""
    return U * (P * D * 2 + 8 * P + G * D * 2 + 64 + 4 * P) + U * (P // 32) * 2


# ---------------------------------------------------------------------------
# workload: generated per unit from the global seed (identical data for every N)
# ---------------------------------------------------------------------------
def _unit_gen(device, seed, u):
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed * 1_000_003 + u)
    return g


def build_cache(args, device, seed, units=None, spare_tokens=None, mirror=None):
    """PagedKvCache holding the global units ``units`` (default: all of args.batch sequences)
    with args.ctx tokens each, K/V ~ N(0,1) rounded to bf16 (harness/workload.py:60-98)."""
    import torch

    import paper_2605_27740_b200 as pt

    H, D, S = args.kv_heads, args.head_dim, args.page
    units = list(range(args.batch * H)) if units is None else list(units)
    Ul = len(units)
    Hl, Bl = (H, Ul // H) if Ul % H == 0 else (1, Ul)
    if spare_tokens is None:
        spare_tokens = (args.warmup + args.steps) * 3 + 256
    P_cap = -(-(args.ctx + spare_tokens) // S)
    layout = pt.CacheLayout(num_kv_heads=Hl, head_dim=D, page_size=S, max_pages=Ul * P_cap)
    sdt = torch.float32 if args.stats_dtype == "f32" else torch.bfloat16
    if mirror is None:
        mirror = not getattr(args, "no_mirror", False) and args.stats_dtype == "f32"
    cache = pt.PagedKvCache(layout, batch=Bl, dtype=torch.bfloat16, stats_dtype=sdt,
                            max_pages_per_head=P_cap, device=device, mirror=mirror)
    for kk, vv in unit_rows(args, device, seed, units):
        cache.extend_units(kk, vv)
        del kk, vv
    torch.cuda.synchronize()
    return cache


def unit_rows(args, device, seed, units, chunk=8192):
    """The workload's K/V rows of the given global units, in chunks of ``chunk`` tokens:
    yields bf16 [len(units), n, D] pairs.  Unit u draws from its own generator (seeded from
    the global seed and u), so a rank holding units [u0, u1) sees exactly the rows the
    unsharded run gives those units."""
    import torch

    D = args.head_dim
    gens = [_unit_gen(device, seed, u) for u in units]
    done = 0
    while done < args.ctx:
        n = min(chunk, args.ctx - done)
        kk = torch.empty(len(gens), n, D, device=device, dtype=torch.bfloat16)
        vv = torch.empty(len(gens), n, D, device=device, dtype=torch.bfloat16)
        for i, g in enumerate(gens):
            kk[i] = torch.randn(n, D, generator=g, device=device, dtype=torch.float32)
            vv[i] = torch.randn(n, D, generator=g, device=device, dtype=torch.float32)
        yield kk, vv
        done += n


def step_inputs(args, device, NQ=4, seed=SEED):
    """NQ rotating query sets [U*G, D] and the new K/V rows [U, D] of the GLOBAL batch (bf16);
    ranks slice their shard's rows."""
    import torch

    H, D = args.kv_heads, args.head_dim
    G = args.q_heads // H
    U = args.batch * H
    g = torch.Generator(device=device)
    g.manual_seed(seed + 7)
    qs = [torch.randn(U * G, D, generator=g, device=device).to(torch.bfloat16) for _ in range(NQ)]
    kn = torch.randn(U, D, generator=g, device=device).to(torch.bfloat16)
    vn = torch.randn(U, D, generator=g, device=device).to(torch.bfloat16)
    return qs, kn, vn


def _sample_arrays(cache, q_bf16, args, seqs=2):
    """Host copies (f32) of the first ``seqs`` sequences of a cache: q, compacted K/V pool,
    page table, lengths, page stats."""
    import torch

    import paper_2605_27740_b200._device as dev

    H, D, S = cache.layout.num_kv_heads, args.head_dim, args.page
    G = args.q_heads // args.kv_heads
    kp = -(-args.budget // S)
    nu = min(cache.num_units, seqs * args.kv_heads)
    units = list(range(nu))
    tab = cache.page_table[:nu].cpu().numpy()
    seq = cache.seq_lens[:nu].cpu().numpy()
    P = int(-(-seq.max() // S))
    pids = np.unique(tab[:, :P][tab[:, :P] >= 0])
    remap = -np.ones(cache.layout.max_pages, dtype=np.int64)
    remap[pids] = np.arange(pids.size)
    idx = torch.from_numpy(pids).to(cache.device)
    kpool = cache.k_pool[idx].to(torch.float32).cpu().numpy()
    vpool = cache.v_pool[idx].to(torch.float32).cpu().numpy()
    tab2 = np.where(tab >= 0, remap[np.maximum(tab, 0)], -1).astype(np.int32)
    means = dev.untile_means(cache.means, cache.num_units, cache.Pmax, D, cache.stats_dtype)
    means = means[:nu].to(torch.float32).cpu().numpy()
    stds = cache.stds[:nu].cpu().numpy()
    q = q_bf16.reshape(cache.num_units, G, D)[:nu].to(torch.float32).cpu().numpy()
    return dict(seqs=nu // args.kv_heads, units=units, q=q, kpool=kpool, vpool=vpool, tab=tab2,
                seq=seq, means=means, stds=stds, kp=kp, S=S, D=D, H=args.kv_heads, pids=pids)


def cpu_baseline(a, budget_s, nthreads):
    """Reference decode_step (oracle port, bit-identical to the compiled backend) on host
    cores over a bounded sample (``a`` from _sample_arrays) of the same workload."""
    from oracle import oracle as O

    reps, t0 = 0, time.perf_counter()
    res = None
    while True:
        res = O.decode_units(a["q"], a["kpool"], a["vpool"], a["tab"], a["seq"], a["means"],
                             a["stds"], a["kp"], 0.5, 1.0 / math.sqrt(a["D"]), a["S"],
                             nthreads=nthreads)
        reps += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = (time.perf_counter() - t0) / reps
    return {
        "value": a["seqs"] / dt,
        "unit": UNIT,
        "cores": nthreads,
        "kind": "port",
        "sample": f"{a['seqs']} sequences x {a['H']} kv-heads (128K ctx, k={a['kp']} pages, bf16 "
                  f"values upcast to f32) per rep, {reps} reps in {time.perf_counter() - t0:.1f}s; "
                  "oracle/pagetopk_oracle.c (bit-identical to _kernels_cy), OpenMP over units",
        "_res": res,
    }


# ---------------------------------------------------------------------------
# reference arm: the reference's CPU path on the host cores
# ---------------------------------------------------------------------------
def reference_workload(args, seqs=2, seed=SEED):
    """A host-only sample of the workload (no GPU, no repo kernels): ``seqs`` sequences,
    K/V/q ~ N(0,1) rounded to bf16 (torch CPU generator), a contiguous page table with one
    spare page per unit for the per-step append, page stats by the oracle's restatement of
    kvcache.py:59-71 (bit-identical to the reference's numpy)."""
    import torch

    from oracle import oracle as O

    H, D, S = args.kv_heads, args.head_dim, args.page
    G = args.q_heads // H
    U = seqs * H
    n = args.ctx
    P = -(-n // S)
    Pc = -(-(n + 1) // S) + 1
    g = torch.Generator()
    g.manual_seed(seed)

    def bf16(*shape):
        return torch.randn(*shape, generator=g).to(torch.bfloat16).to(torch.float32).numpy()

    kpool = np.zeros((U * Pc, S, D), np.float32)
    vpool = np.zeros((U * Pc, S, D), np.float32)
    for u in range(U):
        kpool[u * Pc: u * Pc + P].reshape(-1, D)[:n] = bf16(n, D)
        vpool[u * Pc: u * Pc + P].reshape(-1, D)[:n] = bf16(n, D)
    tab = (np.arange(U)[:, None] * Pc + np.arange(Pc)[None, :]).astype(np.int32)
    seq = np.full(U, n, np.int32)
    means, stds = O.build_stats(kpool, tab, seq, S)
    q = bf16(U, G, D)
    kn, vn = bf16(U, D), bf16(U, D)
    return dict(q=q, kpool=kpool, vpool=vpool, tab=tab, seq=seq, means=means, stds=stds, kn=kn,
                vn=vn, kp=-(-args.budget // S), S=S, D=D, H=H, seqs=seqs)


def run_reference_arm(args, world, config):
    """Each step: per (sequence, kv-head) unit, append the step's K/V row to the tail page
    and refresh its stats (kvcache.py:185-208 + compute_page_stats, numpy), then the
    reference decode_step (attention.py:110-147) on the reference's own compiled kernels
    (oracle/_ref, from pkg/src/pagetopk/_kernels_cy.pyx), units over one forked process per
    host core; without oracle/_ref the oracle port (OpenMP over units) instead."""
    from oracle import oracle as O
    from oracle import ref_arm

    ncores = host_cores()
    w = reference_workload(args)
    steps, warm = max(1, args.steps), max(0, args.warmup)
    if ref_arm.so_path() is not None:
        arm = ref_arm.RefArm(w["q"], w["kpool"], w["vpool"], w["tab"], w["seq"], w["means"],
                             w["stds"], w["kp"], 0.5, w["S"], ncores, k_new=w["kn"], v_new=w["vn"])
        try:
            for _ in range(warm):
                res = arm.run()
            t0 = time.perf_counter()
            for _ in range(steps):
                res = arm.run()
            dt = (time.perf_counter() - t0) / steps
        finally:
            arm.close()
        # cross-check against the port on the post-append cache (seq n + 1)
        kp_, vp_, means, stds, seq = ref_arm.appended(w)
        port = O.decode_units(w["q"], kp_, vp_, w["tab"], seq, means, stds, w["kp"], 0.5,
                              1.0 / math.sqrt(w["D"]), w["S"])
        for u, (phys, out, lse) in enumerate(res):
            if set(phys.tolist()) != set(port["sel"][u][: port["n_sel"][u]].tolist()):
                raise RuntimeError(f"reference kernels and oracle port disagree on unit {u}")
            np.testing.assert_allclose(out, port["out"][u], rtol=1e-5, atol=1e-5)
        kind, cores = "reference", arm.nproc
        how = ("the reference's own compiled kernels (oracle/_ref/_kernels_cy from "
               "pkg/src/pagetopk/_kernels_cy.pyx) driven as attention.decode_step, after a per-unit "
               "append with the reference's numpy page-stats refresh; one unit per task over "
               f"{arm.nproc} forked processes (the kernels hold the GIL)")
    else:
        kp_, vp_, means, stds, seq = ref_arm.appended(w)
        for _ in range(warm):
            O.decode_units(w["q"], kp_, vp_, w["tab"], seq, means, stds, w["kp"], 0.5,
                           1.0 / math.sqrt(w["D"]), w["S"], nthreads=ncores)
        t0 = time.perf_counter()
        for _ in range(steps):
            O.decode_units(w["q"], kp_, vp_, w["tab"], seq, means, stds, w["kp"], 0.5,
                           1.0 / math.sqrt(w["D"]), w["S"], nthreads=ncores)
        dt = (time.perf_counter() - t0) / steps
        kind, cores = "port", ncores
        how = ("oracle/pagetopk_oracle.c (bit-identical to _kernels_cy), OpenMP over units, on the "
               "post-append cache (the append itself untimed)")
    v = w["seqs"] / dt
    sample = (f"each step: {w['seqs']} of the {args.batch} sequences x {w['H']} kv-heads (ctx "
              f"{args.ctx} + 1 appended token, k={w['kp']} pages, bf16 values upcast to f32), "
              f"host-generated workload and stats (no GPU, no repo kernels); {how}; conservative "
              "for the reference: the batch is extrapolated from the sample at constant per-"
              "sequence cost and every host core serves the one rank")
    cb = {"value": v, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample}
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": steps, "warmup": warm, "ms_per_step": 1000.0 * args.batch / v,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic N(0,1) (reference workload distribution)", "config": config,
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# the B200 arm
# ---------------------------------------------------------------------------
def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(args):
    """`--gpus N` without a torchrun environment: re-run this script as N ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


class Ctx:
    """Rank / device / collective plumbing (NCCL on GPUs; BENCH_DIST_BACKEND=gloo lets N
    ranks share one GPU for a functional check of the multi-rank path)."""

    def __init__(self):
        import torch

        self.rank = int(os.environ.get("RANK", "0"))
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        self.dist = None
        cuda = torch.cuda.is_available()
        ndev = torch.cuda.device_count() if cuda else 1
        self.dev_index = self.local % max(ndev, 1)
        self.device = torch.device("cuda", self.dev_index) if cuda else torch.device("cpu")
        if self.world > 1:
            import torch.distributed as dist

            if cuda:
                torch.cuda.set_device(self.dev_index)
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=self.device)
            else:
                dist.init_process_group(self.backend)
            self.dist = dist

    def barrier(self):
        import torch

        if self.dist is not None:
            self.dist.barrier()
        if torch.cuda.is_available():
            torch.cuda.synchronize()

    def max(self, x: float) -> float:
        import torch

        if self.dist is None:
            return x
        dev = self.device if self.backend == "nccl" else torch.device("cpu")
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.dist is not None:
            self.dist.destroy_process_group()


def capture_steps(eng, cache, qs, kn, vn):
    """One CUDA graph of the whole step per rotating query set."""
    import torch

    graphs = []
    for q in qs:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            eng.step(q, kn, vn)
        cache._seq_host -= 1
        graphs.append(g)
    return graphs


def timed_replays(ctx, graphs, cache, steps, sampler=None):
    """K graph replays bracketed by a barrier + synchronize on both sides; device time by
    CUDA events on the launch stream; max over ranks (ms per step)."""
    import torch

    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.barrier()
    if sampler is not None:
        sampler.__enter__()
    e0.record(stream)
    for i in range(steps):
        graphs[i % len(graphs)].replay()
    e1.record(stream)
    ctx.barrier()
    if sampler is not None:
        sampler.__exit__()
    cache._seq_host += steps
    return ctx.max(e0.elapsed_time(e1)) / steps


def parity_check(eng, cache, q_local, args):
    """The oracle (attention.py:110-147 restated) on the first 2 sequences of this rank's
    shard at the current cache state vs one eager engine step on the same queries: selection
    sets, kth and kplus1 bit-exact, outputs within 2e-2 (bf16).  Raises on a mismatch."""
    import torch

    from oracle import oracle as O

    eng.step(q_local)
    torch.cuda.synchronize()
    a = _sample_arrays(cache, q_local, args)
    ref = O.decode_units(a["q"], a["kpool"], a["vpool"], a["tab"], a["seq"], a["means"], a["stds"],
                         a["kp"], 0.5, 1.0 / math.sqrt(a["D"]), a["S"], nthreads=host_cores())
    nu = len(a["units"])
    # engine ids are pool page ids; the sample pool is compacted: map through a["pids"]
    remap = {int(p): i for i, p in enumerate(a["pids"].tolist())}
    sel = eng.sel[:nu].cpu().numpy()
    nsel = eng.n_sel[:nu].cpu().numpy()
    G, D = args.q_heads // args.kv_heads, args.head_dim
    bad = 0
    for u in range(nu):
        got = {remap[int(p)] for p in sel[u, : nsel[u]].tolist()}
        if nsel[u] != ref["n_sel"][u] or got != set(ref["sel"][u, : ref["n_sel"][u]].tolist()):
            bad += 1
    kth_ok = np.array_equal(eng.kth[:nu].cpu().numpy(), ref["kth"])
    kp1_ok = np.array_equal(eng.kplus1[:nu].cpu().numpy(), ref["kplus1"])
    out = eng.out[: nu * G].cpu().numpy().reshape(nu, G, D)
    err = float(np.abs(out - ref["out"]).max())
    res = {"units": nu, "selection_mismatches": bad, "kth_equal": bool(kth_ok),
           "kplus1_equal": bool(kp1_ok), "out_max_abs_err": err, "tolerance": 2e-2,
           "oracle": "oracle/pagetopk_oracle.c decode_units (bit-identical to the reference "
                     "backend), the cache's first 2 sequences"}
    if bad or not kth_ok or not kp1_ok or err > 2e-2:
        raise AssertionError(f"bench parity check failed: {res}")
    return res, a


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "b200":
        self_launch(args)
    import torch

    H, D, S = args.kv_heads, args.head_dim, args.page
    G = args.q_heads // H
    kp = -(-args.budget // S)
    U = args.batch * H
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    n_gpus = max(world_env, args.gpus if args.impl == "reference" else world_env)
    config = {
        "workload": "BASELINE configs[2]: Llama-3.1-8B attn shape, 32q/8kv d128, global batch "
                    f"{args.batch}, ctx {args.ctx}, page {S}, k={args.budget} tokens ({kp} pages), "
                    f"bf16 KV, {args.stats_dtype} page stats"
                    + ("" if args.no_mirror or args.stats_dtype != "f32" else
                       " (+ bf16 mirror for bounded scoring)"),
        "global_batch": args.batch,
        "seq_len": args.ctx,
        "parallelism": f"{U} (sequence, kv-head) units split over {n_gpus} GPU(s) by sequence "
                       "(strong scaling), no data-path collective",
        "l2": "inputs larger than L2 (~0.8 GB touched per step vs 126 MB L2); 4 rotating query sets",
    }

    if args.impl == "reference":
        if int(os.environ.get("RANK", "0")) != 0:
            return
        run_reference_arm(args, n_gpus, config)
        return

    import paper_2605_27740_b200 as pt
    from paper_2605_27740_b200.shard import shard_units

    ctx = Ctx()
    rank, world, device = ctx.rank, ctx.world, ctx.device
    sh = shard_units(args.batch, H, G, world, rank)
    Ul = sh.num_units
    cache = build_cache(args, device, SEED, units=range(sh.u0, sh.u1))
    eng = pt.DecodeEngine(cache, G, kp)
    qs_g, kn_g, vn_g = step_inputs(args, device)
    r0, r1 = sh.q_rows
    qs = [q[r0:r1].contiguous() for q in qs_g]
    kn = kn_g[sh.u0:sh.u1].contiguous()
    vn = vn_g[sh.u0:sh.u1].contiguous()
    stream = torch.cuda.current_stream()

    if args.profile:
        for i in range(max(args.steps, 1)):
            eng.step(qs[i % len(qs)], kn, vn)
        torch.cuda.synchronize()
        if rank == 0:
            print(json.dumps({"profile": "done", "steps": args.steps}))
        ctx.close()
        return

    # warm-up (eager: kernel attributes, path decisions), then one graph per query set
    for i in range(max(args.warmup, 3)):
        eng.step(qs[i % len(qs)], kn, vn)
    torch.cuda.synchronize()
    cache.check_errors()
    graphs = capture_steps(eng, cache, qs, kn, vn)
    for i in range(args.warmup):
        graphs[i % len(graphs)].replay()
        cache._seq_host += 1
    torch.cuda.synchronize()

    # ---- timed region: K graph replays ------------------------------------------------
    sampler = ClockSampler(ctx.dev_index)
    ms_per_step = timed_replays(ctx, graphs, cache, args.steps, sampler)
    value = args.batch / (ms_per_step / 1000.0)
    cache.check_errors()

    # ---- per-kernel times (CUDA events on the launching stream, eager launches) -------
    reps = max(20, min(args.steps, 100))
    names = ["append", "lam_norms", "score", "select_attend"]
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(reps)]
    for r in range(reps):
        q = qs[r % len(qs)]
        ev = evs[r]
        ev[0].record(stream)
        cache.append_batch(kn, vn)
        ev[1].record(stream)
        eng.lam_norms(q)
        ev[2].record(stream)
        eng.score_step(q)
        ev[3].record(stream)
        eng.select_attend(q)
        ev[4].record(stream)
    torch.cuda.synchronize()
    cache.check_errors()
    bounded = bool(eng._step_bounded)
    brk = {n: statistics.median([evs[r][i].elapsed_time(evs[r][i + 1]) * 1000 for r in range(reps)])
           for i, n in enumerate(names)}

    if args.dump_out:  # one eager step (no append) on every rank, gathered in unit order
        eng.step(qs[0])
        outs = eng.out.cpu()
        if ctx.dist is not None:
            src = eng.out if ctx.backend == "nccl" else outs
            parts = [torch.empty_like(src) for _ in range(world)]
            ctx.dist.all_gather(parts, src)
            outs = torch.cat([x.cpu() for x in parts])
        if rank == 0:
            np.save(args.dump_out, outs.numpy())

    # ---- in-bench parity: the oracle on a sample of this very workload ---------------
    parity, sample = None, None
    if rank == 0 and not args.no_parity:
        parity, sample = parity_check(eng, cache, qs[0], args)

    # ---- dense denominator: same GPU, every page of every local unit ------------------
    dense_us = None
    if not args.no_dense:
        for i in range(3):
            eng.dense(qs[i % len(qs)])
        dreps = 20
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record(stream)
        for i in range(dreps):
            eng.dense(qs[i % len(qs)])
        d1.record(stream)
        torch.cuda.synchronize()
        dense_us = ctx.max(d0.elapsed_time(d1) * 1000 / dreps)

    # ---- optional output all-gather (NCCL over NVLink) + the step with it -------------
    allgather_us = step_with_gather_us = None
    if ctx.dist is not None:
        dist = ctx.dist
        comm_dev = device if ctx.backend == "nccl" else torch.device("cpu")
        full = torch.empty(args.batch * H * G, D, dtype=torch.float32, device=comm_dev)

        def gather():
            if ctx.backend == "nccl":
                dist.all_gather_into_tensor(full, eng.out)
            else:  # gloo: list all-gather of host copies (functional check only)
                parts = [torch.empty_like(full[: Ul * G]) for _ in range(world)]
                dist.all_gather(parts, eng.out.cpu())
                full.copy_(torch.cat(parts))

        for _ in range(3):
            gather()
        ctx.barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a0.record(stream)
        for _ in range(20):
            gather()
        a1.record(stream)
        torch.cuda.synchronize()
        ag = a0.elapsed_time(a1) * 1000 / 20 if ctx.backend == "nccl" else (time.perf_counter() - t0) * 1e6 / 20
        allgather_us = ctx.max(ag)
        ctx.barrier()
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        b0.record(stream)
        for i in range(20):
            graphs[i % len(graphs)].replay()
            gather()
        b1.record(stream)
        ctx.barrier()
        cache._seq_host += 20
        sg = b0.elapsed_time(b1) * 1000 / 20 if ctx.backend == "nccl" else (time.perf_counter() - t0) * 1e6 / 20
        step_with_gather_us = ctx.max(sg)
        # the gathered outputs are the unsharded result's rows (order = global unit order)
        assert full.shape[0] == args.batch * H * G

    # ---- e2e: the serving API (PipelinedDecoder) with pinned host buffers --------------
    dec = pt.PipelinedDecoder(cache, G, kp)
    nq, nk = qs[0].numel(), kn.numel()
    host_in = [torch.empty(nq + 2 * nk, dtype=torch.bfloat16).pin_memory() for _ in range(len(qs))]
    for i, q in enumerate(qs):
        host_in[i][:nq].copy_(q.reshape(-1).cpu())
        host_in[i][nq:nq + nk].copy_(kn.reshape(-1).cpu())
        host_in[i][nq + nk:].copy_(vn.reshape(-1).cpu())
    host_out = [torch.empty(Ul * G, D, dtype=torch.float32).pin_memory() for _ in range(2)]
    dec.capture(host_in[0].to(device))
    e2e_steps = max(20, min(args.steps, 200))
    for i in range(6):
        dec.submit(host_in[i % len(host_in)], host_out[i % 2])
    dec.synchronize()
    ctx.barrier()
    t0 = time.perf_counter()
    for i in range(e2e_steps):
        dec.submit(host_in[i % len(host_in)], host_out[i % 2])
    dec.synchronize()
    e2e_s = ctx.max(time.perf_counter() - t0) / e2e_steps
    e2e_value = args.batch / e2e_s
    cache.check_errors()
    h2d = host_in[0].numel() * 2 * world
    d2h = host_out[0].numel() * 4 * world

    # ---- roofline of the dominant kernel + whole step (SURVEY 8(d) bytes) -------------
    peaks, peak_kind = measured_peaks()
    e_st = 2 if (bounded or args.stats_dtype == "bf16") else 4
    P = -(-args.ctx // S)
    by = step_bytes(Ul, G, D, P, kp, S, 2, e_st, args.ctx)
    by_f32 = step_bytes(Ul, G, D, P, kp, S, 2, 4, args.ctx)
    kbytes = {"score": by["score"], "select_attend": by["topk"] + by["attend"]}
    dom = max(("score", "select_attend"), key=lambda n: brk[n])
    dom_bytes = kbytes[dom]
    achieved = dom_bytes / (brk[dom] * 1e-6) / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            t = json.load(open(tf))
            key = ("score_bounded" if bounded else "score") if dom == "score" else dom
            traffic = t.get(key)
            if isinstance(traffic, dict):
                traffic = traffic.get("bytes_per_launch")
        except Exception:
            traffic = None
    step_total = by["append"] + by["score"] + by["topk"] + by["attend"]

    # ---- weak scaling (N > 1): 32 sequences per rank --------------------------------
    weak = None
    if world > 1 and not args.no_weak:
        del dec, eng, graphs, cache
        torch.cuda.empty_cache()
        wargs = argparse.Namespace(**vars(args))
        wcache = build_cache(wargs, device, SEED + 1 + rank)
        weng = pt.DecodeEngine(wcache, G, kp)
        wq = [q.contiguous() for q in qs_g]
        for i in range(3):
            weng.step(wq[i % len(wq)], kn_g, vn_g)
        torch.cuda.synchronize()
        wgraphs = capture_steps(weng, wcache, wq, kn_g, vn_g)
        for i in range(max(args.warmup, 3)):
            wgraphs[i % len(wgraphs)].replay()
            wcache._seq_host += 1
        wms = timed_replays(ctx, wgraphs, wcache, args.steps)
        weak = {"value": world * args.batch / (wms / 1000.0), "unit": UNIT,
                "batch_per_gpu": args.batch, "ms_per_step": wms, "scaling": "weak"}

    cb = None
    if rank == 0 and world == 1 and not args.no_cpu:
        a = sample if sample is not None else _sample_arrays(cache, qs[0], args)
        r = cpu_baseline(a, args.cpu_seconds, host_cores())
        cb = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "us_per_step": ms_per_step * 1000,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic N(0,1) K/V/q per unit from a global seed (reference workload "
                    "distribution), generated on device",
            "config": dict(config, batch_per_gpu=args.batch // world if args.batch % world == 0
                           else round(args.batch / world, 3),
                           units_per_gpu=Ul, scoring="bounded (bf16 mirror)" if bounded else "exact f32 means"),
            "gpu_launches": 4 * args.steps,  # append, lam-norms, score, select+attend per step
            "breakdown_us": brk,
            "step_bytes": step_total,
            "step_bytes_model": "SURVEY 8(d) (page means at the KV element size: e=2)",
            "step_hbm_gbs": step_total / (ms_per_step * 1e-3) / 1e9,
            "step_frac_of_hbm": step_total / (ms_per_step * 1e-3) / 1e9 / peaks["hbm_gbs"],
            "roofline": {
                "kernel": dom,
                "bound": "hbm",
                "achieved": achieved,
                "peak": peaks["hbm_gbs"],
                "peak_kind": peak_kind,
                "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"],
                "bytes_per_launch": dom_bytes,
                "bytes_model": "SURVEY 8(d) algorithmic bytes (e=2 page means)",
                "traffic": traffic,
                "score_bytes_moved": bounded_score_moved(Ul, G, D, P) if bounded else by_f32["score"],
                "score_frac_by_bytes_moved": ((bounded_score_moved(Ul, G, D, P) if bounded else by_f32["score"])
                                              / (brk["score"] * 1e-6) / 1e9 / peaks["hbm_gbs"]),
            },
            "dense_us_per_step": dense_us,
            "x_over_dense": (dense_us / (ms_per_step * 1000)) if dense_us else None,
            "x_over_dense_kernels": (dense_us / (brk["score"] + brk["select_attend"])) if dense_us else None,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1000,
                    "path": "PipelinedDecoder.submit() (native pt_pipe_submit): pinned host "
                            "q|k|v block -> H2D (h2d stream) -> captured step graph (norms, append, "
                            "scorer overlapping the append, select+attend) -> D2H f32 outputs (d2h stream), double-buffered, "
                            "every step; wall clock over the steps, max over ranks"},
            "clocks": sampler.summary(),
            "allgather_us": allgather_us,
            "us_per_step_with_allgather": step_with_gather_us,
            "weak": weak,
            "parity": parity,
            "cpu_baseline": cb,
        }
        print(json.dumps(line), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
