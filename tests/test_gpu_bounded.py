"""Bounded scoring (pt_score_bounded + the resolving pt_select_attend) on the GPU.

The decode engine streams the bf16 mirror of the f32 page means and gets, per page, an
interval [klo, khi] of ordered keys that must contain the reference's exact key
(scoring.py:108-124 -> bf16.py:18-33 -> select.py:51-57); the selection then recomputes the
exact key of every page whose interval is not a single key and reaches the cut.  These tests
check (1) the mirror and its error bound, (2) the intervals contain the exact keys -- on the
reference workload and on adversarial value ranges, every G and D of the envelope -- and
(3) the engine's selections, kth / kplus1 are bit-identical to the exact-key path and to the
CPU oracle (outputs equal up to the f32 merge order), including take-all, no-tile-maxima,
massive ties, multi-round resolution and the early-streaming split.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _force_bounded(monkeypatch):
    """These shapes are small: the engine would pick exact scoring by its cost model."""
    monkeypatch.setenv("PT_BOUNDED", "1")


def _pt():
    import paper_2605_27740_b200 as pt

    return pt


def _cache(K, V, H, S, spare=4, mirror=True):
    pt = _pt()
    U, n, D = K.shape
    B = U // H
    Pcap = -(-n // S) + spare
    layout = pt.CacheLayout(num_kv_heads=H, head_dim=D, page_size=S, max_pages=U * Pcap)
    cache = pt.PagedKvCache(layout, batch=B, dtype=torch.bfloat16, max_pages_per_head=Pcap,
                            mirror=mirror)
    cache.extend_units(torch.from_numpy(K), torch.from_numpy(V))
    return cache


def readback(cache):
    kpool = cache.k_pool.to(torch.float32).cpu().numpy()
    vpool = cache.v_pool.to(torch.float32).cpu().numpy()
    return kpool, vpool, cache.page_table.cpu().numpy(), cache.seq_lens.cpu().numpy()


def _u16(t):
    return t.cpu().numpy().view(np.uint16)


def _bf16_rne_np(x: np.ndarray) -> np.ndarray:
    b = x.astype(np.float32).view(np.uint32).astype(np.uint64)
    return ((b + 0x7FFF + ((b >> 16) & 1)) >> 16).astype(np.uint16)


def test_mirror_is_bf16_of_means_and_err_bounds_it(cuda):
    from paper_2605_27740_b200 import _device as dev

    rng = np.random.default_rng(11)
    U, n, D, S = 4, 16 * 40 + 7, 128, 16
    K = (rng.standard_normal((U, n, D)) * np.exp(rng.uniform(-6, 6, (1, 1, D)))).astype(np.float32)
    cache = _cache(K, K, 2, S)
    # one decode append (the K1b mirror path) on top of the prefill (the fused-extend path)
    kn = torch.from_numpy(rng.standard_normal((U, D)).astype(np.float32)).cuda().to(torch.bfloat16)
    cache.append_batch(kn, kn)
    torch.cuda.synchronize()
    cache.check_errors()
    m32 = dev.untile_means(cache.means, U, cache.Pmax, D, torch.float32).cpu().numpy()
    tiles, rows, err = cache.mirror_views()
    mir = dev.untile_means(tiles, U, cache.Pmax, D, torch.bfloat16)
    mir_bits = mir.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
    mir_f = mir.to(torch.float32).cpu().numpy().astype(np.float64)
    rows = rows.cpu().numpy()
    err = err.cpu().numpy()
    for u in range(U):
        P = cache.num_pages(u)
        np.testing.assert_array_equal(mir_bits[u, :P], _bf16_rne_np(m32[u, :P]))
        np.testing.assert_array_equal(rows[u, :P], m32[u, :P])
        delta = np.linalg.norm(mir_f[u, :P] - m32[u, :P].astype(np.float64), axis=1)
        assert np.all(err[u, :P] >= delta)
        # and not absurdly loose: ||delta|| + the stated accumulation slack only
        mnorm = np.linalg.norm(m32[u, :P].astype(np.float64), axis=1)
        assert np.all(err[u, :P] <= delta + 2.1 * (D + 2) * 2.0 ** -18 * mnorm * 1.001 + 1e-30)


def _intervals_and_exact(cache, G, q, lam=0.5):
    """(klo, khi) from the bounded scorer and the exact keys from the f32-means scorer."""
    pt = _pt()
    eng = pt.DecodeEngine(cache, G, 4, lam=lam)
    assert eng.bounded
    eng.lam_norms(q)
    assert eng.score_bounded(q)
    torch.cuda.synchronize()
    klo, khi = _u16(eng.keys).copy(), _u16(eng.keys_hi).copy()
    tmax = _u16(eng.tile_max).copy()
    assert eng.score_prenorm(q)
    torch.cuda.synchronize()
    exact = _u16(eng.keys).copy()
    return klo, khi, exact, tmax


@pytest.mark.parametrize("G,D", [(1, 128), (3, 128), (4, 128), (8, 128), (4, 64), (7, 64)])
@pytest.mark.parametrize("dist", ["normal", "wide", "offset"])
def test_intervals_contain_exact_keys(cuda, G, D, dist):
    rng = np.random.default_rng(G * 100 + D + len(dist))
    U, S = 8, 16
    n = 16 * 700 + 5
    K = rng.standard_normal((U, n, D)).astype(np.float32)
    if dist == "wide":  # per-dim scales over 10 decades: products of very different size
        K *= np.exp(rng.uniform(-11, 11, (1, 1, D))).astype(np.float32)
    elif dist == "offset":  # large common offset: scores far from zero, small spread
        K += 40.0
    cache = _cache(K, K, 4, S)
    q = torch.from_numpy(rng.standard_normal((U * G, D)).astype(np.float32)).cuda().to(torch.bfloat16)
    klo, khi, exact, tmax = _intervals_and_exact(cache, G, q)
    unsure = 0
    for u in range(U):
        P = cache.num_pages(u)
        assert np.all(klo[u, :P] <= exact[u, :P]), f"lower key above the exact key (unit {u})"
        assert np.all(exact[u, :P] <= khi[u, :P]), f"upper key below the exact key (unit {u})"
        unsure += int(np.sum(klo[u, :P] != khi[u, :P]))
        nt = -(-P // 32)
        pad = np.zeros(nt * 32, np.uint16)
        pad[:P] = klo[u, :P]
        np.testing.assert_array_equal(tmax[u, :nt], pad.reshape(nt, 32).max(axis=1))
    # the mirror must actually decide most keys on the reference distribution
    if dist == "normal":
        assert unsure < 0.6 * U * cache.num_pages(0)


def _engines(cache, G, k):
    pt = _pt()
    a = pt.DecodeEngine(cache, G, k, keep_logical=True)
    b = pt.DecodeEngine(cache, G, k, keep_logical=True)
    b.bounded = False
    assert a.bounded
    return a, b


def _same_step(a, b, q, nsel_check=True):
    a.step(q)
    torch.cuda.synchronize()
    assert a._step_bounded
    oa = (a.out.clone(), a.lse.clone(), a.sel.clone(), a.sel_logical.clone(), a.n_sel.clone(),
          a.kth.clone(), a.kplus1.clone())
    b.step(q)
    torch.cuda.synchronize()
    assert not b._step_bounded
    ob = (b.out, b.lse, b.sel, b.sel_logical, b.n_sel, b.kth, b.kplus1)
    names = ("out", "lse", "sel", "sel_logical", "n_sel", "kth", "kplus1")
    for name, x, y in zip(names, oa, ob):
        if name in ("out", "lse"):
            # same pages; the bounded kernel streams the certainly selected pages first, so the
            # online-softmax page order differs -- and with it the running maximum the bf16
            # probabilities of the PV tensor-core product are rounded against (~2^-9 relative)
            torch.testing.assert_close(x, y, rtol=2e-3, atol=2e-3)
        else:
            assert torch.equal(x, y), f"bounded vs exact: {name} differs"


@pytest.mark.parametrize("n,k,G", [
    (16 * 8192, 128, 4),     # cfg3 per-unit shape (P = 8192, k = 128)
    (16 * 2048 + 9, 128, 4),  # cfg2 per-unit shape
    (16 * 100, 128, 4),      # take-all (P <= k)
    (16 * 1000, 40, 2),      # fewer tiles than k + 1 -> no tile-maximum bound
    (16 * 3000, 7, 8),
])
def test_bounded_selection_equals_exact(cuda, oracle, n, k, G):
    rng = np.random.default_rng(n + k)
    U, D, S = 4, 128, 16
    K = rng.standard_normal((U, n, D)).astype(np.float32)
    V = rng.standard_normal((U, n, D)).astype(np.float32)
    cache = _cache(K, V, 2, S)
    a, b = _engines(cache, G, k)
    for t in range(3):
        q = torch.from_numpy(rng.standard_normal((U * G, D)).astype(np.float32)).cuda().to(torch.bfloat16)
        _same_step(a, b, q)
    # and against the CPU oracle on the last query
    kpool, vpool, table, seq = readback(cache)
    means, stds = oracle.build_stats(kpool, table, seq, S)
    ref = oracle.decode_units(q.to(torch.float32).cpu().numpy().reshape(-1, G, D), kpool, vpool,
                              table, seq, means, stds, k, 0.5, 1.0 / math.sqrt(D), S)
    sel, nsel = a.sel.cpu().numpy(), a.n_sel.cpu().numpy()
    for u in range(U):
        assert nsel[u] == ref["n_sel"][u]
        assert set(sel[u, : nsel[u]].tolist()) == set(ref["sel"][u, : nsel[u]].tolist())
    np.testing.assert_array_equal(a.kth.cpu().numpy(), ref["kth"])
    np.testing.assert_array_equal(a.kplus1.cpu().numpy(), ref["kplus1"])


def test_bounded_massive_ties_and_multi_round_resolution(cuda, monkeypatch):
    """All pages of a unit share one mean (constant keys): every interval straddles or ties,
    the candidate list overflows -> select_block over resolved keys; a 32-page resolve
    capacity forces many resolution rounds."""
    rng = np.random.default_rng(7)
    U, D, S, n, G, k = 2, 128, 16, 16 * 4096, 4, 128
    row = rng.standard_normal(D).astype(np.float32)
    K = np.broadcast_to(row, (U, n, D)).copy()
    K[1] += np.repeat(rng.integers(-2, 3, (n // 16, 1, 1)), 16, axis=0).reshape(n, 1) * 0.25
    V = rng.standard_normal((U, n, D)).astype(np.float32)
    cache = _cache(K, V, 1, S)
    a, b = _engines(cache, G, k)
    q = torch.from_numpy(rng.standard_normal((U * G, D)).astype(np.float32)).cuda().to(torch.bfloat16)
    _same_step(a, b, q)
    monkeypatch.setenv("PT_SA_RCAP", "32")
    q2 = torch.from_numpy(rng.standard_normal((U * G, D)).astype(np.float32)).cuda().to(torch.bfloat16)
    _same_step(a, b, q2)


def test_bounded_eager_steps_with_appends_vs_oracle(cuda, oracle):
    """Back-to-back eager steps with appends and a different query every step (no sync in
    between): each step's selection and output equal the oracle's on that step's cache."""
    pt = _pt()
    rng = np.random.default_rng(21)
    U, H, D, S, G, k = 4, 2, 128, 16, 4, 16
    n = 16 * 300 + 14
    K = rng.standard_normal((U, n, D)).astype(np.float32)
    cache = _cache(K, K, H, S, spare=8)
    eng = pt.DecodeEngine(cache, G, k)
    qs = [torch.from_numpy(rng.standard_normal((U * G, D)).astype(np.float32)).cuda().to(torch.bfloat16)
          for _ in range(6)]
    kn = [torch.from_numpy(rng.standard_normal((U, D)).astype(np.float32)).cuda().to(torch.bfloat16)
          for _ in range(6)]
    snaps = []
    for t in range(6):
        eng.step(qs[t], kn[t], kn[t])
        snaps.append((eng.out.clone(), eng.sel.clone(), eng.n_sel.clone(), eng.kth.clone(),
                      eng.kplus1.clone()))
    torch.cuda.synchronize()
    cache.check_errors()
    kpool, vpool, table, seq = readback(cache)
    # replay the oracle step by step on the growing prefix of the final cache
    for t in range(6):
        seq_t = seq - (5 - t)
        means, stds = oracle.build_stats(kpool, table, seq_t, S)
        ref = oracle.decode_units(qs[t].to(torch.float32).cpu().numpy().reshape(-1, G, D), kpool,
                                  vpool, table, seq_t, means, stds, k, 0.5, 1.0 / math.sqrt(D), S)
        out, sel, nsel, kth, kp1 = (x.cpu().numpy() for x in snaps[t])
        for u in range(U):
            assert set(sel[u, : nsel[u]].tolist()) == set(ref["sel"][u, : ref["n_sel"][u]].tolist())
        np.testing.assert_array_equal(kth, ref["kth"])
        np.testing.assert_array_equal(kp1, ref["kplus1"])
        np.testing.assert_allclose(out.reshape(-1, G, D), ref["out"], rtol=2e-2, atol=2e-2)


def test_bounded_warp_per_unit_selection_equals_exact(cuda, oracle):
    """The warp-per-unit select+attend (>= 4 x SMs units, k <= 64, P <= 2048: the cfg4 shape)
    in bounded mode: bracket by bisection in registers, bracket pages resolved one lane each --
    selections bit-identical to the exact path and to the oracle."""
    pt = _pt()
    rng = np.random.default_rng(4)
    U, D, S, n, G, k = 600, 64, 32, 32 * 100 + 7, 1, 16
    K = rng.standard_normal((U, n, D)).astype(np.float32)
    V = rng.standard_normal((U, n, D)).astype(np.float32)
    Pcap = -(-n // S) + 4
    layout = pt.CacheLayout(num_kv_heads=1, head_dim=D, page_size=S, max_pages=U * Pcap)
    cache = pt.PagedKvCache(layout, batch=U, dtype=torch.bfloat16, max_pages_per_head=Pcap)
    cache.extend_units(torch.from_numpy(K), torch.from_numpy(V))
    del K, V
    a, b = _engines(cache, G, k)
    for _ in range(2):
        q = torch.from_numpy(rng.standard_normal((U * G, D)).astype(np.float32)).cuda().to(torch.bfloat16)
        _same_step(a, b, q)
    kpool, vpool, table, seq = readback(cache)
    means, stds = oracle.build_stats(kpool, table, seq, S)
    ref = oracle.decode_units(q.to(torch.float32).cpu().numpy().reshape(-1, G, D), kpool, vpool,
                              table, seq, means, stds, k, 0.5, 1.0 / math.sqrt(D), S)
    sel, nsel = a.sel.cpu().numpy(), a.n_sel.cpu().numpy()
    for u in range(U):
        assert set(sel[u, : nsel[u]].tolist()) == set(ref["sel"][u, : ref["n_sel"][u]].tolist())
    np.testing.assert_array_equal(a.kth.cpu().numpy(), ref["kth"])
    np.testing.assert_array_equal(a.kplus1.cpu().numpy(), ref["kplus1"])


def test_half_batch_split_step_equals_one_range(cuda, oracle, monkeypatch):
    """The two-stream half-batch step (score A -> [select+attend A on a side stream] beside
    score B -> select+attend B, pt_score_bounded / pt_select_attend over unit ranges) gives
    the selections of the one-range bounded step bit for bit (outputs up to the chunk-merge
    order: a 64-unit range splits each unit over more CTAs), eagerly and from a captured
    graph with appends, and those of the exact path and of the oracle."""
    pt = _pt()
    monkeypatch.setenv("PT_SPLIT", "1")
    rng = np.random.default_rng(99)
    U, H, D, S, G, k = 128, 8, 128, 16, 4, 64
    n = 16 * 400 + 5
    K = rng.standard_normal((U, n, D)).astype(np.float32)
    V = rng.standard_normal((U, n, D)).astype(np.float32)
    cache = _cache(K, V, H, S, spare=8)
    del K, V
    a = pt.DecodeEngine(cache, G, k, keep_logical=True)
    c = pt.DecodeEngine(cache, G, k, keep_logical=True)
    c.split = False
    assert a.split and a.bounded and a.split_at == 64
    _, b = _engines(cache, G, k)

    def outs(e):
        return [x.clone() for x in (e.out, e.lse, e.sel, e.sel_logical, e.n_sel, e.kth, e.kplus1)]

    def _same_outs(x, y):
        # same pages, another streaming order (chunking, sure-first) -- the bf16 probabilities
        # of the PV product are rounded against another running maximum (see _same_step)
        torch.testing.assert_close(x[0], y[0], rtol=2e-3, atol=2e-3)
        torch.testing.assert_close(x[1], y[1], rtol=2e-3, atol=2e-3)
        for i in (3, 4, 5, 6):
            assert torch.equal(x[i], y[i])
        # sel lists the same pages per unit (order: the streaming order of each variant)
        assert torch.equal(torch.sort(x[2], dim=1).values, torch.sort(y[2], dim=1).values)

    for _ in range(2):
        q = torch.from_numpy(rng.standard_normal((U * G, D)).astype(np.float32)).cuda().to(torch.bfloat16)
        a.step(q)
        c.step(q)
        torch.cuda.synchronize()
        _same_outs(outs(a), outs(c))
        _same_step(a, b, q)
    # captured with appends: the replay's outputs equal an eager one-range step afterwards
    qs = torch.empty((U * G, D), dtype=torch.bfloat16, device="cuda")
    kn = torch.empty((U, D), dtype=torch.bfloat16, device="cuda")
    a.capture(qs, kn, kn)
    for _ in range(3):
        qs.copy_(torch.from_numpy(rng.standard_normal((U * G, D)).astype(np.float32)))
        kn.copy_(torch.from_numpy(rng.standard_normal((U, D)).astype(np.float32)))
        a.replay()
        c.step(qs)
        torch.cuda.synchronize()
        _same_outs(outs(a), outs(c))
    cache.check_errors()
    kpool, vpool, table, seq = readback(cache)
    means, stds = oracle.build_stats(kpool, table, seq, S)
    ref = oracle.decode_units(qs.to(torch.float32).cpu().numpy().reshape(-1, G, D), kpool, vpool,
                              table, seq, means, stds, k, 0.5, 1.0 / math.sqrt(D), S)
    sel, nsel = a.sel.cpu().numpy(), a.n_sel.cpu().numpy()
    for u in range(U):
        assert set(sel[u, : nsel[u]].tolist()) == set(ref["sel"][u, : ref["n_sel"][u]].tolist())
    np.testing.assert_array_equal(a.kth.cpu().numpy(), ref["kth"])
    np.testing.assert_array_equal(a.kplus1.cpu().numpy(), ref["kplus1"])


@pytest.mark.parametrize("U,H,n0,ragged", [
    (16, 8, 16 * 4096 - 3, True),    # ~2K tiles over ~1.2K scorer warps: ranges cross units
    (6, 2, 16 * 64 * 3 - 2, False),  # tail page / tail tile boundaries crossed within the run
    (256, 8, 16 * 40 + 5, True),     # many short units: several tail tiles per warp range
])
def test_early_scorer_step_equals_chained_step(cuda, monkeypatch, U, H, n0, ragged):
    """DecodeEngine.step with the scorer overlapping the append (pt_append_step +
    pt_score_bounded_step: non-tail tiles streamed from the snapshot lengths, tail tiles
    deferred until the append's stores are visible) == the append -> norms -> scorer chain
    (PT_EARLY=0): key intervals, tile maxima, selections, kth / kplus1 and outputs bit for bit,
    over eager steps (new pages, new 32-page tiles) and CUDA-graph replays."""
    pt = _pt()
    D, S, G, k = 128, 16, 4, 8
    rng = np.random.default_rng(U + n0)
    nr = (n0 - rng.integers(0, 40, U)) if ragged else np.full(U, n0)
    dev = torch.device("cuda")
    K = torch.randn(U, n0, D, device=dev).to(torch.bfloat16)
    V = torch.randn(U, n0, D, device=dev).to(torch.bfloat16)
    steps = 12
    engines, caches = [], []
    for early in ("1", "0"):
        monkeypatch.setenv("PT_EARLY", early)
        Pcap = -(-(n0 + steps + 8) // S) + 2
        layout = pt.CacheLayout(num_kv_heads=H, head_dim=D, page_size=S, max_pages=U * Pcap)
        cache = pt.PagedKvCache(layout, batch=U // H, dtype=torch.bfloat16, max_pages_per_head=Pcap,
                                mirror=True)
        cache.extend_units(K, V, n_rows=nr)
        eng = pt.DecodeEngine(cache, G, k)
        assert eng.early == (early == "1") and eng.bounded
        engines.append(eng)
        caches.append(cache)
    qs = [torch.randn(U * G, D, device=dev).to(torch.bfloat16) for _ in range(steps)]
    kn = [torch.randn(U, D, device=dev).to(torch.bfloat16) for _ in range(steps)]

    def compare():
        a, b = engines
        seq = caches[0].seq_lens
        assert torch.equal(seq, caches[1].seq_lens)
        P = (-(-seq // S)).cpu().numpy()
        ka, kb = a.keys.cpu().numpy(), b.keys.cpu().numpy()
        ha, hb = a.keys_hi.cpu().numpy(), b.keys_hi.cpu().numpy()
        ta, tb = a.tile_max.cpu().numpy(), b.tile_max.cpu().numpy()
        for u in range(U):
            np.testing.assert_array_equal(ka[u, : P[u]], kb[u, : P[u]])
            np.testing.assert_array_equal(ha[u, : P[u]], hb[u, : P[u]])
            np.testing.assert_array_equal(ta[u, : -(-P[u] // 32)], tb[u, : -(-P[u] // 32)])
        assert torch.equal(a.sel.sort(dim=1).values, b.sel.sort(dim=1).values)
        for x, y in ((a.n_sel, b.n_sel), (a.kth, b.kth), (a.kplus1, b.kplus1), (a.out, b.out),
                     (a.lse, b.lse)):
            assert torch.equal(x, y)

    for t in range(steps // 2):  # eager, back to back (no sync in between), then compared
        for eng in engines:
            eng.step(qs[t], kn[t], kn[t])
        torch.cuda.synchronize()
        compare()
    assert int(engines[0].step_sync[0]) == int(engines[0].step_sync[2]) == steps // 2
    for eng in engines:  # graph replays of the same step
        eng.capture(qs[0], kn[0], kn[0])
    for t in range(steps // 2):
        for eng in engines:
            eng.replay()
        torch.cuda.synchronize()
        compare()
    for c in caches:
        c.check_errors()
