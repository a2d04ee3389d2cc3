"""Paged key/value cache resident in B200 HBM, with per-page key statistics.

Drop-in for the reference ``pagetopk.kvcache`` (kvcache.py:1-341): same types
(``CacheLayout``, ``PageStats``, ``PageTable``, ``PagedKvCache``,
``CapacityError``), same methods and error behaviour, same UNQK snapshot format.
The storage is B200-first:

* one shared physical page pool ``[max_pages][S][D]`` for K and for V (bf16 or f32);
* per-unit logical->physical page tables ``int32 [U][Pmax]`` where a unit is one
  (sequence, kv-head) pair, ``u = b * H_kv + h`` -- ``batch`` independent sequences
  share the pool (the reference holds one sequence; batch=1 is identical to it);
* page means in a page-interleaved tile layout (see csrc/common.cuh) in
  ``stats_dtype`` (float32 = the reference's exact stats, the default; bfloat16 =
  compact mode), stds float32;
* statistics computed on the GPU by the K1 kernel in the reference's float64
  operation order (bit-identical to kvcache.py:59-71).

Appends in the decode loop (``append_batch``) allocate pages on the device
(free list, then bump, in unit order -- kvcache.py:154-176) so a step can be
captured in a CUDA graph; the per-head methods keep the reference signatures.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dev
from . import _lib
from ._lib import CapacityError

SNAPSHOT_MAGIC = b"UNQK"
SNAPSHOT_VERSION = 1

__all__ = [
    "CacheLayout",
    "CapacityError",
    "PageStats",
    "PageTable",
    "PagedKvCache",
    "compute_page_stats",
    "SNAPSHOT_MAGIC",
    "SNAPSHOT_VERSION",
]


@dataclass(frozen=True)
class CacheLayout:
    """Static shape of a cache: heads, head dimension, page size, pool size (kvcache.py:34-47)."""

    num_kv_heads: int
    head_dim: int
    page_size: int = 8
    max_pages: int = 4096

    def __post_init__(self) -> None:
        if self.num_kv_heads < 1 or self.head_dim < 1:
            raise ValueError("num_kv_heads and head_dim must be positive")
        if self.page_size < 1 or self.max_pages < 1:
            raise ValueError("page_size and max_pages must be positive")


@dataclass
class PageStats:
    """Summary of one page: row count, mean key vector, scalar key spread (kvcache.py:50-56)."""

    count: int
    mean: np.ndarray  # (head_dim,) f32
    std: float


def compute_page_stats(keys) -> PageStats:
    """kvcache.py:59-71 on the GPU (K1 kernel): f64 accumulation, f32 results."""
    rows = np.asarray(keys.cpu() if isinstance(keys, torch.Tensor) else keys, dtype=np.float32)
    if rows.ndim != 2 or rows.shape[0] == 0:
        raise ValueError("keys must be a non-empty (count, head_dim) array")
    device = dev.require_cuda()
    c, D = rows.shape
    if D % 4:
        raise NotImplementedError("compute_page_stats on the GPU needs head_dim % 4 == 0")
    pool = torch.from_numpy(np.ascontiguousarray(rows)).to(device).view(1, c, D)
    table = torch.zeros(1, 32, dtype=torch.int32, device=device)
    seq = torch.tensor([c], dtype=torch.int32, device=device)
    means = torch.zeros(32 * D, dtype=torch.float32, device=device)
    stds = torch.zeros(1, 32, dtype=torch.float32, device=device)
    _lib.call("pt_page_stats", pool.data_ptr(), _lib.PT_F32, table.data_ptr(), seq.data_ptr(),
              None, 1, c, D, 32, means.data_ptr(), _lib.PT_F32, stds.data_ptr(), None, None,
              dev.stream_handle())
    mean = dev.untile_means(means, 1, 32, D, torch.float32)[0, 0].cpu().numpy()
    return PageStats(count=c, mean=mean, std=float(stds[0, 0].item()))


class PageTable:
    """Logical-to-physical page mapping per head, plus the pool free list (kvcache.py:74-120).

    A host-side table, used standalone exactly like the reference's (e.g. to drive
    ``radix_topk``).  A device cache exposes the same interface through
    :class:`_DevicePageTable`.
    """

    def __init__(self, num_kv_heads: int) -> None:
        self._pages: list[list[int]] = [[] for _ in range(num_kv_heads)]
        self._where: dict[int, tuple[int, int]] = {}  # physical -> (head, logical)
        self.free_list: list[int] = []

    def num_pages(self, head: int) -> int:
        return len(self._pages[head])

    def append_page(self, head: int, pid: int) -> None:
        pid = int(pid)
        if pid in self._where:
            raise ValueError(f"physical page {pid} already mapped")
        self._where[pid] = (head, len(self._pages[head]))
        self._pages[head].append(pid)

    def mapping(self, head: int) -> np.ndarray:
        """Physical page ids in logical order (read-only)."""
        arr = np.asarray(self._pages[head], dtype=np.int64)
        arr.flags.writeable = False
        return arr

    def physical(self, head: int, logical: int) -> int:
        pages = self._pages[head]
        if logical < 0 or logical >= len(pages):
            raise LookupError(f"logical page {logical} out of range for head {head}")
        return pages[logical]

    def to_logical(self, head: int, physical_ids) -> np.ndarray:
        """Map physical ids back to this head's logical indices (LookupError if foreign)."""
        ids = np.asarray(physical_ids).reshape(-1).tolist()
        res = np.empty(len(ids), dtype=np.int64)
        for j, pid in enumerate(ids):
            hit = self._where.get(int(pid))
            if hit is None or hit[0] != head:
                raise LookupError(f"physical page {pid} not allocated for head {head}")
            res[j] = hit[1]
        return res


class _DevicePageTable:
    """PageTable interface over a device cache's int32 [U][Pmax] table."""

    def __init__(self, cache: "PagedKvCache") -> None:
        self._cache = cache

    def num_pages(self, head: int) -> int:
        return self._cache.num_pages(head)

    @property
    def free_list(self) -> list[int]:
        return self._cache._free_list_host()

    def mapping(self, head: int) -> np.ndarray:
        c = self._cache
        p = c.num_pages(head)
        view = c.page_table[head, :p].to(torch.int64).cpu().numpy()
        view.flags.writeable = False
        return view

    def physical(self, head: int, logical: int) -> int:
        if not 0 <= logical < self._cache.num_pages(head):
            raise LookupError(f"logical page {logical} out of range for head {head}")
        return int(self._cache.page_table[head, logical].item())

    def to_logical(self, head: int, physical_ids) -> np.ndarray:
        mapping = self.mapping(head)
        where = {int(pid): i for i, pid in enumerate(mapping.tolist())}
        out = np.empty(len(physical_ids), dtype=np.int64)
        for i, pid in enumerate(np.asarray(physical_ids).tolist()):
            lg = where.get(int(pid))
            if lg is None:
                raise LookupError(f"physical page {pid} not allocated for head {head}")
            out[i] = lg
        return out


class PagedKvCache:
    """Append-only paged KV storage with cached page statistics, in HBM (kvcache.py:123-341).

    ``batch`` sequences x ``num_kv_heads`` heads = ``num_units`` units; the
    per-head methods take ``head`` = unit index (for batch=1 this is the kv head).
    """

    def __init__(
        self,
        layout: CacheLayout,
        batch: int = 1,
        dtype: torch.dtype = torch.float32,
        stats_dtype: torch.dtype = torch.float32,
        max_pages_per_head: int | None = None,
        device=None,
        mirror: bool | None = None,
    ) -> None:
        if batch < 1:
            raise ValueError("batch must be positive")
        self.layout = layout
        self.batch = batch
        self.dtype = dtype
        self.stats_dtype = stats_dtype
        self.device = torch.device(device) if device is not None else dev.require_cuda()
        dev.require_cuda()
        H, D, S = layout.num_kv_heads, layout.head_dim, layout.page_size
        self.num_units = U = batch * H
        if D % dev.stats_vec(stats_dtype):
            raise NotImplementedError(
                f"head_dim {D} must be a multiple of {dev.stats_vec(stats_dtype)} for "
                f"{stats_dtype} page means"
            )
        if (D * (4 if dtype == torch.float32 else 2)) % 16:
            raise NotImplementedError("head_dim * element size must be a multiple of 16 bytes")
        self.kv_code = dev.dtype_code(dtype)
        self.stats_code = dev.dtype_code(stats_dtype)
        self.Pmax = dev.round_up(max_pages_per_head or layout.max_pages, 32)
        d = self.device
        self.k_pool = torch.zeros(layout.max_pages, S, D, dtype=dtype, device=d)
        self.v_pool = torch.zeros(layout.max_pages, S, D, dtype=dtype, device=d)
        self.page_table = torch.full((U, self.Pmax), -1, dtype=torch.int32, device=d)
        self.seq_lens = torch.zeros(U, dtype=torch.int32, device=d)
        self.means = torch.zeros(U * self.Pmax * D, dtype=stats_dtype, device=d)
        self.stds = torch.zeros(U, self.Pmax, dtype=torch.float32, device=d)
        # bf16 mirror of the f32 means + its per-page error bound (bounded scoring,
        # DESIGN.md): on by default for bf16 KV with exact f32 stats (the decode engine then
        # streams half the scoring bytes and still selects exactly as the f32 reference)
        if mirror is None:
            mirror = stats_dtype == torch.float32 and dtype == torch.bfloat16 and D % 8 == 0
        if mirror and (stats_dtype != torch.float32 or D % 8):
            raise ValueError("the bf16 mirror needs f32 page stats and head_dim % 8 == 0")
        self.mirror = None
        if mirror:
            nb = _lib.load().pt_mirror_bytes(U, self.Pmax, D)
            self.mirror = torch.zeros(nb, dtype=torch.uint8, device=d)
        # {bump_next, free_count, max_pages, error_flag}
        self.pool_state = torch.tensor([0, 0, layout.max_pages, 0], dtype=torch.int32, device=d)
        self.free_list_dev = torch.zeros(layout.max_pages, dtype=torch.int32, device=d)
        self._slot = torch.zeros(2 * U + 4, dtype=torch.int32, device=d)  # targets, flags, lengths
        # extend_units: fused pt_extend (default) or pt_write_rows + pt_page_stats (cross-check)
        self.split_extend = False
        self._seq_host = np.zeros(U, dtype=np.int64)
        self.table = _DevicePageTable(self)

    def _mirror_args(self):
        return (None if self.mirror is None else self.mirror.data_ptr(),)

    def mirror_views(self):
        """(bf16 tiles [U*Pmax*D], f32 rows [U][Pmax][D], err [U][Pmax]) views of the mirror
        block (readback / tests), or None."""
        if self.mirror is None:
            return None
        U, P, D = self.num_units, self.Pmax, self.layout.head_dim
        al = lambda x: (x + 255) // 256 * 256  # noqa: E731
        n = U * P
        t0, t1 = al(n * D * 2), al(n * D * 4)
        tiles = self.mirror[: n * D * 2].view(torch.bfloat16)
        rows = self.mirror[t0 : t0 + n * D * 4].view(torch.float32).view(U, P, D)
        err = self.mirror[t0 + t1 : t0 + t1 + n * 4].view(torch.float32).view(U, P)
        return tiles, rows, err

    # ------------------------------------------------------------------
    # Shape queries

    def seq_len(self, head: int) -> int:
        return int(self._seq_host[head])

    def num_pages(self, head: int) -> int:
        return -(-int(self._seq_host[head]) // self.layout.page_size)

    def total_allocated_pages(self) -> int:
        st = self.pool_state.cpu().numpy()
        return int(st[0] - st[1])

    def _free_list_host(self) -> list[int]:
        n = int(self.pool_state[1].item())
        return self.free_list_dev[:n].cpu().tolist()

    # ------------------------------------------------------------------
    # Appends

    def _host_alloc(self, counts: np.ndarray) -> np.ndarray:
        """Host-side _alloc_page (kvcache.py:154-176) for `counts[u]` new pages per unit,
        in unit order: the free list is popped from its end first, then the bump pointer."""
        st = self.pool_state.cpu().numpy()
        bump, nfree, maxp = int(st[0]), int(st[1]), int(st[2])
        need = int(counts.sum())
        if need > nfree + (maxp - bump):
            raise CapacityError(f"page pool exhausted ({maxp} pages)")
        from_free = min(need, nfree)
        popped = self.free_list_dev[nfree - from_free : nfree].cpu().numpy()[::-1]
        pids = np.concatenate([popped.astype(np.int64),
                               np.arange(bump, bump + need - from_free, dtype=np.int64)])
        self.pool_state[0] = bump + need - from_free
        self.pool_state[1] = nfree - from_free
        return pids  # flat, unit-major (counts[u] ids per unit)

    def extend_units(self, keys: torch.Tensor, values: torch.Tensor, n_rows=None) -> None:
        """Batched extend (kvcache.py:210-233) for every unit at once.

        ``keys``/``values``: [U, n_max, D]; ``n_rows[u]`` rows of unit u are appended
        (default: all n_max).  Pages are mapped on the host, rows are scattered and
        the touched pages' stats recomputed on the device.
        """
        U, S, D = self.num_units, self.layout.page_size, self.layout.head_dim
        if keys.ndim != 3 or keys.shape != values.shape or keys.shape[0] != U or keys.shape[2] != D:
            raise ValueError("keys/values must be matching (units, n, head_dim) arrays")
        n_max = keys.shape[1]
        nr = np.full(U, n_max, dtype=np.int64) if n_rows is None else np.asarray(n_rows, np.int64)
        # device appends may have been refused (pool / page-table exhaustion, reported by
        # check_errors): start from the lengths the device actually holds
        self._seq_host = self.seq_lens.cpu().numpy().astype(np.int64)
        n0 = self._seq_host.copy()
        n1 = n0 + nr
        P0 = -(-n0 // S)
        P1 = -(-n1 // S)
        if np.any(P1 > self.Pmax):
            raise CapacityError(f"page table capacity exhausted ({self.Pmax} pages per head)")
        new_pids = self._host_alloc(P1 - P0)
        d = self.device
        cnt = P1 - P0
        total = int(cnt.sum())
        if total:
            # (unit, logical page) of every new page, vectorised (no per-unit Python loop)
            r = np.repeat(np.arange(U), cnt)
            c = np.arange(total) - np.repeat(np.cumsum(cnt) - cnt, cnt) + np.repeat(P0, cnt)
            flat = torch.from_numpy((r * self.Pmax + c).astype(np.int64)).to(d)
            v = torch.from_numpy(new_pids.astype(np.int32)).to(d)
            self.page_table.view(-1).index_copy_(0, flat, v)
        kk = dev.to_device(keys, self.dtype, d)
        vv = dev.to_device(values, self.dtype, d)
        row_begin = torch.from_numpy(n0.astype(np.int32)).to(d)
        nrows_t = torch.from_numpy(nr.astype(np.int32)).to(d)
        sh = dev.stream_handle()
        self._seq_host = n1
        if not self.split_extend:
            # one launch: rows scattered into their pages and every touched page's stats
            _lib.call("pt_extend", kk.data_ptr(), vv.data_ptr(), n_max, row_begin.data_ptr(),
                      nrows_t.data_ptr(), self.k_pool.data_ptr(), self.v_pool.data_ptr(),
                      self.kv_code, self.page_table.data_ptr(), U, S, D, self.Pmax,
                      self.means.data_ptr(), self.stats_code, self.stds.data_ptr(),
                      *self._mirror_args(), sh)
            self.seq_lens.copy_(torch.from_numpy(n1.astype(np.int32)))
            return
        _lib.call("pt_write_rows", kk.data_ptr(), vv.data_ptr(), n_max, row_begin.data_ptr(),
                  nrows_t.data_ptr(), self.k_pool.data_ptr(), self.v_pool.data_ptr(), self.kv_code,
                  self.page_table.data_ptr(), U, S, D, self.Pmax, sh)
        self.seq_lens.copy_(torch.from_numpy(n1.astype(np.int32)))
        first = np.where(nr > 0, n0 // S, np.iinfo(np.int32).max).astype(np.int32)
        page_begin = torch.from_numpy(first).to(d)
        _lib.call("pt_page_stats", self.k_pool.data_ptr(), self.kv_code,
                  self.page_table.data_ptr(), self.seq_lens.data_ptr(), page_begin.data_ptr(), U,
                  S, D, self.Pmax, self.means.data_ptr(), self.stats_code, self.stds.data_ptr(),
                  *self._mirror_args(), sh)

    def extend(self, head: int, keys, values) -> None:
        """Bulk append to one head; same result as appending row by row (kvcache.py:210-233)."""
        k = keys if isinstance(keys, torch.Tensor) else np.asarray(keys, dtype=np.float32)
        v = values if isinstance(values, torch.Tensor) else np.asarray(values, dtype=np.float32)
        D = self.layout.head_dim
        if k.ndim != 2 or tuple(k.shape) != tuple(v.shape) or k.shape[1] != D:
            raise ValueError("keys/values must be matching (n, head_dim) arrays")
        n = k.shape[0]
        if n == 0:
            return
        U = self.num_units
        kt = torch.zeros(U, n, D, dtype=self.dtype, device=self.device)
        vt = torch.zeros(U, n, D, dtype=self.dtype, device=self.device)
        kt[head] = dev.to_device(k, self.dtype, self.device)
        vt[head] = dev.to_device(v, self.dtype, self.device)
        counts = np.zeros(U, dtype=np.int64)
        counts[head] = n
        self.extend_units(kt, vt, counts)

    def append(self, head: int, key, value) -> int:
        """Append one token's key/value row; returns its logical position (kvcache.py:185-208)."""
        k = key if isinstance(key, torch.Tensor) else np.asarray(key, dtype=np.float32)
        v = value if isinstance(value, torch.Tensor) else np.asarray(value, dtype=np.float32)
        if tuple(k.shape) != (self.layout.head_dim,) or tuple(v.shape) != tuple(k.shape):
            raise ValueError("key/value must be (head_dim,) vectors")
        pos = self.seq_len(head)
        self.extend(head, k[None], v[None])
        return pos

    def append_batch(self, keys: torch.Tensor, values: torch.Tensor, stream=None,
                     step_sync: torch.Tensor | None = None) -> None:
        """Decode-step append: one row per unit, on the device, no host sync (K1b).

        Allocation happens on the device; pool exhaustion sets an error flag that
        :meth:`check_errors` turns into ``CapacityError``.  ``step_sync`` (int32[4]): the
        append of a :class:`DecodeEngine` step whose scorer overlaps it (pt_append_step).
        """
        U, D = self.num_units, self.layout.head_dim
        if tuple(keys.shape) != (U, D) or tuple(values.shape) != (U, D):
            raise ValueError("keys/values must be (units, head_dim)")
        if keys.dtype != self.dtype or values.dtype != self.dtype or not keys.is_cuda:
            raise ValueError("keys/values must be device tensors of the cache dtype")
        keys, values = keys.contiguous(), values.contiguous()
        args = (keys.data_ptr(), values.data_ptr(), self.k_pool.data_ptr(),
                self.v_pool.data_ptr(), self.kv_code, self.page_table.data_ptr(),
                self.seq_lens.data_ptr(), U, self.layout.page_size, D, self.Pmax,
                self.means.data_ptr(), self.stats_code, self.stds.data_ptr(),
                self.pool_state.data_ptr(), self.free_list_dev.data_ptr(),
                self._slot.data_ptr(), *self._mirror_args())
        if step_sync is None:
            _lib.call("pt_append", *args, dev.stream_handle(stream))
        else:
            _lib.call("pt_append_step", *args, step_sync.data_ptr(), dev.stream_handle(stream))
        self._seq_host += 1

    def check_errors(self) -> None:
        """Synchronise the host mirror with device-side appends; raise on exhaustion."""
        if int(self.pool_state[3].item()) == _lib.PT_ERR_CAPACITY:
            self.pool_state[3] = 0
            self._seq_host = self.seq_lens.cpu().numpy().astype(np.int64)
            raise CapacityError(f"page pool exhausted ({self.layout.max_pages} pages)")
        self._seq_host = self.seq_lens.cpu().numpy().astype(np.int64)

    # ------------------------------------------------------------------
    # Reads

    def _means_rowmajor(self, head: int) -> np.ndarray:
        D = self.layout.head_dim
        m = dev.untile_means(self.means, self.num_units, self.Pmax, D, self.stats_dtype)
        return m[head, : self.num_pages(head)].to(torch.float32).cpu().numpy()

    def _counts(self, head: int) -> np.ndarray:
        p, S, n = self.num_pages(head), self.layout.page_size, self.seq_len(head)
        c = np.full(p, S, dtype=np.int64)
        if p:
            c[-1] = n - (p - 1) * S
        return c

    def page_stats(self, head: int, logical: int) -> PageStats:
        self.table.physical(head, logical)
        return PageStats(
            count=int(self._counts(head)[logical]),
            mean=self._means_rowmajor(head)[logical].copy(),
            std=float(self.stds[head, logical].item()),
        )

    def stats_arrays(self, head: int) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """Contiguous (means, stds, counts) in logical page order (kvcache.py:246-253)."""
        p = self.num_pages(head)
        return (
            np.ascontiguousarray(self._means_rowmajor(head)),
            self.stds[head, :p].cpu().numpy().copy(),
            self._counts(head),
        )

    def _owner_rows(self, head: int, physical_ids) -> list[int]:
        logical = self.table.to_logical(head, physical_ids)
        counts = self._counts(head)
        return [int(counts[lg]) for lg in logical]

    def page_rows(self, pid: int) -> int:
        for u in range(self.num_units):
            m = self.table.mapping(u)
            hit = np.nonzero(m == pid)[0]
            if hit.size:
                return int(self._counts(u)[hit[0]])
        return 0

    def page_keys(self, head: int, logical: int) -> np.ndarray:
        pid = self.table.physical(head, logical)
        rows = int(self._counts(head)[logical])
        return self.k_pool[pid, :rows].to(torch.float32).cpu().numpy()

    def page_values(self, head: int, logical: int) -> np.ndarray:
        pid = self.table.physical(head, logical)
        rows = int(self._counts(head)[logical])
        return self.v_pool[pid, :rows].to(torch.float32).cpu().numpy()

    def gather_pages(self, head: int, physical_ids) -> tuple[np.ndarray, np.ndarray]:
        """Concatenate the rows of the given pages, in the given order (kvcache.py:266-280)."""
        rows = self._owner_rows(head, physical_ids)  # ownership check
        ids = np.asarray(physical_ids, dtype=np.int64).tolist()
        D = self.layout.head_dim
        if not ids:
            empty = np.empty((0, D), dtype=np.float32)
            return empty, empty.copy()
        idx = torch.tensor(ids, dtype=torch.int64, device=self.device)
        kp = self.k_pool[idx].to(torch.float32).cpu().numpy()
        vp = self.v_pool[idx].to(torch.float32).cpu().numpy()
        ks = [kp[i, :r] for i, r in enumerate(rows)]
        vs = [vp[i, :r] for i, r in enumerate(rows)]
        return np.concatenate(ks, axis=0), np.concatenate(vs, axis=0)

    def full_kv(self, head: int) -> tuple[np.ndarray, np.ndarray]:
        """All rows of one head in logical order (kvcache.py:282-284)."""
        return self.gather_pages(head, self.table.mapping(head))

    # ------------------------------------------------------------------
    # Snapshots (UNQK v1, kvcache.py:289-341)

    def save(self, path: str) -> None:
        lengths = {self.seq_len(h) for h in range(self.num_units)}
        if len(lengths) != 1:
            raise ValueError("snapshot requires equal seq_len across heads")
        n = lengths.pop()
        with open(path, "wb") as f:
            f.write(SNAPSHOT_MAGIC)
            f.write(struct.pack("<IIIII", SNAPSHOT_VERSION, self.num_units,
                                self.layout.head_dim, self.layout.page_size, n))
            for head in range(self.num_units):
                keys, values = self.full_kv(head)
                f.write(np.ascontiguousarray(keys, dtype="<f4").tobytes())
                f.write(np.ascontiguousarray(values, dtype="<f4").tobytes())

    @classmethod
    def load(cls, path: str, extra_pages: int = 0, **kw) -> "PagedKvCache":
        with open(path, "rb") as f:
            magic = f.read(4)
            if magic != SNAPSHOT_MAGIC:
                raise ValueError(f"bad snapshot magic {magic!r}")
            version, heads, dim, size, n = struct.unpack("<IIIII", f.read(20))
            if version != SNAPSHOT_VERSION:
                raise ValueError(f"unsupported snapshot version {version}")
            pages_per_head = max(1, -(-n // size))
            layout = CacheLayout(num_kv_heads=heads, head_dim=dim, page_size=size,
                                 max_pages=heads * pages_per_head + extra_pages)
            kw.setdefault("max_pages_per_head", pages_per_head + extra_pages)
            cache = cls(layout, **kw)
            count = n * dim
            ks, vs = [], []
            for _ in range(heads):
                ks.append(np.frombuffer(f.read(4 * count), dtype="<f4").reshape(n, dim))
                vs.append(np.frombuffer(f.read(4 * count), dtype="<f4").reshape(n, dim))
        if n:
            cache.extend_units(torch.from_numpy(np.stack(ks)), torch.from_numpy(np.stack(vs)))
        return cache
