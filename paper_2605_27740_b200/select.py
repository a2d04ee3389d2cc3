"""Top-k page selection over bf16 scores (reference select.py:1-150).

Keys: a bf16 pattern with the sign set maps to its complement, otherwise the sign
bit is set, so unsigned key order == float order (NaN rejected).  The pick is the
K3 kernel (csrc/topk.cu): two 8-bit radix histogram rounds plus an ordered
compaction that gives ties at the threshold to the lowest logical page index,
then the logical->physical translation through the page table.

The reference switches to a stable argsort beyond ``STAGED_MAX_PAGES``; the GPU
pick produces the identical set for every P it supports, so ``topk_fallback``
runs the same kernel and only the regime/passes labels differ.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import backend
from .bf16 import bf16_to_f32, is_nan_bf16

REGISTER_MAX_PAGES = 4096
STAGED_MAX_PAGES = 23 * 1024

__all__ = [
    "REGISTER_MAX_PAGES",
    "STAGED_MAX_PAGES",
    "TopKSelection",
    "decode_ordered",
    "encode_ordered",
    "radix_topk",
    "topk_fallback",
]


@dataclass
class TopKSelection:
    """Selected pages of one head; ids are physical and unordered (select.py:37-48)."""

    physical_ids: np.ndarray  # (k,) int64
    kth_score: float
    kplus1_score: float | None
    regime: str
    passes: int | None

    def __len__(self) -> int:
        return int(self.physical_ids.shape[0])


def encode_ordered(bits) -> np.ndarray:
    """bf16 bit patterns -> order-preserving uint16 keys."""
    b = np.asarray(bits, dtype=np.uint16)
    if is_nan_bf16(b).any():
        raise ValueError("cannot order NaN scores")
    neg = (b >> 15).astype(bool)
    return np.where(neg, np.invert(b), np.bitwise_or(b, np.uint16(0x8000))).astype(np.uint16)


def decode_ordered(keys) -> np.ndarray:
    """Inverse of :func:`encode_ordered`."""
    k = np.asarray(keys, dtype=np.uint16)
    pos = (k >> 15).astype(bool)
    return np.where(pos, np.bitwise_and(k, np.uint16(0x7FFF)), np.invert(k)).astype(np.uint16)


def key_to_score(key: int) -> float:
    """Ordered key -> the bf16 score value it encodes, as a float."""
    return float(bf16_to_f32(decode_ordered(np.uint16(key))))


def _regime(n_pages: int) -> str:
    if n_pages <= REGISTER_MAX_PAGES:
        return "registers"
    return "staged" if n_pages <= STAGED_MAX_PAGES else "fallback"


def _checked_keys(scores, k: int) -> np.ndarray:
    if k < 1:
        raise ValueError("k must be at least 1")
    keys = encode_ordered(scores.scores_bf16)
    if keys.shape[0] == 0:
        raise ValueError("no pages to select from")
    return keys


def _pick(scores, k: int, table, head: int, fallback: bool) -> TopKSelection:
    keys = _checked_keys(scores, k)
    P = keys.shape[0]
    mapping = table.mapping(head)
    if P <= k:  # every page (select.py:75-84)
        regime = "fallback" if (fallback and P > STAGED_MAX_PAGES) else _regime(P)
        return TopKSelection(physical_ids=np.array(mapping, dtype=np.int64, copy=True),
                             kth_score=key_to_score(int(keys.min())), kplus1_score=None,
                             regime=regime, passes=None if fallback else 1)
    ids, kth, kp1, passes = backend.radix_select_desc(keys, k)
    beyond = P > STAGED_MAX_PAGES
    return TopKSelection(
        physical_ids=np.asarray(mapping, dtype=np.int64)[ids],
        kth_score=key_to_score(kth),
        kplus1_score=key_to_score(kp1),
        regime="fallback" if (fallback or beyond) else _regime(P),
        passes=None if (fallback or beyond) else int(passes),
    )


def radix_topk(scores, k: int, table, head: int) -> TopKSelection:
    """The k highest-scoring pages, ties to the lowest logical index (select.py:87-115)."""
    return _pick(scores, k, table, head, fallback=False)


def topk_fallback(scores, k: int, table, head: int) -> TopKSelection:
    """Same selection labelled as the reference's sort fallback (select.py:118-150)."""
    return _pick(scores, k, table, head, fallback=True)
