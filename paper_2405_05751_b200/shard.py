"""Multi-GPU sharding of the Z_p×Z_q verifier.

Candidates are independent units (``SPEC.md:467-468``: rounds independent,
RNG stream per (seed, round)), so verification shards by candidate index
with no data-path collective.  Each rank verifies a contiguous index range
and writes packed accept bits (bit k set iff candidate k is Equivalent);
one ``all_gather`` of the packed words at the end reassembles the global
bit vector on every rank (NCCL over NVLink on the GPU box, gloo in the CPU
tests).

Partitioning is by cumulative estimated cost, not by count: per-candidate
cost varies ~60x across families (``op_madds`` x expected attempts), and
contiguous ranges keep each rank's pool slice and the seed rule
``candidate i -> seed i`` intact.

Several candidate families (pools) verified in one step share ONE packed
word space (:class:`WordLayout`: family f owns words [base_f, base_f +
ceil(n_f / 32))), so a rank's share is one contiguous word range and the
step ends with a single all-gather of one buffer (:func:`gather_words`),
whatever the number of families.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np


def even_range(n_total: int, world: int, rank: int, align: int = 32) -> Tuple[int, int]:
    """Contiguous [first, first + n) of ``n_total`` for ``rank``; shard
    boundaries are multiples of ``align`` so packed accept words never
    straddle ranks."""
    units = -(-n_total // align)
    per, extra = divmod(units, world)
    u0 = rank * per + min(rank, extra)
    u1 = u0 + per + (1 if rank < extra else 0)
    first, last = min(u0 * align, n_total), min(u1 * align, n_total)
    return first, last - first


def cost_ranges(costs: Sequence[float], world: int, align: int = 32) -> List[Tuple[int, int]]:
    """Contiguous ranges [(first, n)] over candidates with per-candidate
    ``costs`` such that every rank gets ~1/world of the total cost.  Cuts are
    placed on ``align`` boundaries (packed-bit words)."""
    c = np.asarray(costs, dtype=np.float64)
    n = len(c)
    if world <= 1 or n == 0:
        return [(0, n)] + [(n, 0)] * (world - 1)
    words = -(-n // align)
    wc = np.add.reduceat(np.pad(c, (0, words * align - n)), np.arange(0, words * align, align))
    cum = np.cumsum(wc)
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):
        w = int(np.searchsorted(cum, total * r / world, side="left")) + 1
        cuts.append(max(cuts[-1], min(w, words)))
    cuts.append(words)
    out = []
    for r in range(world):
        a, b = min(cuts[r] * align, n), min(cuts[r + 1] * align, n)
        out.append((a, b - a))
    return out


def pack_bits(accept: Sequence[bool]) -> np.ndarray:
    """bool per candidate -> little-endian packed uint32 words (bit k of word
    k // 32), the layout ``tpo_gpu_verify_pool`` writes to ``accept_dev``."""
    a = np.asarray(accept, dtype=bool)
    pad = (-len(a)) % 32
    return np.packbits(np.pad(a, (0, pad)), bitorder="little").view(np.uint32)


def unpack_bits(words: np.ndarray, n: int) -> np.ndarray:
    return np.unpackbits(np.ascontiguousarray(words).view(np.uint8), bitorder="little")[:n].astype(bool)


def gather_accept(local_words, ranges: List[Tuple[int, int]], n_total: int, dist=None):
    """All-gather every rank's packed words (a 1-D int32 torch tensor of
    ceil(n_r / 32) words) and reassemble the global accept vector (numpy
    bool[n_total]).  Shards are padded to the longest so the collective
    has equal-size buffers; ``dist`` is ``torch.distributed`` (or None for
    a single rank)."""
    import torch
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return unpack_bits(local_words.cpu().numpy(), n_total)
    world = dist.get_world_size()
    wmax = max(-(-n // 32) for _, n in ranges)
    buf = torch.zeros(wmax, dtype=torch.int32, device=local_words.device)
    buf[: local_words.numel()] = local_words
    outs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf)
    res = np.zeros(n_total, dtype=bool)
    for r, (first, n) in enumerate(ranges):
        if n:
            res[first:first + n] = unpack_bits(outs[r].cpu().numpy(), n)
    return res


class WordLayout:
    """Packed accept words of several candidate families in one index space:
    family f (n_f candidates) owns words [base[f], base[f] + words[f]); bit
    k of family f lives in word base[f] + k // 32."""

    def __init__(self, counts: Sequence[int]):
        self.counts = [int(c) for c in counts]
        self.words = [-(-c // 32) for c in self.counts]
        self.base = [int(x) for x in np.concatenate([[0], np.cumsum(self.words)[:-1]])] if counts else []
        self.total_words = int(sum(self.words))

    def word_costs(self, per_candidate_cost: Sequence[float]) -> np.ndarray:
        """Cost of every word from a per-family cost per candidate."""
        wc = np.zeros(self.total_words)
        for f, (c, n) in enumerate(zip(per_candidate_cost, self.counts)):
            k = np.full(self.words[f], 32.0)
            if n % 32:
                k[-1] = n % 32
            wc[self.base[f]: self.base[f] + self.words[f]] = k * float(c)
        return wc

    def rank_words(self, word_costs: Sequence[float], world: int) -> List[Tuple[int, int]]:
        """Contiguous word ranges [(w0, nw)] per rank, balanced by cost."""
        wc = np.asarray(word_costs, dtype=np.float64)
        if world <= 1:
            return [(0, self.total_words)]
        cum = np.cumsum(wc)
        total = cum[-1] if len(cum) else 0.0
        cuts = [0]
        for r in range(1, world):
            w = int(np.searchsorted(cum, total * r / world, side="left")) + 1 if total > 0 else \
                (self.total_words * r) // world
            cuts.append(max(cuts[-1], min(w, self.total_words)))
        cuts.append(self.total_words)
        return [(cuts[r], cuts[r + 1] - cuts[r]) for r in range(world)]

    def jobs(self, w0: int, nw: int) -> List[Tuple[int, int, int, int]]:
        """The verify_pool calls of a rank owning words [w0, w0 + nw):
        (family, first candidate, candidates, word offset in the local buffer)."""
        out = []
        for f in range(len(self.counts)):
            a, b = max(w0, self.base[f]), min(w0 + nw, self.base[f] + self.words[f])
            if a >= b:
                continue
            first = (a - self.base[f]) * 32
            last = min((b - self.base[f]) * 32, self.counts[f])
            out.append((f, first, last - first, a - w0))
        return out

    def unpack(self, words: np.ndarray) -> List[np.ndarray]:
        """Global word vector -> per-family bool accept arrays."""
        w = np.ascontiguousarray(words).view(np.uint32)
        return [unpack_bits(w[self.base[f]: self.base[f] + self.words[f]], n)
                for f, n in enumerate(self.counts)]


def gather_words(local_words, ranges: List[Tuple[int, int]], dist=None):
    """The step's single collective: all-gather every rank's word range
    (1-D int32 tensor, padded to the longest range) and return the global
    word vector on the device (no host traffic; unpack it afterwards)."""
    import torch
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return local_words
    world = dist.get_world_size()
    wmax = max(max(nw for _, nw in ranges), 1)
    buf = torch.zeros(wmax, dtype=torch.int32, device=local_words.device)
    buf[: local_words.numel()] = local_words
    outs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf)
    return torch.cat([outs[r][:nw] for r, (_, nw) in enumerate(ranges)])
