"""Bit-exact device samplers (K2) behind the reference's RNG calls.

``pcg64_state(entropy)`` reproduces ``np.random.default_rng(entropy)``'s
PCG64 seeding (SeedSequence) in the C library; ``permutation`` and ``choice``
return the exact arrays numpy 2.x's Generator.permutation /
Generator.choice(replace=False) produce for that state
(trainer.py:196-199 and 317-324), computed on the GPU.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import check, ptr, stream_ptr, u64arr


def pcg64_state(entropy) -> np.ndarray:
    """(state_hi, state_lo, inc_hi, inc_lo) of default_rng(entropy)."""
    ent, p = u64arr([int(e) for e in entropy])
    out = np.zeros(4, dtype=np.uint64)
    check(_lib.load().sptk_pcg64_seed(p, len(ent), out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))),
          "sptk_pcg64_seed")
    return out


class Workspace:
    """Grow-only device scratch buffer."""

    def __init__(self, device=None):
        self.buf = None
        self.device = device

    def get(self, nbytes: int):
        import torch

        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=self.device or "cuda")
        return self.buf


def permutation(entropy, n: int, out=None, ws: Workspace | None = None, state=None, stream=None):
    """Device int32 tensor == default_rng(entropy).permutation(n)."""
    import torch

    _lib.require_cuda()
    L = _lib.load()
    st = state if state is not None else pcg64_state(entropy)
    stc, sp = u64arr(st)
    if out is None:
        out = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    need = int(L.sptk_permutation_ws_bytes(n))
    w = (ws or Workspace()).get(need)
    check(L.sptk_permutation(sp, n, ptr(out), ptr(w), w.numel(), stream_ptr(stream)), "sptk_permutation")
    return out[:n] if n else out[:0]


def permute_records(n: int, src, rw: int, out, ws: Workspace | None = None, state=None, entropy=None,
                    perm_out=None, stream=None):
    """out[k] = src[perm[k]] for the records of one block (rw int32 words each),
    perm = default_rng(entropy).permutation(n): the visit-ordered records of
    trainer.py:196-199 (``visit = ids[perm]``) in one fused sampler call."""
    _lib.require_cuda()
    L = _lib.load()
    st = state if state is not None else pcg64_state(entropy)
    stc, sp = u64arr(st)
    w = (ws or Workspace()).get(int(L.sptk_permutation_ws_bytes(n)))
    check(L.sptk_permute_records(sp, n, ptr(src), rw, ptr(out), ptr(perm_out), ptr(w), w.numel(),
                                 stream_ptr(stream)), "sptk_permute_records")
    return out


def permutation_j(entropy, n: int, out=None, ws: Workspace | None = None, state=None, stream=None):
    """The Fisher-Yates index sequence j_i (i = 1..n-1) of permutation(n)
    (the first half of ``permutation``; ``fy_apply`` is the second)."""
    import torch

    _lib.require_cuda()
    L = _lib.load()
    stc, sp = u64arr(state if state is not None else pcg64_state(entropy))
    if out is None:
        out = torch.zeros(max(n, 1), dtype=torch.int32, device="cuda")
    w = (ws or Workspace()).get(int(L.sptk_permutation_j_ws_bytes(n)))
    check(L.sptk_permutation_j(sp, n, ptr(out), ptr(w), w.numel(), stream_ptr(stream)), "sptk_permutation_j")
    return out[:n]


def permutation_j_batch(states, ns, offsets, out, ws: Workspace | None = None, stream=None):
    """j-sequences of several permutations at once: block b (PCG64 state
    states[b], size ns[b]) into out[offsets[b] : offsets[b] + ns[b]] (the
    DSGD blocks of one process, one launch per segment phase for all)."""
    _lib.require_cuda()
    L = _lib.load()
    st, sp = u64arr(np.asarray(states, dtype=np.uint64).reshape(-1))
    nn, pn = _lib.i64arr(ns)
    oo, po = _lib.i64arr(offsets)
    w = (ws or Workspace()).get(int(L.sptk_permutation_j_batch_ws_bytes(pn, len(nn))))
    check(L.sptk_permutation_j_batch(sp, pn, po, len(nn), ptr(out), ptr(w), w.numel(), stream_ptr(stream)),
          "sptk_permutation_j_batch")
    return out


def fy_apply(j, n: int, out=None, ws: Workspace | None = None, stream=None):
    """Apply the Fisher-Yates sequence j (from ``permutation_j``; j[0] is
    overwritten) to the identity: the permutation itself."""
    import torch

    _lib.require_cuda()
    L = _lib.load()
    if out is None:
        out = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    w = (ws or Workspace()).get(int(L.sptk_fy_apply_ws_bytes(n)))
    check(L.sptk_fy_apply(ptr(j), n, ptr(out), ptr(w), w.numel(), stream_ptr(stream)), "sptk_fy_apply")
    return out[:n]


def choice(entropy, pop: int, k: int, shuffle: bool = True, out=None, ws: Workspace | None = None,
           state=None, stream=None):
    """Device int32 tensor == default_rng(entropy).choice(pop, k, replace=False)
    (shuffle=False: the same set, in Floyd draw order).  Returns (ids, path)."""
    import torch

    _lib.require_cuda()
    L = _lib.load()
    st = state if state is not None else pcg64_state(entropy)
    stc, sp = u64arr(st)
    if out is None:
        out = torch.empty(max(k, 1), dtype=torch.int32, device="cuda")
    need = int(L.sptk_choice_ws_bytes(pop, k))
    w = (ws or Workspace()).get(need)
    path = ctypes.c_int(0)
    check(L.sptk_choice(sp, pop, k, 1 if shuffle else 0, ptr(out), ptr(w), w.numel(), ctypes.byref(path),
                        stream_ptr(stream)), "sptk_choice")
    return out[:k], ("tail" if path.value == 1 else "floyd")


def u32_stream(entropy, n: int, q0: int = 0):
    import torch

    _lib.require_cuda()
    stc, sp = u64arr(pcg64_state(entropy))
    out = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    check(_lib.load().sptk_u32_stream(sp, q0, n, ptr(out), stream_ptr()), "sptk_u32_stream")
    return out[:n]


BLOCK_JOB_DTYPE = np.dtype([("off", "<i8"), ("out_base", "<i8"), ("n", "<i4"), ("first", "<i4"), ("m", "<i4"),
                            ("slot", "<i4"), ("nmin", "<i4"), ("pad", "<i4")])
BLOCK_PERM_MAX = 28000  # 8 bytes of shared memory per nonzero in one CTA (16-bit entries)


class BlockOrders:
    """Visit orders of every DSGD block of an epoch in one launch
    (sptk_block_perm): block b's default_rng([seed, 1, t, *b]).permutation(n_b)
    (trainer.py:196-199), mapped to record positions (visit = ids[perm], the
    block's records lying at [off_b, off_b + n_b) in the partitioned layout)
    and laid out round by round with the round's blocks interleaved.

    rounds: list of rounds, each a list of (block tuple, off, n)."""

    def __init__(self, rounds, order: int, device, big: bool = False, pad: int = 1):
        import torch

        # big=True: blocks above BLOCK_PERM_MAX; only the job table is built
        # and interleave() lays out visit orders drawn elsewhere
        self.big = big
        self.round_start, self.round_end = [], []
        jobs, coords, base = [], [], 0
        for rnd in rounds:
            first, m = len(jobs), len(rnd)
            if m > 64:
                raise ValueError("at most 64 blocks per round")
            nmin = min((n for _, _, n in rnd), default=0)
            for slot, (block, off, n) in enumerate(rnd):
                if n > BLOCK_PERM_MAX and not big:
                    raise ValueError(f"block of {n} nonzeros exceeds {BLOCK_PERM_MAX}")
                jobs.append((off, base, n, first, m, slot, nmin, 0))
                coords.append(tuple(int(c) for c in block))
            self.round_start.append(base)
            self.round_end.append(base + sum(n for _, _, n in rnd))
            # pad > 1: every round starts on a multiple of pad (and takes at
            # least one pad unit even when empty); the gaps stay untouched
            base += sum(n for _, _, n in rnd)
            if pad > 1:
                base = max(base, self.round_start[-1] + pad)
                base = (base + pad - 1) // pad * pad
        self.round_start.append(base)
        self.total = base
        self.group_start, self.group_end = self.round_start, self.round_end
        self.n_jobs = len(jobs)
        self.order = order
        self.cap = max([j[2] for j in jobs], default=1)
        if int(_lib.load().sptk_block_job_bytes()) != BLOCK_JOB_DTYPE.itemsize:
            raise RuntimeError("BlockJob layout mismatch between libsptk and sampler.py")
        tab = np.array(jobs, dtype=BLOCK_JOB_DTYPE)
        self.jobs = torch.from_numpy(tab.view(np.uint8).copy()).to(device)
        self.coords = torch.from_numpy(np.asarray(coords, dtype=np.int32).reshape(-1, order)).to(device)
        # j-sequence scratch (uint16, indexed like the records)
        span = max([j[0] + j[2] for j in jobs], default=1)
        self.js = None if big else torch.empty(max(span, 1), dtype=torch.int16, device=device)

    @classmethod
    def from_arrays(cls, blocks, offs, cnts, order: int, device, big: bool = False, pad: int = 1, groups=None):
        """The same table from arrays: blocks [R, M, order], offs / cnts [R, M]
        (record offset and size of each round's blocks; empty blocks are
        dropped).  Vectorised: the NF W=24 table (13,824 jobs) in ~2 ms instead
        of the ~50 ms of the tuple loops.

        groups [R] (non-decreasing group ids, optional): consecutive rounds of
        one group lie end to end without padding and the padding to ``pad``
        applies per group (group_start / group_end; by default every round is
        its own group)."""
        import torch

        self = cls.__new__(cls)
        self.big = big
        cnts = np.asarray(cnts, dtype=np.int64)
        offs = np.asarray(offs, dtype=np.int64)
        blocks = np.asarray(blocks, dtype=np.int64)
        R = cnts.shape[0]
        mask = cnts > 0
        m_r = mask.sum(axis=1)
        if (m_r > 64).any():
            raise ValueError("at most 64 blocks per round")
        if not big and cnts.max(initial=0) > BLOCK_PERM_MAX:
            raise ValueError(f"block of {int(cnts.max())} nonzeros exceeds {BLOCK_PERM_MAX}")
        sums = np.where(mask, cnts, 0).sum(axis=1)
        nmin = np.where(mask, cnts, np.iinfo(np.int64).max).min(axis=1, initial=np.iinfo(np.int64).max)
        nmin = np.where(m_r > 0, nmin, 0)
        g = np.arange(R) if groups is None else np.asarray(groups, dtype=np.int64)
        n_g = int(g.max()) + 1 if R else 0
        gsum = np.bincount(g, weights=sums, minlength=n_g).astype(np.int64) if R else np.zeros(0, np.int64)
        if pad > 1:
            gstep = np.maximum(gsum, pad)
            gstep = (gstep + pad - 1) // pad * pad
        else:
            gstep = gsum
        gstart = np.zeros(n_g + 1, dtype=np.int64)
        gstart[1:] = np.cumsum(gstep)
        excl = np.cumsum(sums) - sums  # rounds of a group lie end to end
        first_of = np.zeros(n_g, dtype=np.int64)
        first_of[g[::-1]] = np.arange(R)[::-1]
        starts = np.zeros(R + 1, dtype=np.int64)
        starts[:R] = gstart[g] + excl - excl[first_of[g]]
        starts[R] = gstart[-1]
        self.round_start = starts.tolist()
        self.round_end = (starts[:-1] + sums).tolist()
        self.group_start = gstart.tolist()
        self.group_end = (gstart[:-1] + gsum).tolist()
        self.total = int(gstart[-1])
        first = np.concatenate([[0], np.cumsum(m_r)[:-1]])
        slot = np.cumsum(mask, axis=1) - 1
        rr, cc = np.nonzero(mask)
        tab = np.zeros(len(rr), dtype=BLOCK_JOB_DTYPE)
        tab["off"] = offs[rr, cc]
        tab["out_base"] = starts[rr]
        tab["n"] = cnts[rr, cc]
        tab["first"] = first[rr]
        tab["m"] = m_r[rr]
        tab["slot"] = slot[rr, cc]
        tab["nmin"] = nmin[rr]
        self.n_jobs = len(rr)
        self.order = order
        self.cap = int(cnts.max(initial=1)) if self.n_jobs else 1
        if int(_lib.load().sptk_block_job_bytes()) != BLOCK_JOB_DTYPE.itemsize:
            raise RuntimeError("BlockJob layout mismatch between libsptk and sampler.py")
        self.jobs = torch.from_numpy(tab.view(np.uint8).copy()).to(device)
        self.coords = torch.from_numpy(np.ascontiguousarray(blocks[rr, cc], dtype=np.int32).reshape(-1, order)).to(
            device)
        span = int((offs + cnts)[mask].max(initial=1)) if self.n_jobs else 1
        self.js = None if big else torch.empty(max(span, 1), dtype=torch.int16, device=device)
        return self

    def draw(self, seed: int, t: int, out, stream=None) -> None:
        """visit orders of epoch t into out[0:total] (int32, device)."""
        check(_lib.load().sptk_block_perm(ptr(self.jobs), ptr(self.coords), self.n_jobs, self.order, int(seed),
                                          int(t), max(self.cap, 1), ptr(self.js), ptr(out), stream_ptr(stream)),
              "sptk_block_perm")

    def interleave(self, perm, rel_lo: int, out, stream=None) -> None:
        """out[0:total] = the round-interleaved visit list of per-block orders
        perm[off_b + p] (entries relative to off_b, or to rel_lo >= 0)."""
        check(_lib.load().sptk_interleave_rounds(ptr(self.jobs), self.n_jobs, ptr(perm), int(rel_lo), ptr(out),
                                                 int(max(self.cap, 1)), stream_ptr(stream)), "sptk_interleave_rounds")
