"""K2 samplers on the GPU: bit-exact against the reference's numpy draws."""

import hashlib

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def h32(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<i4").tobytes()).hexdigest()


def test_seed_states(golden, golden_meta):
    from paper_2204_07104_b200.sampler import pcg64_state

    for i in range(golden_meta["n_entropies"]):
        assert np.array_equal(pcg64_state(golden[f"rng_entropy_{i}"].tolist()), golden[f"rng_state_{i}"])


@pytest.mark.parametrize("q0", [0, 1, 7, 1000001])
def test_u32_stream(q0):
    from paper_2204_07104_b200.sampler import u32_stream

    got = u32_stream([3, 1, 4], 5000, q0=q0).cpu().numpy().view(np.uint32)
    want = O.u32_stream(O.pcg64_state([3, 1, 4]), q0 + 5000)[q0:]
    assert np.array_equal(got, want)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 17, 100, 1000, 4097, 65536, 100_003])
def test_permutation_golden(golden, n):
    from paper_2204_07104_b200.sampler import permutation

    ent = golden[f"perm_{n}_ent"].tolist()
    assert np.array_equal(permutation(ent, n).cpu().numpy(), golden[f"perm_{n}"])


@pytest.mark.parametrize("n", [2, 3, 4, 9, 33, 4096, 8191, 8192, 8193, 70_000, 262_145, 1_000_003])
def test_permutation_j_sequence(n):
    from paper_2204_07104_b200.sampler import permutation_j

    ent = [11, 1, n]
    got = permutation_j(ent, n).cpu().numpy()
    _, want = O.permutation(ent, n, return_j=True)
    assert np.array_equal(got[1:], want[1:])


@pytest.mark.parametrize("n", [50_000, 3_000_017])
def test_permutation_random_seeds(n):
    from paper_2204_07104_b200.sampler import permutation

    for s in range(3):
        ent = [s, 1, 2, 0, 1]
        assert np.array_equal(permutation(ent, n).cpu().numpy(), O.permutation(ent, n))


def test_permutation_large_hashes(golden_meta):
    from paper_2204_07104_b200.sampler import permutation

    for key in ("perm_1048576", "perm_3000017", "perm_12345678"):
        g = golden_meta["big"][key]
        p = permutation(g["entropy"], g["n"]).cpu().numpy()
        assert p[:64].tolist() == g["head"]
        assert h32(p) == g["sha256_i32"]


def test_permutation_netflix_size(golden_meta):
    """The factor-phase visit order of the Netflix-shaped bench (99,072,112
    nonzeros, seed 1, epochs 0 and 1) equals numpy's."""
    from paper_2204_07104_b200.sampler import permutation

    for t in range(2):
        g = golden_meta["big"][f"perm_NF_t{t}"]
        p = permutation(g["entropy"], g["n"]).cpu().numpy()
        assert p[:64].tolist() == g["head"] and p[-64:].tolist() == g["tail"]
        assert h32(p) == g["sha256_i32"]


@pytest.mark.parametrize("pop,k", [(100, 10), (10000, 9000), (10001, 9000), (500_000, 5000),
                                   (500_000, 20_000), (4_000_000, 1 << 20), (200, 200)])
def test_choice_golden(golden, pop, k):
    from paper_2204_07104_b200.sampler import choice

    ent = golden[f"choice_{pop}_{k}_ent"].tolist()
    got, path = choice(ent, pop, k, shuffle=True)
    assert np.array_equal(got.cpu().numpy(), golden[f"choice_{pop}_{k}"])
    got_set, _ = choice(ent, pop, k, shuffle=False)
    assert np.array_equal(np.sort(got_set.cpu().numpy()), np.sort(golden[f"choice_{pop}_{k}"]))


def test_choice_edge_cases():
    from paper_2204_07104_b200.sampler import choice

    for pop, k in [(1, 1), (5, 5), (7, 0), (10000, 200), (10001, 201), (20001, 401), (30000, 29999)]:
        ent = [5, 2, pop, k]
        got, _ = choice(ent, pop, k, shuffle=True)
        want, _ = O.choice(ent, pop, k)
        assert np.array_equal(got.cpu().numpy(), want), (pop, k)


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("pop,k", [(3_000_000, 60_000), (1_000_000, 500_000), (2_000_001, 40_000)])
def test_choice_parallel_walk_vs_oracle(seed, pop, k):
    """Draw counts where the chunked parallel Lemire walk runs (both choice paths,
    and the _shuffle_int walk after Floyd): identical to the oracle."""
    from paper_2204_07104_b200.sampler import choice

    ent = [11, seed, pop, k]
    got, _ = choice(ent, pop, k, shuffle=True)
    want, _ = O.choice(ent, pop, k)
    assert np.array_equal(got.cpu().numpy(), want)


def test_choice_parallel_walk_fallback(monkeypatch):
    """A window too narrow for the true rejection offsets makes the parallel
    walk hand over to the sequential walker: same draws."""
    from paper_2204_07104_b200.sampler import choice

    ent = [11, 7, 3_000_000, 60_000]
    want, _ = O.choice(ent, 3_000_000, 60_000)
    monkeypatch.setenv("SPTK_LP_W", "1")
    got, _ = choice(ent, 3_000_000, 60_000, shuffle=True)
    assert np.array_equal(got.cpu().numpy(), want)


def test_choice_netflix_core_batch(golden_meta):
    """Psi = choice(99,072,112, 2^20) of the bench (Floyd path), exact order and set."""
    from paper_2204_07104_b200.sampler import choice

    for t in range(2):
        g = golden_meta["big"][f"psi_NF_t{t}"]
        got, path = choice(g["entropy"], g["pop"], g["k"], shuffle=True)
        got = got.cpu().numpy()
        assert path == "floyd"
        assert got[:64].tolist() == g["head"]
        assert h32(got) == g["sha256_i32"]
        s, _ = choice(g["entropy"], g["pop"], g["k"], shuffle=False)
        assert h32(np.sort(s.cpu().numpy())) == g["sha256_sorted_i32"]


@pytest.mark.parametrize("n,order", [(1, 3), (2, 3), (100, 3), (65536, 3), (1_000_003, 3), (70_001, 4),
                                     (40_000, 6)])
def test_permute_records_equals_visit_gather(n, order):
    """sptk_permute_records: the block's records in the order of
    default_rng(entropy).permutation(n) (trainer.py:196-199), bit for bit,
    together with the permutation itself."""
    import torch

    from paper_2204_07104_b200.device import DeviceCoo
    from paper_2204_07104_b200.sampler import permute_records

    rng = np.random.default_rng(n)
    idx = rng.integers(0, 1 << 20, (n, order))
    vals = rng.normal(size=n)
    recs = DeviceCoo(idx, vals)
    out = torch.empty_like(recs.rec)
    perm = torch.empty(n, dtype=torch.int32, device="cuda")
    ent = [7, 1, 3, n]
    permute_records(n, recs.rec, recs.rw, out, entropy=ent, perm_out=perm)
    want = O.permutation(ent, n)
    assert np.array_equal(perm.cpu().numpy(), want)
    src = recs.rec.view(-1, recs.rw).cpu().numpy()
    assert np.array_equal(out.view(-1, recs.rw).cpu().numpy(), src[want])


def test_permute_records_netflix_size(golden_meta):
    """The fused gather at the bench size: the permutation it applies is numpy's."""
    import torch

    from paper_2204_07104_b200.sampler import permute_records

    g = golden_meta["big"]["perm_NF_t0"]
    n = g["n"]
    src = torch.arange(n, dtype=torch.int32, device="cuda").repeat_interleave(4)
    out = torch.empty_like(src)
    permute_records(n, src, 4, out, entropy=g["entropy"])
    p = out.view(-1, 4)[:, 0].cpu().numpy()
    assert p[:64].tolist() == g["head"] and p[-64:].tolist() == g["tail"]
    assert h32(p) == g["sha256_i32"]


def test_permutation_j_batch_equals_per_block():
    """The batched j-generation (a rank's DSGD blocks, segment levels in lock
    step) gives every block exactly its own permutation's j-sequence, for
    blocks of different sizes (including tiny and empty ones)."""
    import torch

    from paper_2204_07104_b200.sampler import pcg64_state, permutation_j_batch

    ns = [193_001, 1, 0, 17, 5000, 262_145, 70_000, 193_777]
    offs = np.concatenate([[0], np.cumsum(ns)[:-1]])
    ents = [[1, 1, 0, b, 3] for b in range(len(ns))]
    states = np.stack([pcg64_state(e) for e in ents])
    out = torch.zeros(int(sum(ns)) + 1, dtype=torch.int32, device="cuda")
    permutation_j_batch(states, ns, offs, out)
    got = out.cpu().numpy()
    for n, o, e in zip(ns, offs, ents):
        if n < 2:
            continue
        _, want = O.permutation(e, n, return_j=True)
        assert np.array_equal(got[o + 1:o + n], want[1:]), n


def _interleave_reference(rounds, perms):
    """Host restatement of the flattened DSGD visit list: per round, the
    blocks' visit lists (off + perm) interleaved position by position."""
    out = []
    for rnd, prs in zip(rounds, perms):
        longest = max((n for _, _, n in rnd), default=0)
        for p in range(longest):
            for (block, off, n), pr in zip(rnd, prs):
                if p < n:
                    out.append(off + pr[p])
    return np.array(out, dtype=np.int64)


@pytest.mark.parametrize("order,sizes_seed", [(3, 0), (4, 1), (2, 2)])
def test_block_perm_matches_reference(order, sizes_seed):
    """sptk_block_perm: every block's permutation equals
    default_rng([seed,1,t,*block]).permutation(n) (via the pinned oracle),
    placed at the round-interleaved slots."""
    import torch

    from paper_2204_07104_b200.sampler import BlockOrders

    rng = np.random.default_rng(sizes_seed)
    rounds, off = [], 0
    for r in range(5):
        rnd = []
        for s in range(int(rng.integers(1, 9))):
            n = int(rng.choice([0, 1, 2, 3, 17, 255, 256, 257, 1000, 4097, 17000]))
            block = tuple(int(x) for x in rng.integers(0, 9, order))
            rnd.append((block, off, n))
            off += n
        rounds.append(rnd)
    bo = BlockOrders(rounds, order, "cuda")
    out = torch.full((max(bo.total, 1),), -1, dtype=torch.int32, device="cuda")
    seed, t = 12345, 3
    bo.draw(seed, t, out)
    got = out[:bo.total].cpu().numpy().astype(np.int64)
    perms = [[O.permutation([seed, 1, t, *block], n) if n else np.zeros(0, np.int64) for block, _, n in rnd]
             for rnd in rounds]
    np.testing.assert_array_equal(got, _interleave_reference(rounds, perms))


@pytest.mark.parametrize("big", [18000, 24811, 28000])
def test_block_perm_max_block(big):
    """The largest blocks one CTA takes (up to 28,000 nonzeros: 8 bytes of
    shared memory each; NF at W = 16 has ~24.2K per block), bit-exact."""
    import torch

    from paper_2204_07104_b200.sampler import BlockOrders

    rounds = [[((3, 1, 4), 0, big), ((2, 7, 1), big, 1)]]
    bo = BlockOrders(rounds, 3, "cuda")
    out = torch.empty(bo.total, dtype=torch.int32, device="cuda")
    bo.draw(7, 0, out)
    perms = [[O.permutation([7, 1, 0, 3, 1, 4], big), O.permutation([7, 1, 0, 2, 7, 1], 1)]]
    np.testing.assert_array_equal(out.cpu().numpy().astype(np.int64), _interleave_reference(rounds, perms))


@pytest.mark.parametrize("pad", [1, 128])
def test_block_orders_padding_and_interleave(pad):
    """Padded rounds (the fused DSGD layout: every round on a multiple of 128,
    empty rounds one padding unit, gaps untouched) and sptk_interleave_rounds
    (the same layout from per-block orders in the partitioned layout) agree
    with the host restatement."""
    import torch

    from paper_2204_07104_b200.sampler import BlockOrders

    rng = np.random.default_rng(4)
    rounds, off = [], 0
    for r in range(6):
        rnd = []
        for s in range(int(rng.integers(0, 4))):
            n = int(rng.choice([1, 5, 300, 2000]))
            rnd.append((tuple(int(x) for x in rng.integers(0, 9, 3)), off, n))
            off += n
        rounds.append(rnd)
    bo = BlockOrders(rounds, 3, "cuda", pad=pad)
    out = torch.full((max(bo.total, 1),), -1, dtype=torch.int32, device="cuda")
    bo.draw(99, 1, out)
    perms = [[O.permutation([99, 1, 1, *block], n) for block, _, n in rnd] for rnd in rounds]
    want = np.full(bo.total, -1, dtype=np.int64)
    for r, (rnd, prs) in enumerate(zip(rounds, perms)):
        seg = _interleave_reference([rnd], [prs])
        assert bo.round_end[r] - bo.round_start[r] == len(seg)
        want[bo.round_start[r]: bo.round_start[r] + len(seg)] = seg
        if pad > 1:
            assert bo.round_start[r] % pad == 0 and bo.round_start[r + 1] > bo.round_start[r]
    np.testing.assert_array_equal(out[:bo.total].cpu().numpy().astype(np.int64), want)
    # the interleave kernel from per-block orders (entries relative to off_b)
    flat = np.zeros(off, dtype=np.int32)
    for rnd, prs in zip(rounds, perms):
        for (block, o, n), pr in zip(rnd, prs):
            flat[o: o + n] = pr
    big = BlockOrders(rounds, 3, "cuda", big=True, pad=pad)
    out2 = torch.full((max(big.total, 1),), -1, dtype=torch.int32, device="cuda")
    big.interleave(torch.from_numpy(flat).cuda(), -1, out2)
    np.testing.assert_array_equal(out2[:big.total].cpu().numpy().astype(np.int64), want)
