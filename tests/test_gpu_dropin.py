"""Drop-in semantics of the per-party API (needs a B200).

The reference's callers see numpy uint64 shares (sharing.py:37-103), one
lockstep counter sequence per purpose with a freshness ledger
(sharing.py:190-230) and CommStats that count every round
(transport.py:52-105).  These tests pin those contracts on the B200 engine,
including the paths where the engine fuses or replays work (CUDA graphs,
one-launch chains, batch shards).
"""

import numpy as np
import pytest

from oracle import rss as R

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_2104_10949_b200 as M  # noqa: E402
from paper_2104_10949_b200 import nn  # noqa: E402
from paper_2104_10949_b200.engine import ReciprocalConfig, RssTensor, TrioSession  # noqa: E402
from paper_2104_10949_b200.prf import PURPOSE_ARITH_ZERO as ARITH  # noqa: E402
from paper_2104_10949_b200.sharing import pairwise_random, zero_share, zero_share_xor  # noqa: E402

U64 = np.uint64


def test_shares_are_numpy_uint64_and_map_accepts_numpy_functions():
    x = M.fx_encode(np.arange(12.0).reshape(3, 4) - 6)

    def job(ctx):
        xs = M.distribute_input(ctx, x if ctx.party == 0 else None, np.random.default_rng(1), shape=x.shape)
        assert isinstance(xs.lo, np.ndarray) and xs.lo.dtype == U64 and xs.hi.shape == (3, 4)
        padded = xs.map(lambda v: np.pad(v, ((1, 1), (0, 0))))  # numpy-only: runs on the host copy
        flat = xs.map(lambda v: v.reshape(-1))  # torch-compatible: stays on the device
        r = M.relu(ctx, padded)
        return M.open_share(ctx, r), M.open_share(ctx, flat)

    outs = M.run_in_process(job, seed=2)
    want = np.pad(np.where(x.view(np.int64) > 0, x, U64(0)), ((1, 1), (0, 0)))
    for opened_relu, opened_flat in outs:
        assert np.array_equal(opened_relu, want)
        assert np.array_equal(opened_flat, x.reshape(-1))


def test_counters_and_freshness_shared_with_the_engine():
    """After an engine mul (ARITH counter 0), ctx.take hands out counter 1,
    and drawing counter 0 through zero_share raises FreshnessError
    (sharing.py:198-204)."""
    x = M.fx_encode(np.ones((2, 2)))

    def job(ctx):
        xs = M.distribute_input(ctx, x if ctx.party == 0 else None, np.random.default_rng(1), shape=(2, 2))
        M.mul(ctx, xs, xs)
        j = ctx.take(ARITH)
        z = zero_share(ctx, ARITH, j, (5,))
        stale = None
        try:
            zero_share_xor(ctx, ARITH, 0, (5,))
        except M.FreshnessError as e:
            stale = e
        return j, z, stale

    res = M.run_in_process(job, seed=4)
    assert [r[0] for r in res] == [1, 1, 1]
    assert all(isinstance(r[2], M.FreshnessError) for r in res)
    # zero shares telescope to zero (sharing.py:233-240)
    assert np.array_equal(res[0][1] + res[1][1] + res[2][1], np.zeros(5, U64))


def test_per_party_counters_then_engine_stays_fresh():
    """Counters a party drew by hand are skipped by the next engine kernel."""

    def job(ctx):
        for _ in range(3):
            ctx.take(ARITH)
        w = pairwise_random(ctx, ctx.succ, ARITH, 2, (4,))
        xs = M.distribute_input(ctx, M.fx_encode(np.ones(4)) if ctx.party == 0 else None, np.random.default_rng(1),
                                shape=(4,))
        M.mul(ctx, xs, xs)
        return w, ctx.session.seq[ARITH]

    res = M.run_in_process(job, seed=4)
    assert all(r[1] == 4 for r in res)  # the engine's mul drew counter 3
    keys = R.party_keys(4)
    for p in range(3):  # party p shares k_p with its successor (sharing.py:253-267)
        assert np.array_equal(res[p][0], R.prf_words(keys[p], ARITH, 2, 4))


def test_graph_replay_charges_the_eager_step_commstats():
    s = TrioSession(0)
    model = M.lenet()
    st = nn.TrainState(s, model, M.TrainConfig(0.01, 8, 4, seed=0))
    rng = np.random.default_rng(0)
    xe = M.fx_encode(rng.uniform(0, 1, (8, 1, 28, 28)))
    ye = M.fx_encode(nn.one_hot(rng.integers(0, 10, 8), 10))
    b = [st.deal_batch(xe, ye) for _ in range(3)]
    base = [t.stats.copy() for t in s.ledger.parties]
    st.step(*b[0])
    eager = [t.stats.since(bs) for t, bs in zip(s.ledger.parties, base)]
    xs, ys = RssTensor(b[1][0].data.clone()), RssTensor(b[1][1].data.clone())
    g = st.capture(xs, ys)
    base = [t.stats.copy() for t in s.ledger.parties]
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    replayed = [t.stats.since(bs) for t, bs in zip(s.ledger.parties, base)]
    for e, r in zip(eager, replayed):
        assert r.rounds == 2 * e.rounds
        assert r.round_labels == e.round_labels * 2
        assert r.payload_bytes_sent() == 2 * e.payload_bytes_sent()


def test_long_reciprocal_chain_runs_unfused_and_matches_oracle():
    """ReciprocalConfig(iterations=20) exceeds one chain launch (48 steps):
    it runs as separate mul+truncate launches with the same counters."""
    rng = np.random.default_rng(3)
    y = R.share(R.fx_encode(rng.uniform(1, 150, 33)), rng)
    s = TrioSession(6)
    got = s.reciprocal(s.from_components(y), ReciprocalConfig(200.0, 20))
    ref = R.reciprocal(R.Session(6), y, 200.0, 20)
    assert np.array_equal(got.data.cpu().numpy().view(U64), ref)
    short = TrioSession(6).reciprocal(TrioSession(6).from_components(y), ReciprocalConfig(200.0, 13))
    assert np.array_equal(short.data.cpu().numpy().view(U64), R.reciprocal(R.Session(6), y, 200.0, 13))


def test_bit_inject_batch_shard_draws_global_words():
    from paper_2104_10949_b200.nn import DataParallel

    rng = np.random.default_rng(9)
    bits = rng.integers(0, 2, (3, 8, 5), dtype=U64)
    s = TrioSession(2)
    full = s.bit_inject(s.from_components(bits)).data.cpu().numpy().view(U64)
    assert np.array_equal(full, R.bit_inject(R.Session(2), bits))
    for r in range(2):
        sh = TrioSession(2)
        sh.dp = DataParallel(r, 2, None)
        part = sh.bit_inject(sh.from_components(np.ascontiguousarray(bits[:, 4 * r:4 * r + 4])))
        assert np.array_equal(part.data.cpu().numpy().view(U64), full[:, 4 * r:4 * r + 4])


def test_frozen_weights_repack_after_inplace_sgd():
    """Packed weight operands cached under frozen_weights are dropped when
    the in-place SGD kernel rewrites the parameters."""
    rng = np.random.default_rng(1)
    s = TrioSession(1)
    x = s.share(M.fx_encode(rng.uniform(-1, 1, (4, 6))), rng)
    w = s.share(M.fx_encode(rng.uniform(-1, 1, (6, 5))), rng)
    g = s.share(M.fx_encode(rng.uniform(-1, 1, (6, 5))), rng)
    with s.frozen_weights():
        s.matmul(x, w)
        s.sgd_inplace([w], [g], int(M.fx_encode(0.5)))
        seq = dict(s.seq)
        after = s.matmul(x, w)
    fresh = TrioSession(1)
    fresh.rewind(seq)
    want = fresh.matmul(x, w)
    assert np.array_equal(after.data.cpu().numpy(), want.data.cpu().numpy())
