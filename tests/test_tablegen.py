"""The counter-based, table-driven workload generator (tracegen/tablegen.py;
SURVEY §8(f) f3): determinism, the W1/W2/W3 arrival processes of P:884 and
the recipe's distributions, on the host.  Its device twin (augsched_generate)
is checked bit for bit against it in tests/test_gpu_generate.py."""
import numpy as np

from tracegen import tablegen as tg


def test_mix64_is_splitmix64():
    assert int(tg.mix64(np.uint64(0))) == 0xE220A8397B1DCDAF
    assert int(tg.mix64(np.uint64(1))) == 0x910A2DEC89025CC1


def test_deterministic_and_seeded():
    T = tg.build_tables()
    a = tg.generate(T, 7, 3, 500, [2.0, 4.0, 8.0])
    b = tg.generate(T, 7, 3, 500, [2.0, 4.0, 8.0])
    c = tg.generate(T, 8, 3, 500, [2.0, 4.0, 8.0])
    for k in a.arrays():
        assert np.array_equal(a.arrays()[k], b.arrays()[k]), k
    assert not np.array_equal(a.l_pre, c.l_pre)


def test_w2_counts_and_poisson_rate():
    T = tg.build_tables()
    tr = tg.generate(T, 1, 4, 20000, [1.0, 2.0, 4.0, 8.0])
    assert list(tr.req_off) == [0, 20000, 40000, 60000, 80000]
    for k, rate in enumerate([1.0, 2.0, 4.0, 8.0]):
        arr = tr.arr_tick[tr.req_off[k]:tr.req_off[k + 1]].astype(np.int64)
        gaps = np.diff(np.concatenate([[0], arr]))
        assert abs(1e6 / gaps.mean() / rate - 1) < 0.03
        assert abs(gaps.std() / gaps.mean() - 1) < 0.05        # exponential: CV 1
        assert np.all(np.diff(arr) >= 0)


def test_w3_gamma_cv_and_w1_horizon():
    horizon = 1800 * 10**6                                     # 30 minutes
    for cv in (0.5, 2.0, 3.0):
        T = tg.build_tables(cv=cv)
        tr = tg.generate(T, 3, 2, 40000, [4.0, 2.0], horizon_ticks=horizon)
        for k in range(2):
            arr = tr.arr_tick[tr.req_off[k]:tr.req_off[k + 1]].astype(np.int64)
            assert arr[-1] <= horizon
            gaps = np.diff(np.concatenate([[0], arr]))
            assert abs(gaps.std() / gaps.mean() / cv - 1) < 0.12
        # the cut is exactly "arrivals at or before the horizon"
        full = tg.generate(T, 3, 1, 40000, [4.0])
        n = int(tr.req_off[1])
        assert full.arr_tick[n - 1] <= horizon < full.arr_tick[n]


def test_recipe_distributions():
    T = tg.build_tables()
    tr = tg.generate(T, 5, 2, 50000, [4.0])
    assert abs(np.median(tr.l_pre) - 400) <= 8
    assert 8 <= tr.l_pre.min() and tr.l_pre.max() <= 4096
    assert 1 <= tr.gen_true.min() and tr.gen_true.max() <= 1024
    # calls per request: mixture of U{1..4}, U{1..3}, U{1..3}, U{2..5} with shares .25/.30/.25/.20
    calls = tr.n_seg.astype(np.int64) - 1
    assert abs(calls.mean() - (0.25 * 2.5 + 0.30 * 2 + 0.25 * 2 + 0.20 * 3.5)) < 0.03
    # bucket predictor hit rate 0.65
    b_true = np.searchsorted(tg.BUCKET_EDGES, tr.gen_true, side="right") - 1
    b_pred = np.searchsorted(tg.BUCKET_MID, tr.gen_pred)
    assert abs((b_true == b_pred).mean() - 0.65) < 0.01
    last = np.zeros(tr.gen_true.shape[0], bool)
    last[tr.seg_off.astype(np.int64) + tr.n_seg.astype(np.int64) - 1] = True
    assert not tr.dur_true[last].any() and not tr.ret_len[last].any() and not tr.dur_pred[last].any()
    assert tr.dur_true[~last].min() >= 1


def test_oracle_predictor_and_no_call_share():
    T = tg.build_tables(predictor="oracle", p_nocall=0.3)
    tr = tg.generate(T, 9, 1, 20000, [4.0])
    assert np.array_equal(tr.gen_true, tr.gen_pred)
    assert abs((tr.n_seg == 1).mean() - 0.3) < 0.02
