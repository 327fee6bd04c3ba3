"""augsched_generate (the device twin of tracegen/tablegen.py, SURVEY §8(f)
f3): generated traces equal the host generator's bit for bit for W1, W2 and
W3 recipes, and simulating device-generated traces equals the oracle on the
host-generated ones."""
import numpy as np
import pytest

import oracle
import tracegen
from tracegen import tablegen as tg

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_04013_b200 as aug  # noqa: E402

CASES = {
    "w2_bucket": (dict(), 11, 5, 3000, [2.0, 3.0, 4.0, 5.0, 8.0], 0),
    "w1_oracle_nocall": (dict(predictor="oracle", p_nocall=0.3), 12, 3, 20000, [4.0, 6.0, 1.0], 1800 * 10**6),
    "w3_cv2": (dict(cv=2.0), 13, 4, 20000, [2.0, 4.0], 1800 * 10**6),
    "w3_cv05_short": (dict(cv=0.5, accuracy=0.85), 14, 2, 700, [3.0], 60 * 10**6),
}


@pytest.mark.parametrize("name", list(CASES))
def test_device_traces_equal_host_traces(name):
    kw, seed, n_traces, n_max, rates, horizon = CASES[name]
    T = tg.build_tables(**kw)
    host = tg.generate(T, seed, n_traces, n_max, rates, horizon_ticks=horizon)
    s = aug.Scheduler(tracegen.PRESET_7B, tracegen.inst_params(1), 1, 8)
    dev = aug.GeneratedTraces(s, T, seed, n_traces, n_max, rates, horizon_ticks=horizon)
    g = dev.to_numpy()
    s.close()
    for k, v in host.arrays().items():
        assert g[k].dtype == v.dtype and np.array_equal(g[k], v), f"{name}: {k}"


def test_simulate_on_generated_traces_equals_oracle():
    T = tg.build_tables(cv=1.5)
    seed, n_traces, n_max, rates, horizon = 21, 3, 400, [3.0, 5.0, 8.0], 120 * 10**6
    host = tg.generate(T, seed, n_traces, n_max, rates, horizon_ticks=horizon)
    ip = tracegen.inst_params(6, ranking=[0, 1, 2, 0, 0, 1], rank_seed=5, budget_mode=[0, 1, 0, 0, 1, 0])
    tid = np.array([0, 0, 1, 1, 2, 2], np.uint32)
    ma = int(np.diff(host.req_off).max())
    s = aug.Scheduler(tracegen.PRESET_7B, ip, 6, ma)
    dev = aug.GeneratedTraces(s, T, seed, n_traces, n_max, rates, horizon_ticks=horizon)
    out = s.simulate(dev, torch.from_numpy(tid.astype(np.int32)).cuda())
    g = aug.results_to_numpy(out)
    s.sync()
    s.close()
    o = oracle.simulate(tracegen.PRESET_7B, ip, host, tid)
    assert g.tobytes() == o.tobytes()
