"""Pins of reading B12: ranking mode 3 orders by the
time-invariant form V + alpha*last*T of Eq.26's score (P:677-685, P:1219,
values fixed between events P:1199-1210).

- With alpha = 0 it is R3's key exactly (both are fp32(V)).
- The key does not depend on `now`: a queue that nothing touches keeps its
  keys and its order from step to step.
- In exact arithmetic V - alpha*(now - last)*T = (V + alpha*last*T) -
  alpha*now*T, so wherever the fp32 keys are distinct the mode-3 order is
  the order of the exact Eq.26 scores (brute force with Fractions).
- The hand-worked golden P11 (anti-starvation with alpha > 0,
  tests/golden/r2_pins.json) schedules identically in mode 3: its values
  and waits are exact in binary64 and distinct in fp32."""
import json
import os
import struct
from fractions import Fraction

import numpy as np
import pytest

import oracle
import tracegen
from oracle import K_IMPORT

T = 100_000
G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "r2_pins.json")))


def cfg0(cap=1_000_000):
    return dict(tracegen.PRESET_G0, g_total=1000 + cap, g_model=1000)


def inst0(B, **kw):
    return tracegen.inst_params(1, base=tracegen.INST_G0, l_static=B, **kw)


def queue(rng, n, now):
    status = rng.integers(1, 4, n)
    la = rng.integers(1, 400, n)
    lb = rng.integers(1, 60, n)
    last = rng.integers(0, now + 1, n)
    return oracle.records(n, kind=K_IMPORT, id=np.arange(n), la=la, lb=lb, flags=(status << 4) | (2 << 8),
                          last=last, pend=rng.integers(1, 50, n)), status, la, lb, last


def f32(x):
    return struct.unpack("<f", struct.pack("<f", x))[0]


def test_alpha_zero_equals_R3():
    rng = np.random.default_rng(1)
    r, *_ = queue(rng, 40, 50)
    keys = []
    for mode in (0, 3):
        st = oracle.Step(cfg0(), inst0(0, ranking=mode), 40)
        st.enqueue(0, r)
        o = st.step(50)
        keys.append((o["order"][0].tolist(), o["keys"][0].tolist()))
    assert keys[0] == keys[1]


def test_keys_do_not_depend_on_now():
    rng = np.random.default_rng(2)
    r, *_ = queue(rng, 60, 100)
    out = {}
    for mode in (0, 3):
        st = oracle.Step(cfg0(), inst0(0, ranking=mode, alpha=7.0), 60)   # static limit 0: nothing changes
        st.enqueue(0, r)
        out[mode] = [st.step(now) for now in (100, 137, 5000)]
    ti = out[3]
    assert all(x["keys"][0].tolist() == ti[0]["keys"][0].tolist() for x in ti)
    assert all(x["order"][0].tolist() == ti[0]["order"][0].tolist() for x in ti)
    r3 = out[0]
    assert r3[0]["keys"][0].tolist() != r3[2]["keys"][0].tolist()      # Eq.26's form moves with now


@pytest.mark.parametrize("seed", range(12))
def test_order_is_exact_score_order_when_keys_distinct(seed):
    rng = np.random.default_rng(100 + seed)
    n, now = 7, 400
    alpha = float(rng.choice([0.5, 3.0, 40.0]))
    r, status, la, lb, last = queue(rng, n, now)
    st = oracle.Step(cfg0(), inst0(0, ranking=3, alpha=alpha), n)
    st.enqueue(0, r)
    o = st.step(now)
    order, keys = o["order"][0].tolist(), dict(zip(o["order"][0].tolist(), o["keys"][0].tolist()))
    if len(set(keys.values())) < n:
        pytest.skip("fp32 tie: the order is by id, not by the exact score")
    # values: Stage I without a call (Eq.9-10, Discard form): pre + dec, M = 1, T = 0.1, N = 50
    Ts = Fraction(1, 10)
    def V(j):
        L, O = Fraction(int(la[j])), Fraction(int(lb[j]))
        return Fraction(1, 2) * Ts / 50 * L * L + Ts * (L * O + Fraction(1, 2) * O * O)
    exact = {j: V(j) - Fraction(alpha) * (now - int(last[j])) * Ts for j in range(n)}
    want = sorted(range(n), key=lambda j: (int(status[j]), exact[j], j))
    assert order == want


def test_P11_schedules_identically_in_mode_3():
    g = G["P11_last_on_grant_sim"]
    reqs = []
    for q in g["requests"]:
        segs = [(s[0], s[0], 0, 0.0, 0) for s in q["segs"]]
        reqs.append({"arr": q["arr"], "l_pre": q["l_pre"], "segs": segs})
    tr = tracegen.from_requests([reqs])
    rec, ft, fin = oracle.simulate_detail(cfg0(), inst0(10, alpha=1000.0, ranking=3), tr)
    assert list(ft) == g["first_token_iter"] and list(fin) == g["finish_iter"]
