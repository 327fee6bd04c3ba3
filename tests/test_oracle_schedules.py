"""Pins of the oracle's scheduler loop (Algorithm 1) against the
hand-worked schedules of SURVEY §8(c).3 (tests/golden/survey_schedules.json),
brute force on tiny queues, closed forms and invariants (§8(c).4)."""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
import tracegen
from oracle import K_NEW, K_IMPORT

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "survey_schedules.json")))
T = 100_000  # cfg0: 0.1 s per iteration


def cfg0(cap=1_000_000):
    return dict(tracegen.PRESET_G0, g_total=1000 + cap, g_model=1000)


def inst0(B, **kw):
    return tracegen.inst_params(1, base=tracegen.INST_G0, l_static=B, **kw)


def req(arr, l_pre, segs):
    """segs: [(gen_true, dur_true_ticks, dur_pred_s, ret_len), ..., (gen_true,)];
    oracle predictor: gen_pred = gen_true."""
    out = []
    for s in segs:
        if len(s) == 1:
            out.append((s[0], s[0], 0, 0.0, 0))
        else:
            out.append((s[0], s[0], s[1], s[2], s[3]))
    return {"arr": arr, "l_pre": l_pre, "segs": out}


# ---------------------------------------------------------------- G3 (one step)
@pytest.mark.parametrize("ranking,key", [(0, "augserve"), (1, "fcfs")])
def test_G3_one_step_order_and_chunked_prefix(ranking, key):
    g = G["G3"]
    st = oracle.Step(cfg0(), inst0(g["B"], ranking=ranking), max_active=4)
    la = [r["l_pre"] for r in g["requests"]]
    lb = [r["segs"][0][0] for r in g["requests"]]
    ta = [r["segs"][0][1] if len(r["segs"][0]) > 1 else 0.0 for r in g["requests"]]
    fl = [1 if len(r["segs"]) > 1 else 0 for r in g["requests"]]
    assert st.enqueue(0, oracle.records(4, kind=K_NEW, id=[0, 1, 2, 3], la=la, lb=lb, ta=ta,
                                        flags=fl)) == 0
    out = st.step(0)
    assert out["rc"] == 0 and out["B"][0] == g["B"] and out["n_active"][0] == 4
    assert list(out["order"][0]) == g[key]["order"]
    grants = dict(zip(out["order"][0].tolist(), out["grant"][0].tolist()))
    assert [grants[i] for i in g[key]["order"]] == g[key]["grant"]
    if ranking == 0:
        # R1 (no call) and R3 (Preserve with 0 s) have bit-identical values:
        # equal keys, tie broken by id
        k = dict(zip(out["order"][0].tolist(), out["keys"][0].tolist()))
        assert k[1] == k[3]
        # values: the key of request 0 is the fp32 key of 115.0 etc.
        import struct
        for i, v in enumerate(g["values"]):
            u = struct.unpack("<I", struct.pack("<f", v))[0]
            assert k[i] == (u | 0x80000000)


# ---------------------------------------------------------------- G4-G8 (whole runs)
def run(B, reqs, cap=1_000_000, **kw):
    tr = tracegen.from_requests([reqs])
    return oracle.simulate_detail(cfg0(cap), inst0(B, **kw), tr)


def test_G4_single_request():
    g = G["G4"]
    rec, ft, fin = run(g["B"], [req(0, 10, [(5,)])])
    assert ft[0] * T == g["ttft_s"] * 1e6 and fin[0] * T == g["finish_s"] * 1e6
    assert rec["busy_steps"] == g["busy_steps"] and rec["completed"] == 1 and rec["slo_ok"] == 1


def test_G5_swap_round_trip():
    g = G["G5"]
    rec, ft, fin = run(g["B"], [req(0, 10, [(2, 300_000, 0.3, 5), (1,)])], cap=g["cap"])
    assert ft[0] * T == round(g["ttft_s"] * 1e6) and fin[0] * T == round(g["finish_s"] * 1e6)
    assert rec["busy_steps"] == g["busy_steps"]
    assert rec["calls_swap"] == 1 and rec["calls_preserve"] == 0 and rec["returns"] == 1
    assert rec["slo_ok"] == g["slo_ok"]
    # token conservation: 10 prefill + 2 decode + 12 swap-in + 5 assimilate + 1 decode
    assert rec["tokens_granted"] == 10 + 2 + 12 + 5 + 1
    # final ctx = 18 = l_pre + gen + ret
    assert rec["sum_gen_tokens"] == 3


def test_G5_values():
    """V1 = 2.336 (Swap, Eq.15) and V2 = 1.931 (Eq.21) for G5."""
    c = cfg0(1000)
    assert abs(oracle.stage1(c, 50, 10, 2, 0.3, oracle.SWAP) - G["G5"]["V1"]) < 1e-12
    assert oracle.select_policy(c, 50, 12, 0.3, 0) == oracle.SWAP
    assert abs(oracle.stage2(c, 50, 12, 5, 1, oracle.SWAP) - G["G5"]["V2"]) < 1e-12


def test_G6_tail_eviction():
    g = G["G6"]
    rec, ft, fin = run(g["B"], [req(0, 10, [(10,)]), req(0, 10, [(10,)])], cap=g["cap"])
    assert [f * T for f in fin] == [round(x * 1e6) for x in g["finish_s"]]
    assert rec["busy_steps"] == g["busy_steps"] and rec["slo_ok"] == g["slo_ok"]
    # t6: R1 evicted (kv 15); t7-t10: its recompute grant is cancelled each step
    assert rec["evictions"] == 5
    assert rec["err"] == 0


def test_G7_preserve_demotion():
    g = G["G7"]
    reqs = [req(0, 10, [(1, 5_000_000, 0.0, 2), (1,)]), req(300_000, 25, [(1,)])]
    rec, ft, fin = run(g["B"], reqs, cap=g["cap"])
    assert [f * T for f in fin] == [round(x * 1e6) for x in g["finish_s"]]
    arr = [0, 300_000]
    assert [ft[i] * T - arr[i] for i in range(2)] == [round(x * 1e6) for x in g["ttft_s"]]
    assert rec["busy_steps"] == g["busy_steps"] and rec["slo_ok"] == g["slo_ok"]
    assert rec["demotions"] == g["demotions"] and rec["calls_preserve"] == 1
    # R0 returns as Discard: recompute 11 + assimilate 2 = 13 tokens in one grant
    assert rec["tokens_granted"] == 10 + 1 + 25 + 1 + 13 + 1


def test_G8_serial_fcfs():
    g = G["G8"]
    rec, ft, fin = run(g["B"], [req(0, 3, [(2,)]), req(0, 3, [(2,)])], ranking=1)
    assert list(ft) == g["first_token_iter"] and list(fin) == g["finish_iter"]


# ---------------------------------------------------------------- brute force (tiny queues)
def rand_queue(rng, n, now):
    """Random IMPORT records over all tiers/stages."""
    kind = np.full(n, K_IMPORT)
    status = rng.integers(1, 4, n)                     # RUNNING/SWAPPED/WAITING
    stage2 = rng.integers(0, 2, n)
    pol = rng.integers(0, 3, n)
    flags = rng.integers(0, 2, n) | (status << 4) | (pol << 8) | (stage2 << 12)
    la = rng.integers(1, 300, n)
    lb = rng.integers(0, 50, n)
    lc = rng.integers(0, 50, n)
    ta = rng.choice([0.0, 0.5, 2.0], n).astype(np.float32)
    last = rng.integers(max(0, now - 40), now + 1, n)
    ctx = rng.integers(0, 200, n)
    kv = np.minimum(ctx, rng.integers(0, 200, n))
    cpu = np.where(status == 2, rng.integers(0, 300, n), 0)
    pend = rng.integers(0, 60, n)
    # force value ties: duplicate some feature rows
    if n >= 3:
        for a, b in ((0, 1), (1, 2)):
            if rng.random() < 0.5:
                la[b], lb[b], lc[b], ta[b], flags[b], last[b] = la[a], lb[a], lc[a], ta[a], flags[a], last[a]
    return oracle.records(n, kind=kind, id=np.arange(n), la=la, lb=lb, lc=lc, ta=ta, flags=flags,
                          last=last, ctx=ctx, kv=kv, cpu=cpu, pend=pend)


def demand(r, j, s_in=200):
    if r["cpu"][j] > 0:
        return min(int(r["cpu"][j]), s_in)
    todo = int(r["ctx"][j]) - int(r["kv"][j]) + int(r["pend"][j])
    return todo if todo > 0 else 1


@pytest.mark.parametrize("seed", range(40))
def test_bruteforce_order_and_admission(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 7))
    now = 100
    B = int(rng.integers(1, 400))
    alpha = float(rng.choice([0.0, 1.0, 50.0]))
    st = oracle.Step(cfg0(), inst0(B, alpha=alpha), max_active=n)
    r = rand_queue(rng, n, now)
    st.enqueue(0, r)
    out = st.step(now)
    assert out["rc"] == 0
    order = out["order"][0][:n].tolist()
    keys = dict(zip(order, out["keys"][0][:n].tolist()))
    tier = {j: int((r["flags"][j] >> 4) & 7) for j in range(n)}
    # the order is the lexicographic minimum over all n! permutations of (tier, key, id)
    best = min(itertools.permutations(range(n)),
               key=lambda p: [(tier[j], keys[j], j) for j in p])
    assert order == list(best)
    # admission: check every subset: the admitted set is the longest prefix whose
    # preceding demand sum stays below B (R17)
    d = [demand(r, j) for j in order]
    g = out["grant"][0][:n].tolist()
    admitted = {order[i] for i in range(n) if g[i] > 0}
    feasible = []
    for mask in range(1 << n):
        S = [i for i in range(n) if mask >> i & 1]
        if S != list(range(len(S))):
            continue                                   # must be a prefix of the order
        if all(sum(d[:i]) < B for i in S):
            feasible.append(S)
    best_prefix = max(feasible, key=len)
    assert admitted == {order[i] for i in best_prefix}
    assert sum(g) <= B
    for i in best_prefix:
        assert g[i] == min(d[i], B - sum(d[:i]))


def test_fcfs_recovered_constant_values():
    """§8(c).4: identical values and alpha = 0 give order (tier, id)."""
    n = 50
    rng = np.random.default_rng(7)
    st = oracle.Step(cfg0(), inst0(10**6), max_active=n)
    status = rng.integers(1, 4, n)
    r = oracle.records(n, kind=K_IMPORT, id=np.arange(n), la=100, lb=10, ta=1.0,
                       flags=1 | (status << 4), last=rng.integers(0, 5, n), pend=5)
    st.enqueue(0, r)
    out = st.step(10)
    assert out["order"][0].tolist() == sorted(range(n), key=lambda j: (status[j], j))


def test_spt_special_case():
    """§8(c).4: no-call requests differing only in L (or only in O) are ordered
    shortest-processing-time first; brute force over all schedules of a
    one-at-a-time server confirms that order minimizes total completion."""
    rng = np.random.default_rng(9)
    n = 6
    for vary in ("L", "O"):
        L = rng.permutation(np.arange(20, 20 + 37 * n, 37)) if vary == "L" else np.full(n, 64)
        O = rng.permutation(np.arange(3, 3 + 11 * n, 11)) if vary == "O" else np.full(n, 16)
        st = oracle.Step(cfg0(), inst0(10**6), max_active=n)
        st.enqueue(0, oracle.records(n, kind=K_NEW, id=np.arange(n), la=L, lb=O))
        order = st.step(0)["order"][0].tolist()
        svc = [L[j] / 50 + O[j] for j in range(n)]     # service time in iterations (Eq.1)

        def total_completion(p):
            t, s = 0.0, 0.0
            for j in p:
                t += svc[j]
                s += t
            return s
        best = min(total_completion(p) for p in itertools.permutations(range(n)))
        assert abs(total_completion(order) - best) < 1e-9
        assert order == sorted(range(n), key=lambda j: svc[j])


# ---------------------------------------------------------------- invariants on runs
@pytest.fixture(scope="module")
def small_traces():
    return tracegen.gen_traces(4, 120, [2.0, 4.0, 6.0, 8.0], seed=11, p_nocall=0.2)


def test_invariants_random_runs(small_traces):
    cfg = tracegen.PRESET_7B
    n_inst = 4 * 7
    tid = np.repeat(np.arange(4), 7).astype(np.uint32)
    ip = tracegen.inst_params(n_inst, ranking=[0, 1, 0, 0, 0, 0, 2] * 4,
                              budget_mode=[0, 0, 1, 0, 0, 0, 0] * 4,
                              policy_mode=[0, 0, 0, 1, 2, 3, 0] * 4, rank_seed=([0] * 6 + [99]) * 4)
    res = oracle.simulate(cfg, ip, small_traces, tid)
    for i in range(n_inst):
        d = oracle.as_dict(res[i])
        assert d["err"] == 0
        assert d["completed"] == d["n_requests"] == 120
        assert d["slo_ok"] <= d["slo_ok_5x"] <= d["completed"]
        assert d["admitted"] <= d["decisions"]
        assert d["calls_preserve"] + d["calls_swap"] + d["calls_discard"] == d["returns"]
        assert int(d["hist_ttft"].sum()) == d["completed"] == int(d["hist_norm"].sum())


def test_token_conservation_closed_form(small_traces):
    """Forced Preserve with ample memory: every granted token is a prompt,
    decoded or returned token exactly once.  Forced Discard: plus one
    recompute of the context at every call (ctx at call k = l_pre + sum of
    gen up to k + sum of returns before k)."""
    tr = small_traces
    big = dict(tracegen.PRESET_7B, g_total=10**15)
    for pm in (1, 3):
        ip = tracegen.inst_params(4, policy_mode=pm)
        res = oracle.simulate(big, ip, tr, np.arange(4, dtype=np.uint32))
        for i in range(4):
            want = 0
            for r in range(int(tr.req_off[i]), int(tr.req_off[i + 1])):
                s0, ns = int(tr.seg_off[r]), int(tr.n_seg[r])
                gen = tr.gen_true[s0:s0 + ns].astype(np.int64)
                ret = tr.ret_len[s0:s0 + ns].astype(np.int64)
                want += int(tr.l_pre[r]) + int(gen.sum()) + int(ret.sum())
                if pm == 3:
                    ctx = int(tr.l_pre[r])
                    for k in range(ns - 1):
                        ctx += int(gen[k])
                        want += ctx           # recompute at return
                        ctx += int(ret[k])
            d = oracle.as_dict(res[i])
            assert d["tokens_granted"] == want
            assert d["evictions"] == 0 and d["demotions"] == 0


def test_slo_sweep_leaves_schedule_unchanged(small_traces):
    """R30 / §8(c).4: the SLO only classifies; schedules are identical and
    slo_ok is nondecreasing in the threshold."""
    slos = [200_000, 1_000_000, 5_000_000]
    ip = tracegen.inst_params(3, slo_ttft_ticks=slos)
    res = oracle.simulate(tracegen.PRESET_7B, ip, small_traces, np.zeros(3, np.uint32))
    ds = [oracle.as_dict(r) for r in res]
    for k in oracle.FIELDS:
        if k not in ("slo_ok", "slo_ok_5x"):
            assert ds[0][k] == ds[1][k] == ds[2][k], k
    assert ds[0]["slo_ok"] <= ds[1]["slo_ok"] <= ds[2]["slo_ok"]


def test_max_iters_prefix(small_traces):
    """Stopping at max_iters and the full run agree on everything finished
    before the cut (the loop state at the top of an iteration is a function
    of the inputs only)."""
    full = oracle.as_dict(oracle.simulate(tracegen.PRESET_7B, tracegen.inst_params(1), small_traces,
                                          [1])[0])
    cut = oracle.as_dict(oracle.simulate(tracegen.PRESET_7B, tracegen.inst_params(1), small_traces,
                                         [1], max_iters=full["final_t"] // 2)[0])
    assert cut["final_t"] >= full["final_t"] // 2
    assert cut["completed"] <= full["completed"]
    assert cut["busy_steps"] < full["busy_steps"]


def test_ablation_directions():
    """Directional reproduction of the paper's comparative findings inside the
    simulator (SPEC acceptance 4 and 8): on an
    overloaded 7B-preset workload (4 traces x 500 requests at 4 req/s)
      - random scheduling beats FCFS,
      - AugServe's goodput is >= 1.5x FCFS and its mean TTFT <= 0.5x FCFS,
      - the dynamic token limit helps FCFS and AugServe (ablation),
      - the two-stage ordering adds on top of dynamic batching."""
    tr = tracegen.gen_traces(4, 500, [4.0] * 4, seed=21)
    tid = np.arange(4, dtype=np.uint32)
    modes = {"augserve": dict(ranking=0, budget_mode=0), "aug_static": dict(ranking=0, budget_mode=1),
             "fcfs_static": dict(ranking=1, budget_mode=1), "fcfs_dyn": dict(ranking=1, budget_mode=0),
             "random_static": dict(ranking=2, budget_mode=1, rank_seed=5)}
    good, ttft = {}, {}
    for name, m in modes.items():
        ip = tracegen.inst_params(4, l_static=500, **m)
        d = [oracle.as_dict(x) for x in oracle.simulate(tracegen.PRESET_7B, ip, tr, tid, threads=4)]
        good[name] = sum(x["slo_ok"] for x in d)
        ttft[name] = sum(x["sum_ttft_ticks"] for x in d) / sum(x["completed"] for x in d)
    assert good["random_static"] > good["fcfs_static"]
    assert good["augserve"] >= 1.5 * good["fcfs_static"]
    assert ttft["augserve"] <= 0.5 * ttft["fcfs_static"]
    assert good["fcfs_dyn"] > good["fcfs_static"]
    assert good["augserve"] > good["aug_static"]
    assert good["augserve"] > good["fcfs_dyn"]


def test_cv_robustness_direction():
    """SPEC acceptance 7 / tab:cv: on W3 arrivals (Gamma, 30-minute
    horizon) at 2 req/s, raising the coefficient of variation from 1 to 2
    costs FCFS a larger relative share of its goodput than AugServe, and
    AugServe's goodput stays far above FCFS's."""
    from tracegen import tablegen as tg
    H = 1800 * 10**6
    good = {}
    for cv in (1.0, 2.0):
        tr = tg.generate(tg.build_tables(cv=cv), 31, 2, 20000, [2.0, 2.0], horizon_ticks=H)
        tid = np.arange(2, dtype=np.uint32)
        for mode, kw in (("fcfs", dict(ranking=1, budget_mode=1, l_static=500)),
                         ("aug", dict(ranking=0, budget_mode=0))):
            ip = tracegen.inst_params(2, **kw)
            d = [oracle.as_dict(x) for x in oracle.simulate(tracegen.PRESET_7B, ip, tr, tid, threads=2)]
            good[(cv, mode)] = sum(x["slo_ok"] for x in d)
    loss = {m: 1 - good[(2.0, m)] / good[(1.0, m)] for m in ("fcfs", "aug")}
    assert loss["fcfs"] > loss["aug"]
    assert good[(2.0, "aug")] > 5 * good[(2.0, "fcfs")]
