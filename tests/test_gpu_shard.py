"""The sharded single huge queue against the oracle: one
global queue split over G shards (single-instance handles on this GPU, the
collectives done by the test: a sum of the ledgers and a concatenation of
the offers, as all-reduce / all-gather would), random NEW / CALL / RETURN /
FINISH events over many steps.  Every step's global prefix (order, keys,
grants), limit, queue size and admitted count, and every shard's slot state
and ledger, must equal the oracle's full-order step over the whole queue
(global slot id = shard * max_active + local slot).  Small capacities force
the cross-shard R20 resolution (demotion and tail eviction over the
gathered KV holders)."""
import numpy as np
import pytest

import oracle
import tracegen

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2512_04013_b200 as aug  # noqa: E402
from test_gpu_step import random_events  # noqa: E402


def split_records(rec, G, MA):
    """Global records -> per-shard records with local slot ids."""
    ids = rec["id"].astype(np.int64)
    out = []
    for r in range(G):
        m = (ids // MA) == r
        if not m.any():
            out.append(None)
            continue
        sub = {k: np.ascontiguousarray(v[m]) for k, v in rec.items()}
        sub["id"] = (ids[m] - r * MA).astype(np.uint32)
        out.append(sub)
    return out


def run_sharded(G, MA, cap, ranking, steps, seed, p_new0=0.6, p_new=0.08):
    rng = np.random.default_rng(seed)
    cfg = dict(tracegen.PRESET_G0, g_total=1000 + cap, g_model=1000)
    ip = tracegen.inst_params(1, base=tracegen.INST_G0, ranking=ranking, budget_mode=0, target_max=200,
                              alpha=1.5, rank_seed=seed)
    st = oracle.Step(cfg, ip, G * MA)
    hs = [aug.Scheduler(cfg, ip, 1, MA) for _ in range(G)]
    ob = hs[0].shard_offer_bytes()
    ledgers = [torch.zeros(2, dtype=torch.int64, device="cuda") for _ in range(G)]
    offers = [torch.zeros(ob, dtype=torch.uint8, device="cuda") for _ in range(G)]
    for t in range(steps):
        rec = random_events(rng, st.slots(0), t, p_new=p_new0 if t == 0 else p_new)
        if rec is not None:
            assert st.enqueue(0, rec) == 0
            for r, sub in enumerate(split_records(rec, G, MA)):
                if sub is not None:
                    hs[r].enqueue(0, sub)
        o = st.step(t)
        assert o["rc"] == 0
        for r in range(G):
            hs[r].shard_begin(t, ledgers[r])
        lsum = torch.stack(ledgers).sum(0)
        for r in range(G):
            hs[r].shard_offer(lsum, offers[r])
        allo = torch.cat(offers)
        outs = [hs[r].shard_commit(allo, G, r) for r in range(G)]
        res = [hs[r].shard_result(outs[r]) for r in range(G)]
        label = f"G={G} ranking={ranking} cap={cap} step {t}"
        a = int(o["admitted"][0])
        for r in range(G):
            g = res[r]
            assert g["B"] == int(o["B"][0]), label
            assert g["n_active"] == int(o["n_active"][0]), label
            assert g["admitted"] == a, f"{label}: admitted {g['admitted']} vs {a}"
            assert g["order"].tolist() == o["order"][0][:a].tolist(), label
            assert g["keys"].tolist() == o["keys"][0][:a].tolist(), label
            assert g["grant"].tolist() == o["grant"][0][:a].tolist(), label
        if t % 4 == 3 or t == steps - 1:
            osl = st.slots(0)
            for r in range(G):
                gsl, osr = hs[r].slots(0), osl[r * MA:(r + 1) * MA]
                bad = np.nonzero((gsl != osr).any(1))[0]
                assert len(bad) == 0, f"{label}: shard {r} slots {bad[:5]} gpu {gsl[bad[:3]].tolist()} " \
                    f"oracle {osr[bad[:3]].tolist()}"
            A, P = st.ledger(0)
            assert sum(h.ledger(0)[0] for h in hs) == A and sum(h.ledger(0)[1] for h in hs) == P, label
    for h in hs:
        h.sync()
        h.close()


@pytest.mark.parametrize("G,cap,ranking", [(2, 10**6, 0), (3, 10**6, 0), (2, 700, 0), (3, 450, 0),
                                           (2, 600, 3), (4, 10**6, 1)])
def test_sharded_queue_equals_single_queue(G, cap, ranking):
    run_sharded(G, 400, cap, ranking, steps=24, seed=G * 100 + cap % 97 + ranking)


def test_sharded_cfg4_million():
    """cfg4's 1M-request queue split over 4 shards of 250,000 slots: six
    steps equal the oracle's single-queue steps."""
    n, G = 1_000_000, 4
    MA = n // G
    rec = tracegen.cfg4_records(n)
    cfg, ip = tracegen.PRESET_CFG4, tracegen.inst_params(1)
    st = oracle.Step(cfg, ip, n)
    assert st.enqueue(0, rec) == 0
    hs = [aug.Scheduler(cfg, ip, 1, MA) for _ in range(G)]
    for r, sub in enumerate(split_records(rec, G, MA)):
        hs[r].enqueue(0, sub)
    ob = hs[0].shard_offer_bytes()
    ledgers = [torch.zeros(2, dtype=torch.int64, device="cuda") for _ in range(G)]
    offers = [torch.zeros(ob, dtype=torch.uint8, device="cuda") for _ in range(G)]
    t0 = 65536
    for k in range(6):
        o = st.step(t0 + k)
        for r in range(G):
            hs[r].shard_begin(t0 + k, ledgers[r])
        lsum = torch.stack(ledgers).sum(0)
        for r in range(G):
            hs[r].shard_offer(lsum, offers[r])
        allo = torch.cat(offers)
        g = hs[0].shard_result(hs[0].shard_commit(allo, G, 0))
        for r in range(1, G):
            hs[r].shard_commit(allo, G, r)
        a = int(o["admitted"][0])
        assert g["admitted"] == a and g["B"] == int(o["B"][0]) and g["n_active"] == int(o["n_active"][0])
        assert g["order"].tolist() == o["order"][0][:a].tolist()
        assert g["grant"].tolist() == o["grant"][0][:a].tolist()
    osl = st.slots(0)
    for r in range(G):
        assert np.array_equal(hs[r].slots(0), osl[r * MA:(r + 1) * MA])
        hs[r].close()


def test_sharded_edge_cases():
    """Degenerate shards: one shard holds no request at all (its slots are
    never used), a static limit of 0 for a few steps (nothing admitted), one
    shard alone (G = 1)."""
    for G, MA, used in ((3, 200, [0, 2]), (1, 300, [0])):
        rng = np.random.default_rng(G)
        cfg = dict(tracegen.PRESET_G0, g_total=1000 + 500, g_model=1000)
        for lim in (0, 150):
            ip = tracegen.inst_params(1, base=tracegen.INST_G0, budget_mode=1, l_static=lim, target_max=100)
            st = oracle.Step(cfg, ip, G * MA)
            hs = [aug.Scheduler(cfg, ip, 1, MA) for _ in range(G)]
            ob = hs[0].shard_offer_bytes()
            led = [torch.zeros(2, dtype=torch.int64, device="cuda") for _ in range(G)]
            off = [torch.zeros(ob, dtype=torch.uint8, device="cuda") for _ in range(G)]
            for t in range(8):
                slots = st.slots(0)
                rec = random_events(rng, slots, t, p_new=0.5 if t == 0 else 0.1)
                if rec is not None:
                    keep = np.isin(rec["id"].astype(np.int64) // MA, used)
                    rec = {k: np.ascontiguousarray(v[keep]) for k, v in rec.items()}
                if rec is not None and len(rec["id"]):
                    assert st.enqueue(0, rec) == 0
                    for r, sub in enumerate(split_records(rec, G, MA)):
                        if sub is not None:
                            hs[r].enqueue(0, sub)
                o = st.step(t)
                for r in range(G):
                    hs[r].shard_begin(t, led[r])
                ls = torch.stack(led).sum(0)
                for r in range(G):
                    hs[r].shard_offer(ls, off[r])
                allo = torch.cat(off)
                outs = [hs[r].shard_commit(allo, G, r) for r in range(G)]
                g = hs[0].shard_result(outs[0])
                a = int(o["admitted"][0])
                assert g["admitted"] == a and g["B"] == int(o["B"][0]) and g["n_active"] == int(o["n_active"][0])
                assert g["order"].tolist() == o["order"][0][:a].tolist()
                assert g["grant"].tolist() == o["grant"][0][:a].tolist()
            for h in hs:
                h.sync()
                h.close()
