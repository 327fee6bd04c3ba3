#!/usr/bin/env python
"""Mutation check of the oracle's pins.

Each mutant is one plausible slip in oracle/augsched_oracle.cpp (a dropped
term, a flipped comparison, a wrong operand).  The script builds every mutant
into a temporary library and runs the CPU pin tests against it
(AUGSCHED_ORACLE_LIB); a mutant "survives" if all of them still pass.
Exit status 1 if any mutant survives.

    python tools/oracle_mutants.py [--only NAME ...]
"""
from __future__ import annotations

import argparse
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "augsched_oracle.cpp")
TESTS = ["tests/test_oracle_formulas.py", "tests/test_oracle_schedules.py", "tests/test_oracle_pins_r2.py",
         "tests/test_oracle_ti.py"]

# name -> (passage, [(old, new), ...]); every `old` must occur exactly once
MUTANTS = {
    "issue_cother_sim": ("R13/Eq.5 C_other at issuance (simulate)",
                         [("(uint64_t)(A_snap - kv_snap)", "(uint64_t)A_snap")]),
    "issue_cother_step": ("R13/Eq.5 C_other at issuance (step)",
                          [("(uint64_t)(A_evt - s.kv)", "(uint64_t)A_evt")]),
    "demote_kv_asc_step": ("R20 demotion kv desc (step)",
                           [("if (I.s[a].kv != I.s[b].kv) return I.s[a].kv > I.s[b].kv;",
                             "if (I.s[a].kv != I.s[b].kv) return I.s[a].kv < I.s[b].kv;")]),
    "demote_id_desc_step": ("R20 demotion id asc on kv ties (step)",
                            [("      return a < b;\n    });\n    for (uint32_t id : pres) {\n      if (need <= free_) break;\n      SSlot&",
                              "      return a > b;\n    });\n    for (uint32_t id : pres) {\n      if (need <= free_) break;\n      SSlot&")]),
    "demote_kv_asc_sim": ("R20 demotion kv desc (simulate)",
                          [("if (R[a].kv != R[b].kv) return R[a].kv > R[b].kv;",
                            "if (R[a].kv != R[b].kv) return R[a].kv < R[b].kv;")]),
    "evict_keeps_cpu_step": ("B2 eviction drops the CPU copy (step)",
                             [("g[j] = 0; s.kv = 0; s.cpu = 0; s.status = WAITING;",
                               "g[j] = 0; s.kv = 0; s.status = WAITING;")]),
    "evict_keeps_cpu_sim": ("B2 eviction drops the CPU copy (simulate)",
                            [("g[j] = 0; r.kv = 0; r.cpu = 0; r.status = WAITING;",
                              "g[j] = 0; r.kv = 0; r.status = WAITING;")]),
    "slo5x_ttft_1x": ("P:1320 5x SLO (TTFT term)",
                      [("ttft < 5 * ip.slo_ttft_ticks", "ttft < ip.slo_ttft_ticks")]),
    "slo5x_norm_1x": ("P:1320 5x SLO (normalized-latency term)",
                      [("< 5 * (uint64_t)ip.slo_norm_num", "< (uint64_t)ip.slo_norm_num")]),
    "admitted_counts_grants": ("admitted = prefix length (P:1225-1229)",
                               [("    ++n_prefix;\n", ""),
                                ("  // S9 + token accounting of the granted batch\n",
                                 "  for (int64_t x : g) n_prefix += x > 0;\n  // S9 + token accounting of the granted batch\n")]),
    "return_before_snapshot": ("S1 snapshot before returns (R23): A_snap after Preserve returns",
                               [("    const int64_t A_snap = A;\n", "    int64_t A_snap = A;\n"),
                                ("    // S3 arrivals (Algorithm 1 lines 2-9; Eq.4-15)\n",
                                 "    A_snap = A;\n    // S3 arrivals (Algorithm 1 lines 2-9; Eq.4-15)\n")]),
    "swap_cost_no_N": ("Eq.6 keeps the N^fwd_max multiplier (R6)",
                       [("return ((2.0 * (((double)C / k.Sout) * k.Ts)) * k.N) * k.M;",
                         "return (2.0 * (((double)C / k.Sout) * k.Ts)) * k.M;")]),
    "budget_gamma_dropped": ("Eq.31 gamma*P term",
                             [("std::max<int64_t>(free_, 0) +\n                (int64_t)(((uint64_t)c.gamma_num * (uint64_t)P) / c.gamma_den);",
                               "std::max<int64_t>(free_, 0);")]),
    "last_not_set_on_grant": ("R14 last = t on a grant > 0 (simulate)",
                              [("      r.last = t;\n      r.status = RUNNING;\n", "      r.status = RUNNING;\n")]),
    "ti_key_sign": ("B12 time-invariant key V + alpha*last*T",
                    [("double s = V + (alpha * ((double)last * Ts));", "double s = V - (alpha * ((double)last * Ts));")]),
    "tie_by_id_desc": ("R2 ties by id ascending (simulate order)",
                       [("    std::sort(ord.begin(), ord.end(), [](const Ent& a, const Ent& b) {\n      return std::tie(a.tier, a.key, a.id) < std::tie(b.tier, b.key, b.id);\n    });\n    // S7 admission: a prefix",
                         "    std::sort(ord.begin(), ord.end(), [](const Ent& a, const Ent& b) {\n      return std::tie(a.tier, a.key, b.id) < std::tie(b.tier, b.key, a.id);\n    });\n    // S7 admission: a prefix")]),
}


def build_mutant(src: str, edits, out: str):
    for old, new in edits:
        c = src.count(old)
        if c != 1:
            raise SystemExit(f"pattern occurs {c} times: {old!r}")
        src = src.replace(old, new)
    cpp = out[:-3] + ".cpp"
    open(cpp, "w").write(src)
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                           "-shared", "-pthread", "-o", out, cpp])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*")
    args = ap.parse_args()
    src = open(SRC).read()
    survivors = []
    with tempfile.TemporaryDirectory() as td:
        for name, (cite, edits) in MUTANTS.items():
            if args.only and name not in args.only:
                continue
            lib = os.path.join(td, f"m_{name}.so")
            build_mutant(src, edits, lib)
            env = dict(os.environ, AUGSCHED_ORACLE_LIB=lib)
            r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "not gpu", "-p", "no:randomly",
                                *TESTS], cwd=ROOT, env=env, capture_output=True, text=True)
            killed = r.returncode != 0
            first = ""
            for line in r.stdout.splitlines():
                if line.startswith("FAILED") or line.startswith("ERROR"):
                    first = line
                    break
            print(f"{'killed ' if killed else 'SURVIVED'} {name:26s} ({cite}) {first}", flush=True)
            if not killed:
                survivors.append(name)
    print(f"{len(survivors)} survivor(s)" + (": " + ", ".join(survivors) if survivors else ""))
    sys.exit(1 if survivors else 0)


if __name__ == "__main__":
    main()
