#!/usr/bin/env python
"""Mutation probe of the oracle pins (-m "not gpu" CPU tests).

Copies the repo to a scratch directory, applies one plausible mistake to oracle/ at a time,
runs the oracle pin suites there and reports whether at least one pin fails ("killed").
A mutation that survives means part of the oracle is unpinned.

    python tools/mutation_probe.py            # all mutations
    python tools/mutation_probe.py band sum   # a subset by name
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITES = ["tests/test_oracle_pins.py", "tests/test_oracle_band_pins.py", "tests/test_planning_pins.py"]

# name -> (file, old, new)
MUTATIONS = {
    "band_1e-2": ("oracle/rtg_oracle.c", "#define ORC_BAND 1e-6", "#define ORC_BAND 1e-2"),
    "no_collide_bit": ("oracle/rtg_oracle.c", "if (do_collision && !(f & 1u))", "if (do_collision && !(f & 2u))"),
    "pair_mask_ignores_flag": ("oracle/rtg_oracle.c", "            if (flags && (flags[g] & 1u)) continue;\n", ""),
    "sum_is_xi": ("oracle/oracle.py", "util, u_lo, u_hi = g.copy(), g_lo.copy(), g_hi.copy()",
                  "util, u_lo, u_hi = xi.copy(), xi_lo.copy(), xi_hi.copy()"),
    "vis_band_ignores_definite_out": ("oracle/rtg_oracle.c", "*amb = (!definitely_out) && near;", "*amb = near;"),
    "col_amb_keeps_definite": ("oracle/rtg_oracle.c", "(unsigned char)(!c_def && c_amb)", "(unsigned char)(c_amb)"),
    "allowed_drops_band": ("oracle/oracle.py", "            if col_amb[k, t]:\n                allowed[k, t] = True",
                           "            if False:\n                allowed[k, t] = True"),
    "acceptable_no_tol": ("oracle/oracle.py", "util_hi >= m - tol * abs(m)", "util_hi >= m"),
    "gain_hi_drops_band": ("oracle/rtg_oracle.c", "if (definite || ab) {", "if (definite) {"),
    "strict_far_plane": ("oracle/rtg_oracle.c", "if (!(sg[j] >= 0.0)) nominal = 0;", "if (!(sg[j] > 0.0)) nominal = 0;"),
    # control: a dropped term in the inflated semi-axis (must be killed by the original pins)
    "control_semi_axis": ("oracle/rtg_oracle.c", "double a_i = lambda_g * s[i] + r_robot;",
                          "double a_i = lambda_g * s[i] + 0.9 * r_robot;"),
}


def run(name: str) -> bool:
    f, old, new = MUTATIONS[name]
    tmp = tempfile.mkdtemp(prefix=f"mut_{name}_")
    try:
        shutil.copytree(ROOT, os.path.join(tmp, "r"), ignore=shutil.ignore_patterns(
            ".git", "gpurun_out", "profiles", "build", "_build", "*.so", "__pycache__"), symlinks=True)
        r = os.path.join(tmp, "r")
        # the product library is not needed by the oracle suites, but its module must import
        so = os.path.join(ROOT, "paper_2409_18122_b200", "librtg.so")
        if os.path.exists(so):
            shutil.copy(so, os.path.join(r, "paper_2409_18122_b200", "librtg.so"))
        path = os.path.join(r, f)
        src = open(path).read()
        assert src.count(old) >= 1, f"{name}: pattern not found in {f}"
        open(path, "w").write(src.replace(old, new))
        p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "not gpu", "-p", "no:cacheprovider",
                            *SUITES], cwd=r, capture_output=True, text=True)
        killed = p.returncode != 0
        tail = [ln for ln in p.stdout.splitlines() if ln.startswith("FAILED")][:1]
        print(f"{name:32s} {'killed' if killed else 'SURVIVED'}  {tail[0] if tail else ''}", flush=True)
        return killed
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


def main(argv):
    names = argv or list(MUTATIONS)
    res = {n: run(n) for n in names}
    surv = [n for n, k in res.items() if not k]
    print(f"{len(res) - len(surv)}/{len(res)} killed" + (f"; survived: {surv}" if surv else ""))
    return 1 if surv else 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
