"""Writes tests/golden/*.json by calling ONLY oracle/ (tier T1, the dense definition).

Run: python tests/golden/make_golden.py
c1_double_integrator.json: BASELINE configs[0] (double integrator; terminal equality
condensed as eta e1 e1^T; delta = 1/eta), solved by assembling the §1.4
KKT system densely and calling LAPACK.  It also records u_0 of the delta = 0
(classic LQR) solve, the eta -> inf limit.
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402
import synth  # noqa: E402


def main():
    p = synth.double_integrator_c1()
    d = oracle.rr_solve_dense(p)
    d0 = oracle.rr_solve_dense(p.with_delta(0.0))
    out = {
        "source": "oracle T1 (dense LAPACK solve of the §1.4 system), tests/golden/make_golden.py",
        "config": "C1: double integrator h=0.1 N=10, Q=I, R=0.1, Q_N=10I + 1e4 e1e1^T, c0=(5,0), delta=1e-4",
        "x": d["x"].tolist(), "u": d["u"].tolist(), "y": d["y"].tolist(),
        "u0_delta0": float(d0["u"][0, 0]),
    }
    with open(os.path.join(HERE, "c1_double_integrator.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
