"""Writes tests/golden/eq41_closed_forms.json: closed-form values of Eq. 4.1/4.2.

Source: PAPER.md P:2720-2741 (eq:force  F_N = k*delta - gamma*sqrt(r*delta);
eq:force-radius r = r1*r2/(r1+r2); k = 2, gamma = 1 "as in Cortex3D").
delta = r1 + r2 - |c1 - c2| (reading R2); the force on sphere 1 points along
(c1 - c2) and is positive when repulsive (reading R1).

Values are evaluated here with 50-digit decimal arithmetic -- pure mathematics at a
fixed point, independent of both the oracle and the CUDA path.  Nothing is imported
from oracle/ or from the product package.
"""
import json
import os
from decimal import Decimal as D, getcontext

getcontext().prec = 50
K, GAMMA = D(2), D(1)


def eq41(r1, r2, c1, c2):
    r1, r2 = D(r1), D(r2)
    diff = [D(a) - D(b) for a, b in zip(c1, c2)]
    dist = sum(v * v for v in diff).sqrt()
    delta = r1 + r2 - dist
    rbar = r1 * r2 / (r1 + r2)
    Fn = K * delta - GAMMA * (rbar * delta).sqrt()
    force1 = [Fn * v / dist for v in diff]
    return Fn, force1


CASES = [
    # name, r1, r2, c1, c2, note
    ("equal_radii_delta1", 5, 5, (0, 0, 0), (9, 0, 0), "delta=1, rbar=2.5: F_N = 2 - sqrt(2.5)"),
    ("unequal_radii", 4, 6, (0, 0, 0), (9, 0, 0), "delta=1, rbar=2.4: F_N = 2 - sqrt(2.4)"),
    ("exact_zero", 5, 5, (0, 0, 0), ("9.375", 0, 0),
     "delta=5/8, rbar*delta=25/16: F_N = 5/4 - 5/4 = 0 exactly (k*delta = gamma*sqrt(rbar*delta))"),
    ("max_attraction", 5, 5, (0, 0, 0), ("9.84375", 0, 0),
     "delta=5/32 = gamma^2 rbar/(4k^2): F_N = 5/16 - 5/8 = -5/16 exactly; force on sphere 1 is +5/16 (towards sphere 2)"),
    ("off_axis", 5, 5, (0, 0, 0), (3, 4, 6), "D=61: F_N = 2(10-sqrt61) - sqrt(2.5(10-sqrt61)) along -(3,4,6)/sqrt61"),
    ("cap_case", 200, 200, (0, 0, 0), (1, 0, 0),
     "delta=399, rbar=100: F_N = 798 - sqrt(39900); dt*F_N = 5.98 > 3 so the displacement is capped to 3"),
]

out = {"source": "PAPER.md P:2720-2741 eq:force / eq:force-radius, k=2 gamma=1", "cases": []}
for name, r1, r2, c1, c2, note in CASES:
    Fn, f1 = eq41(r1, r2, c1, c2)
    out["cases"].append({
        "name": name, "r1": r1, "r2": r2, "c1": [str(v) for v in c1], "c2": [str(v) for v in c2],
        "F_N": str(+Fn), "force_on_1": [str(+v) for v in f1], "note": note,
    })

# superposition: three collinear spheres r=5 at x=0, 9, 17.5; force on the middle one
Fl = eq41(5, 5, (9, 0, 0), (0, 0, 0))[1][0]
Fr = eq41(5, 5, (9, 0, 0), ("17.5", 0, 0))[1][0]
out["collinear_middle"] = {
    "x": ["0", "9", "17.5"], "r": 5, "left_term": str(+Fl), "right_term": str(+Fr),
    "sum": str(+(Fl + Fr)),
    "note": "sqrt(3.75) - sqrt(2.5) - 1; with x = 0, 9, 18 the two terms cancel (net 0, nnz = 2)",
}
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "eq41_closed_forms.json")
with open(path, "w") as f:
    json.dump(out, f, indent=1)
print(path)
