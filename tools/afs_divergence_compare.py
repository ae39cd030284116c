"""CPU side of tools/afs_divergence_dump.py: compares the product's and the
oracle's relocation trajectories at the cfg4 AFS iteration where the sampled
sequences part, and adds an independent numpy/LAPACK restatement of
relocate_poles (tests/test_oracle_crosscheck.py: np_relocate) as the third
opinion. Prints one JSON object.

Usage: python tools/afs_divergence_compare.py gpurun_out/cfg4_afs_dump.npz"""
import json
import sys

import numpy as np

sys.path[:0] = [".", "oracle", "tests"]
import pyoracle as O  # noqa: E402
from test_oracle_crosscheck import np_relocate  # noqa: E402


def dist(a, b):
    """max over b of the relative distance to the nearest pole of a"""
    return float(max(min(abs(x - y) / abs(y) for x in a) for y in b))


d = np.load(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/cfg4_afs_dump.npz")
J, orf = int(d["J"]), d["orf"]
sj, vj = d["samples"][:J], d["values"][:J][:, orf]
out = {"J": J, "orf": orf.tolist()}
for tag in ("high", "low"):
    po, pp, one = d[f"{tag}_oracle"], d[f"{tag}_product"], d[f"{tag}_product_one_step"]
    pn = [po[0]]
    none = []
    for i in range(3):
        pn.append(O.canonical_poles(np_relocate(sj, vj, O.canonical_poles(pn[-1]))[0]))
        none.append(O.canonical_poles(np_relocate(sj, vj, O.canonical_poles(po[i]))[0]))
    rows = []
    for i in range(1, 4):
        rows.append(dict(step=i, product_vs_oracle=dist(pp[i], po[i]), numpy_vs_oracle=dist(pn[i], po[i]),
                         product_vs_numpy=dist(pp[i], pn[i]),
                         one_step_product_vs_oracle=dist(one[i - 1], po[i]),
                         one_step_numpy_vs_oracle=dist(none[i - 1], po[i])))
    # the pole that differs most at the end, and how far it sits from the band
    fin_o, fin_p = po[3], pp[3]
    errs = [min(abs(x - y) / abs(y) for x in fin_p) for y in fin_o]
    w = int(np.argmax(errs))
    out[tag] = dict(order=int(len(po[0])), steps=rows, worst_pole=[fin_o[w].real, fin_o[w].imag],
                    worst_rel=float(errs[w]), band=float(max(abs(sj.imag))),
                    poles_within_1e6=int(sum(e < 1e-6 for e in errs)))
print(json.dumps(out, indent=1))
