"""Generate tests/golden/tape_ref.json: the reference tape's memory-plan
hand-off counts (Graph::planned_reuse_count, dl/tape.hpp:486-491) for its own
model graphs, on the committed golden inputs (ref_vectors.npz gp cases,
kalman_ref.npz cases), through oracle/_ref (TEST INFRASTRUCTURE).

    python tests/golden/make_golden_tape.py
"""
import ctypes as C
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402


def main():
    O.build(ref=True)
    lib = O.ref().lib
    lib.ref_gp_plan_count.restype = C.c_int64
    lib.ref_kalman_plan_count.restype = C.c_int64
    P = lambda a: np.ascontiguousarray(a).ctypes.data_as(C.c_void_p)  # noqa: E731
    out = {}
    g = np.load(os.path.join(HERE, "ref_vectors.npz"))
    for key in ("gp:96", "gp:300"):
        x, y = np.ascontiguousarray(g[key + "/x"]), np.ascontiguousarray(g[key + "/y"])
        out[key] = int(lib.ref_gp_plan_count(C.c_int64(x.shape[0]), C.c_int64(x.shape[1]), P(x), P(y)))
    k = np.load(os.path.join(HERE, "kalman_ref.npz"))
    for name in ("h2d2T5", "h4d3T20", "h3d5T10"):
        m = [np.ascontiguousarray(k[f"{name}/in/{n}"]) for n in ("a", "b", "sh", "sv", "mu0", "s0", "obs")]
        h, d, T = m[0].shape[0], m[1].shape[0], m[6].shape[0]
        out["kalman:" + name] = int(lib.ref_kalman_plan_count(C.c_int64(h), C.c_int64(d), C.c_int64(T),
                                                               *[P(a) for a in m]))
    json.dump(out, open(os.path.join(HERE, "tape_ref.json"), "w"), indent=1)
    print(out)


if __name__ == "__main__":
    main()
