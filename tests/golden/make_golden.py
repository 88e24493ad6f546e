"""Regenerate the golden fixtures from the UNMODIFIED reference library.

Run in the build container (needs oracle/_ref/libcsr5ref.so, which is built from
/root/reference/proj/core/src by oracle/Makefile):

    python tests/golden/make_golden.py            # everything
    python tests/golden/make_golden.py --dumps    # ref_dumps.json.gz only

Writes tests/golden/ref_w32.npz (reference csr_to_csr5 arrays and deterministic
spmv_csr5 y at omega=32 over a sigma sweep) and tests/golden/ref_edges.json
(the edge-case metadata dumps listed in SURVEY.md section 8c), and
tests/golden/ref_dumps.json.gz (the reference's dump_format text of every
ref_w32 case, format.cpp:267-305).  Inputs are
stored alongside the outputs so the fixtures do not depend on any generator.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
from oracle.oracle import Csr, Oracle, Ref  # noqa: E402

SIGMAS = [1, 2, 3, 4, 5, 8, 12, 16, 17, 18, 24, 27, 32, 40, 48]


def corpus(o: Oracle):
    """Shapes from the reference acceptance corpus (acceptance.cpp:53-104),
    sized so one tile row of ω=32 tiles is exercised with tails and empties."""
    g = o.rng(2024)
    mats = []
    mats.append(("all_empty", o.coo_to_csr([], [], [], 37, 11)))
    mats.append(("regular", o.generate_synthetic(0, 150, 150, 1200, 3)))
    mats.append(("singletons", o.generate_synthetic(0, 200, 200, 200, 4)))
    mats.append(("one_long_row", o.generate_synthetic(1, 120, 1500, 2000, 5, 0.3)))
    mats.append(("skew", o.generate_synthetic(2, 300, 120, 2500, 6)))
    mats.append(("skew_sparse", o.generate_synthetic(2, 900, 60, 700, 7)))
    mats.append(("tiny", o.generate_synthetic(2, 3, 50, 17, 8)))
    mats.append(("exact_multiple", o.generate_synthetic(0, 96, 96, 1536, 9)))
    for k in range(4):
        m = 1 + g() % 200
        n = 1 + g() % 200
        mats.append((f"random{k}", g.random_csr(m, n, g() % 3000)))
    # leading / trailing empty rows and a long run of empties inside
    rows = [5] * 40 + [6] * 3 + [400] * 70 + [401] * 2
    cols = list(range(40)) + [0, 1, 2] + list(range(70)) + [3, 4]
    mats.append(("empty_runs", o.coo_to_csr(rows, cols, [1.0 + 0.5 * i for i in range(len(rows))], 450, 80)))
    return mats


def main():
    o, r = Oracle(), Ref()
    out = {}
    meta = []
    k = 0
    for mi, (name, a) in enumerate(corpus(o)):
        x = o.rng(1000 + mi).random_x(a.n)
        out[f"m{mi}_row_ptr"] = a.row_ptr
        out[f"m{mi}_col_idx"] = a.col_idx.astype(np.int32)
        out[f"m{mi}_val"] = a.val
        out[f"m{mi}_x"] = x
        for sigma in SIGMAS:
            A = r.build(a, 32, sigma)
            y = r.spmv(a, x, 32, sigma, 0)
            key = f"c{k}"
            out[f"{key}_tile_ptr"] = A.tile_ptr
            out[f"{key}_tile_desc"] = A.tile_desc
            out[f"{key}_eo_ptr"] = A.eo_ptr
            out[f"{key}_eo"] = A.eo
            out[f"{key}_tcol"] = A.col_idx.astype(np.int32)
            out[f"{key}_y"] = y
            meta.append(dict(key=key, mat=f"m{mi}", name=name, m=a.m, n=a.n, nnz=a.nnz, omega=32, sigma=sigma,
                             p=A.p, pc=A.pc, tail=A.tail_len, word_bits=A.word_bits))
            k += 1
    np.savez_compressed(os.path.join(HERE, "ref_w32.npz"), meta=json.dumps(meta), **out)

    # SURVEY.md 8c edge dumps, recomputed from the reference.
    edges = []
    def dump(name, row_ptr, omega, sigma, n=None):
        row_ptr = np.array(row_ptr, dtype=np.int64)
        m = len(row_ptr) - 1
        nnz = int(row_ptr[-1])
        n = n or max(nnz, 1)
        cols = []
        for i in range(m):
            cols += list(range(int(row_ptr[i + 1] - row_ptr[i])))
        a = Csr(m, n, row_ptr, np.array(cols, dtype=np.int64), np.arange(1, nnz + 1, dtype=np.float64))
        A = r.build(a, omega, sigma)
        edges.append(dict(name=name, row_ptr=row_ptr.tolist(), omega=omega, sigma=sigma,
                          tile_ptr=[int(v) for v in A.tile_ptr], tile_desc=[int(v) for v in A.tile_desc],
                          eo_ptr=A.eo_ptr.tolist(), eo=A.eo.tolist(), p=A.p, pc=A.pc, tail=A.tail_len))
    dump("leading_empty", [0, 0, 0, 3, 4, 4, 8, 10, 10], 2, 2)
    dump("nnz0_m3", [0, 0, 0, 0], 2, 2)
    dump("exact_multiple_trailing_empty", [0, 2, 4, 4, 4], 2, 2)
    dump("spurious_flag", [0, 4, 8, 8, 12], 2, 2)
    cols8 = [[0, 1, 2, 3, 4, 5], [], [0, 2, 4, 6, 7], [1, 3, 5, 6, 7], [0, 1, 2, 3, 4, 5, 6],
             [1, 2, 3, 5, 6, 7], [0, 3, 6], [2, 5]]
    rp = [0]
    for c in cols8:
        rp.append(rp[-1] + len(c))
    a8 = Csr(8, 8, np.array(rp, dtype=np.int64), np.array(sum(cols8, []), dtype=np.int64),
             np.arange(1, 35, dtype=np.float64))
    A = r.build(a8, 4, 4)
    edges.append(dict(name="eight_by_eight_w4s4", row_ptr=rp, col_idx=sum(cols8, []), omega=4, sigma=4,
                      tile_ptr=[int(v) for v in A.tile_ptr], tile_desc=[int(v) for v in A.tile_desc],
                      eo_ptr=A.eo_ptr.tolist(), eo=A.eo.tolist(), p=A.p, pc=A.pc, tail=A.tail_len))
    with open(os.path.join(HERE, "ref_edges.json"), "w") as f:
        json.dump(edges, f, indent=1)
    print(f"wrote {len(meta)} w32 cases, {len(edges)} edge dumps")


def dumps():
    """dump_format of the reference's build of every golden case, keyed like
    ref_w32.npz (the inputs are read back from it)."""
    import gzip
    r = Ref()
    z = np.load(os.path.join(HERE, "ref_w32.npz"))
    meta = json.loads(str(z["meta"]))
    out = {}
    for c in meta:
        mk = c["mat"]
        a = Csr(c["m"], c["n"], z[f"{mk}_row_ptr"], z[f"{mk}_col_idx"].astype(np.int64),
                z[f"{mk}_val"])
        out[c["key"]] = r.dump_format(a, 32, c["sigma"])
    with gzip.open(os.path.join(HERE, "ref_dumps.json.gz"), "wt") as f:
        json.dump(out, f)
    print(f"wrote {len(out)} reference dumps")


if __name__ == "__main__":
    if "--dumps" not in sys.argv:
        main()
    dumps()
