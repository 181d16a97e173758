"""Regenerate tests/golden/* by running the REFERENCE library itself.

The reference is compiled in place from /root/reference/proj/include by
oracle/Makefile into oracle/_ref/libmhref.so (this container only; the GPU box
and the CPU suite use the committed fixtures).  Fixtures:

  bench_trials_seed0_n64_t8_q2.csv
      mh::run_trials({n=64,t=8,q=2,seed=0,trials=20}) -> write_trials_csv with the
      two timing columns stripped: the reference's own golden CSV
      (bench_test.cpp:528-549) reproduced by running it.
  first_draw_seed0_n64_t8_q2.json
      gen_problem's first draw at seed 0: descriptor triple + h = h*31 + v over the
      output container (bench_test.cpp:56-72).
  frozen_seed0_gf2.json
      multiply_test.cpp:134-163: 4x4 views A@(1,2) += B@(3,1) * C@(2,4) in 8x8
      containers (t=4, q=2) filled row-major from std::mt19937_64(0) % 2, run
      through the reference's mm_naive.
  cases.json
      seeded problems (gen_problem draws over several (n, t, q), three ops)
      with the reference's mm_oblivious Counters and the SHA-256 of the whole
      output container afterwards.

Usage: python tests/golden/make_golden.py
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.binding import OP_ADD, OP_SET, OP_SUB, Oracle, Reference  # noqa: E402

CASE_CONFIGS = [
    # (n, t, q, seed, draws)
    (32, 4, 2, 11, 4),
    (32, 8, 97, 12, 4),
    (64, 8, 65521, 13, 4),
    (64, 16, 2147483647, 14, 3),
    (128, 32, 65521, 15, 3),
    (128, 64, 16777213, 16, 2),
    (48, 3, 257, 17, 3),   # non-power-of-two tile side (layout_test.cpp:23)
]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.uint32).tobytes()).hexdigest()


def main():
    ref, orc = Reference(), Oracle()

    tmp = os.path.join(HERE, "_trials.csv")
    ref.run_trials_csv(64, 8, 2, 0, 20, 2, tmp)
    with open(tmp) as f:
        lines = f.read().splitlines()
    os.remove(tmp)
    with open(os.path.join(HERE, "bench_trials_seed0_n64_t8_q2.csv"), "w") as f:
        for ln in lines:
            f.write(",".join(ln.split(",")[:-2]) + "\n")

    out, lhs, rhs, aligned, v = ref.gen_problem(64, 8, 2, 0)
    h = 0
    for x in out:
        h = (h * 31 + int(x)) & (2 ** 64 - 1)
    with open(os.path.join(HERE, "first_draw_seed0_n64_t8_q2.json"), "w") as f:
        json.dump({"aligned": aligned, "out_origin": v.out_origin, "rows": v.rows, "cols": v.cols,
                   "lhs_origin": v.lhs_origin, "inner": v.inner, "rhs_origin": v.rhs_origin,
                   "out_hash31": h}, f, indent=1)

    g = orc.rng(0)
    grids = [np.array([g.next() % 2 for _ in range(64)], np.uint32).reshape(8, 8)
             for _ in range(3)]
    cells = [orc.rowmajor_to_mh(8, 4, gr) for gr in grids]
    from oracle.binding import Views
    vv = Views(orc.encode(8, 4, 1, 2), orc.encode(8, 4, 3, 1), orc.encode(8, 4, 2, 4), 4, 4, 4)
    a = cells[0].copy()
    ref.mm(0, 8, 4, 2, a, cells[1], cells[2], vv)
    res = orc.mh_to_rowmajor(8, 4, a)
    with open(os.path.join(HERE, "frozen_seed0_gf2.json"), "w") as f:
        json.dump({"grids_rowmajor": [gr.tolist() for gr in grids],
                   "result_rowmajor": res.tolist(),
                   "frozen_view": res[1:5, 2:6].tolist()}, f)

    cases = []
    for (n, t, q, seed, draws) in CASE_CONFIGS:
        g = orc.rng(seed)
        for d in range(draws):
            o, l_, r_, al, v = orc.gen_problem(g, n, t, q)
            for op in (OP_ADD, OP_SUB, OP_SET):
                a = o.copy()
                ctr = ref.mm(2, n, t, q, a, l_, r_, v, op=op)
                cases.append({"n": n, "t": t, "q": q, "seed": seed, "draw": d, "op": op,
                              "views": [v.out_origin, v.lhs_origin, v.rhs_origin, v.rows,
                                        v.inner, v.cols],
                              "counters": list(ctr.as_tuple()),
                              "out_sha256": sha(a)})
    with open(os.path.join(HERE, "cases.json"), "w") as f:
        json.dump(cases, f, indent=0)
    print(f"wrote {len(cases)} cases")


if __name__ == "__main__":
    main()
