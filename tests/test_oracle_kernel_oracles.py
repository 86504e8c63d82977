"""`adipc verify kernel-oracles` (tools/verify_suites.hpp:140-253, acceptance
#1) replayed on the oracle: the same seed (90210), the same draw sequence and
the same budgets (deterministic exact, parallel 1e-12, two-level 1e-10).
The per-case inputs are produced by the generators in kernel_cases.py, which
the GPU parity tests reuse."""
import numpy as np
import pytest

import oracle_py as O
from helpers import dense_from, map_accumulate
from kernel_cases import abd_cases, hash_cases, segment_cases, spmv_cases

# every test runs on the restatement and on the compiled reference (conftest)
pytestmark = pytest.mark.usefixtures("oracle_backend")

DET = O.ExecPolicy(deterministic=True)
PAR = O.ExecPolicy(threads=4, lane_width=8)


def test_kernel_oracles_suite():
    rng = O.Rng(90210)
    # lane walkthrough (:150-159)
    for pol in (DET, PAR):
        assert list(O.fast_segment_reduction([0, 0, 0, 1, 1, 1, 2, 2], np.ones(8), 3, pol)) == [3.0, 3.0, 2.0]

    seg_det_fail, seg_par_rel = 0, 0.0
    for Oseg, V, n_seg in segment_cases(rng):  # :161-191
        want = np.zeros(n_seg)
        for i in range(len(V)):
            want[Oseg[i]] += V[i]
        if not np.array_equal(O.fast_segment_reduction(Oseg, V, n_seg, DET), want):
            seg_det_fail += 1
        got = O.fast_segment_reduction(Oseg, V, n_seg, PAR)
        seg_par_rel = max(seg_par_rel, float(np.max(np.abs(got - want) / np.maximum(1, np.abs(want)))))
    assert seg_det_fail == 0 and seg_par_rel <= 1e-12

    hash_det_fail, hash_par_rel = 0, 0.0
    for n_blocks, keys, vals in hash_cases(rng):  # :192-215
        oracle = map_accumulate(keys, vals)
        sk, sv = O.sort_stream(keys, vals, DET)
        rows, cols, blocks = O.fast_hash_reduction(sk, sv, n_blocks, DET)
        if len(blocks) != len(oracle):
            hash_det_fail += 1
        else:
            for r, c, b in zip(rows, cols, blocks):
                if not np.array_equal(b, oracle.get((int(r) << 32) | int(c))):
                    hash_det_fail += 1
                    break
        sk, sv = O.sort_stream(keys, vals, PAR)
        rows, cols, blocks = O.fast_hash_reduction(sk, sv, n_blocks, PAR)
        for r, c, b in zip(rows, cols, blocks):
            want = oracle[(int(r) << 32) | int(c)]
            hash_par_rel = max(hash_par_rel, np.linalg.norm(b - want) / max(1, np.linalg.norm(want)))
    assert hash_det_fail == 0 and hash_par_rel <= 1e-12

    repro_fail, spmv_rel = 0, 0.0
    for n_blocks, rows, cols, blocks, x in spmv_cases(rng):  # :217-252
        want = dense_from(n_blocks, rows, cols, blocks) @ x
        scale = max(1.0, np.linalg.norm(want))
        y1 = O.srbk_spmv(n_blocks, rows, cols, blocks, x, DET)
        y2 = O.srbk_spmv(n_blocks, rows, cols, blocks, x, DET)
        yp = O.srbk_spmv(n_blocks, rows, cols, blocks, x, PAR)
        repro_fail += int(not np.array_equal(y1, y2))
        spmv_rel = max(spmv_rel, np.max(np.linalg.norm((y1 - want).reshape(-1, 3), axis=1)) / scale,
                       np.max(np.linalg.norm((yp - want).reshape(-1, 3), axis=1)) / scale)
    assert repro_fail == 0 and spmv_rel <= 1e-12

    abd_rel = 0.0
    for case in abd_cases(rng):  # :254-343
        for pol in (DET, PAR):
            tk, tv = O.two_level_abd_reduce(case["keys"], case["vals"], case["n_fem"], case["n_bodies"],
                                            case["body"], case["jac36"], pol)
            sk, sv = O.sort_stream(tk, tv, pol)
            rows, cols, blocks = O.fast_hash_reduction(sk, sv, case["n_blocks"], pol)
            D = dense_from(case["n_blocks"], rows, cols, blocks)
            abd_rel = max(abd_rel, np.linalg.norm(D - case["naive"]) / np.linalg.norm(case["naive"]))
    assert abd_rel <= 1e-10
