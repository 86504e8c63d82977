"""GPU parity of the assembly path through the C-ABI against the oracle:
sort_stream, fast_hash_reduction (bit-exact with the reference's
deterministic mode), fast_segment_reduction, filter_pinned and
two_level_abd_reduce — the reference's kernel-oracle suites (seed 90210,
tools/verify_suites.hpp:140-343), its unit fixtures, edge cases (empty,
single, long rows crossing the warp / CTA sort limits) and the configs."""
import numpy as np
import pytest

import oracle_py as O
import paper_2411_06224_b200 as P
import scenegen as scenes
from paper_2411_06224_b200.context import Context, InvalidArgument
from helpers import Stream, cm, dense_from, map_accumulate
from kernel_cases import abd_cases, hash_cases, segment_cases

pytestmark = pytest.mark.gpu
DET = O.ExecPolicy(deterministic=True)


@pytest.fixture(scope="module")
def ctx():
    c = Context(0)
    yield c
    c.close()


def oracle_assemble(keys, vals, n):
    sk, sv = O.sort_stream(keys, vals, DET)
    return O.fast_hash_reduction(sk, sv, n, DET)


def gpu_assemble(ctx, keys, vals, n):
    U = ctx.assemble(keys, vals, n)
    nn, rows, cols, blocks = ctx.copy_matrix()
    assert nn == n and len(rows) == U
    return rows, cols, blocks


def assert_bitwise(got, want):
    for g, w in zip(got, want):
        assert g.shape == w.shape
        assert np.array_equal(g.view(np.uint8) if g.dtype == np.float64 else g,
                              w.view(np.uint8) if w.dtype == np.float64 else w)


def test_emission_fixture(ctx):  # test_block_sparse.cpp:72-91
    B1 = np.array([[1, 2, 3], [4, 5, 6], [7, 8, 9]], float)
    s = Stream()
    s.emit(2, 1, B1)
    s.emit(1, 2, 2 * np.eye(3))
    s.emit(1, 1, np.array([[0, 1, 0], [1, 0, 2], [0, 2, 0]], float))
    k, v = ctx.sort_stream(*s.arrays())
    ok, ov = O.sort_stream(*s.arrays())
    assert np.array_equal(k, ok) and np.array_equal(v, ov)
    rows, cols, blocks = gpu_assemble(ctx, *s.arrays(), 3)
    assert list(rows) == [1, 1] and list(cols) == [1, 2]
    assert np.array_equal(blocks[1], cm(B1.T) + cm(2 * np.eye(3)))


def test_sort_stream_random(ctx):  # :93-101 + stability
    rng = O.Rng(7)
    keys, vals = O.random_stream(rng, 40, 5000)
    k, v = ctx.sort_stream(keys, vals)
    ok, ov = O.sort_stream(keys, vals)
    assert np.array_equal(k, ok) and np.array_equal(v, ov)


def test_hash_reduction_suite_bitwise(ctx):  # verify_suites.hpp:192-215, 1000 cases
    rng = O.Rng(90210)
    for _ in segment_cases(rng):  # advance the shared RNG like the suite does
        pass
    fails = 0
    for n_blocks, keys, vals in hash_cases(rng):
        got = gpu_assemble(ctx, keys, vals, n_blocks)
        want = oracle_assemble(keys, vals, n_blocks)
        oracle = map_accumulate(keys, vals)
        assert len(got[2]) == len(oracle)
        for r, c, b in zip(*got):
            if not np.array_equal(b, oracle[(int(r) << 32) | int(c)]):
                fails += 1
        assert_bitwise(got, want)
    assert fails == 0


def test_segment_reduction_suite_bitwise(ctx):  # verify_suites.hpp:161-191
    rng = O.Rng(90210)
    for Oseg, V, n_seg in segment_cases(rng):
        want = np.zeros(n_seg)
        for i in range(len(V)):
            want[Oseg[i]] += V[i]
        got = ctx.segment_reduce(Oseg, V, n_seg)
        assert np.array_equal(got, want)
    assert list(ctx.segment_reduce([0, 0, 0, 1, 1, 1, 2, 2], np.ones(8), 3)) == [3.0, 3.0, 2.0]
    assert list(ctx.segment_reduce([0] * 12, np.ones(12), 1)) == [12.0]
    # Vec3 / Mat3 widths
    rng = np.random.default_rng(0)
    Oseg = np.sort(rng.integers(0, 50, 700)).astype(np.int32)
    for w in (3, 9):
        V = rng.standard_normal((700, w))
        assert np.array_equal(ctx.segment_reduce(Oseg, V, 50), O.fast_segment_reduction(Oseg, V, 50, DET))
    with pytest.raises(InvalidArgument):
        P.fast_segment_reduction([0, 0, 1], np.ones(2), 2)


def test_edge_cases(ctx):
    assert ctx.assemble(np.zeros(0, np.uint64), np.zeros((0, 9)), 5) == 0
    assert ctx.matrix_info() == (5, 0)
    keys = np.array([O.make_block_key(3, 4)], np.uint64)
    vals = np.arange(9, dtype=float).reshape(1, 9)
    assert_bitwise(gpu_assemble(ctx, keys, vals, 5), oracle_assemble(keys, vals, 5))
    with pytest.raises(InvalidArgument):  # row >= n_block_rows
        ctx.assemble(keys, vals, 3)


@pytest.mark.parametrize("row_len", [1, 2, 31, 32, 33, 63, 64, 65, 127, 128, 129, 255, 256, 257, 1000, 8191, 8192,
                                     8193, 32768, 32769, 40000, 65537, 140000])
def test_row_lengths(ctx, row_len):
    """Every row-sort regime: the register bitonic sorts of 32 / 64 / 128 / 256
    entries per warp and their boundaries, then rows longer than the warp sort
    (256) and the CTA sort (8192) limits: contact rows of affine bodies
    collect very many tiles; many duplicates."""
    rng = np.random.default_rng(row_len)
    cols = rng.integers(3, 3 + max(2, row_len // 7), row_len)
    keys = ((np.uint64(3) << np.uint64(32)) | cols.astype(np.uint64)).astype(np.uint64)
    extra = rng.integers(0, 50, 500)
    keys = np.concatenate([keys, ((extra.astype(np.uint64) << np.uint64(32)) | (extra + 1).astype(np.uint64))])
    perm = rng.permutation(len(keys))
    keys = keys[perm]
    vals = rng.standard_normal((len(keys), 9))
    n = int(max(cols.max(), 51)) + 1
    assert_bitwise(gpu_assemble(ctx, keys, vals, n), oracle_assemble(keys, vals, n))


def test_mixed_huge_rows(ctx):
    """Several rows beyond the multi-CTA sort limit (32,768 entries) with
    different merge-pass counts (odd and even: they finish in different
    ping-pong buffers), CTA-sorted rows, warp-sorted rows and long runs of
    one column (the segment reduction's single-run windows) in one stream."""
    rng = np.random.default_rng(77)
    parts = []
    for row, ln, ncol in ((5, 50000, 40), (9, 70000, 3000), (2, 20000, 7), (11, 300, 50), (0, 40, 10)):
        cols = rng.integers(row, row + ncol, ln)
        parts.append((np.uint64(row) << np.uint64(32)) | cols.astype(np.uint64))
    keys = np.concatenate(parts).astype(np.uint64)
    keys = keys[rng.permutation(len(keys))]
    vals = rng.standard_normal((len(keys), 9))
    n = 3100
    assert_bitwise(gpu_assemble(ctx, keys, vals, n), oracle_assemble(keys, vals, n))


@pytest.mark.parametrize("name", ["cfg1_soft_cube", "stiff_beam", "cfg2_cloth"])
def test_config_assembly_bitwise(ctx, name):
    sc = scenes.CONFIGS[name]()
    fk, fv = ctx.filter_pinned(sc.keys, sc.vals, sc.pinned)
    ok, ov = O.filter_pinned(sc.keys, sc.vals, sc.pinned)
    assert np.array_equal(fk, ok) and np.array_equal(fv, ov)
    assert_bitwise(gpu_assemble(ctx, fk, fv, sc.n_blocks), oracle_assemble(ok, ov, sc.n_blocks))


def test_two_level_suite(ctx):  # verify_suites.hpp:254-343, tiles bitwise + sandwich 1e-10
    rng = O.Rng(90210)
    for _ in segment_cases(rng):
        pass
    for _ in hash_cases(rng):
        pass
    from kernel_cases import spmv_cases
    for _ in spmv_cases(rng):
        pass
    worst = 0.0
    for case in abd_cases(rng):
        args = (case["keys"], case["vals"], case["n_fem"], case["n_bodies"], case["body"], case["jac36"])
        tk, tv = ctx.two_level_abd_reduce(*args)
        ok, ov = O.two_level_abd_reduce(*args, DET)
        assert np.array_equal(tk, ok) and np.array_equal(tv, ov)
        rows, cols, blocks = gpu_assemble(ctx, tk, tv, case["n_blocks"])
        D = dense_from(case["n_blocks"], rows, cols, blocks)
        worst = max(worst, np.linalg.norm(D - case["naive"]) / np.linalg.norm(case["naive"]))
    assert worst <= 1e-10


@pytest.mark.parametrize("name", ["cfg3_abd_stack", "cfg4_hybrid"])
def test_contact_configs_bitwise(ctx, name):
    """Two-level contact reduction + global assembly of the contact configs,
    bit-exact with the oracle's deterministic mode."""
    sc = scenes.CONFIGS[name]()
    args = (sc.node_keys, sc.node_vals, sc.n_fem, sc.n_bodies, sc.abd_body, sc.jac36)
    tk, tv = ctx.two_level_abd_reduce(*args)
    ok, ov = O.two_level_abd_reduce(*args, DET)
    assert np.array_equal(tk, ok) and np.array_equal(tv, ov)
    keys = np.concatenate([sc.keys, tk])
    vals = np.concatenate([sc.vals, tv])
    assert_bitwise(gpu_assemble(ctx, keys, vals, sc.n_blocks), oracle_assemble(keys, vals, sc.n_blocks))


def test_api_mirror(ctx):
    """api.py mirrors the reference signatures (block_coo.hpp / reduction.hpp)."""
    rng = O.Rng(11)
    keys, vals = O.random_stream(rng, 12, 400)
    s = P.BlockTripletStream(keys, vals)
    P.sort_stream(s, P.ExecPolicy(deterministic=True))
    A = P.fast_hash_reduction(s, 12, P.ExecPolicy(deterministic=True))
    want = oracle_assemble(keys, vals, 12)
    assert_bitwise((A.rows, A.cols, A.blocks), want)


@pytest.mark.parametrize("name", ["stiff_beam", "cfg1_soft_cube"])
def test_assemble_filtered_bitwise(ctx, name):
    """adipc_gpu_assemble_filtered = filter_pinned + sort_stream +
    fast_hash_reduction (incremental_potential.hpp:255-257), host and device
    pointers, bit-exact with the oracle."""
    import torch

    sc = scenes.CONFIGS[name]()
    pinned = sc.pinned.copy()
    pinned[::97] = 1
    ok, ov = O.filter_pinned(sc.keys, sc.vals, pinned)
    want = oracle_assemble(ok, ov, sc.n_blocks)
    ctx.assemble_filtered(sc.keys, sc.vals, sc.n_blocks, pinned)
    assert_bitwise(ctx.copy_matrix()[1:], want)
    dk = torch.from_numpy(sc.keys.view(np.int64)).cuda()
    dv = torch.from_numpy(sc.vals).cuda()
    dp = torch.from_numpy(pinned).cuda()
    torch.cuda.synchronize()  # the context runs on its own non-blocking stream
    ctx.assemble_filtered(dk, dv, sc.n_blocks, dp)
    assert_bitwise(ctx.copy_matrix()[1:], want)


@pytest.mark.parametrize("name", ["cfg4_hybrid", "stiff_beam"])
def test_against_compiled_reference(ctx, name):
    """GPU output against the reference's own code (oracle/_ref) directly:
    two-level tiles and the assembled matrix, bit-exact."""
    if not O.reference_available():
        pytest.skip("oracle/_ref unavailable")
    sc = scenes.CONFIGS[name]()
    keys, vals = O.filter_pinned(sc.keys, sc.vals, sc.pinned)
    with O.use_backend("reference"):
        if sc.n_bodies:
            args = (sc.node_keys, sc.node_vals, sc.n_fem, sc.n_bodies, sc.abd_body, sc.jac36)
            tk, tv = ctx.two_level_abd_reduce(*args)
            rk, rv = O.two_level_abd_reduce(*args, DET)
            assert np.array_equal(tk, rk) and np.array_equal(tv.view(np.uint8), rv.view(np.uint8))
            keys, vals = np.concatenate([keys, rk]), np.concatenate([vals, rv])
        want = oracle_assemble(keys, vals, sc.n_blocks)
    assert_bitwise(gpu_assemble(ctx, keys, vals, sc.n_blocks), want)


@pytest.mark.parametrize("case", ["empty", "all_pinned", "none_pinned", "random"])
def test_assemble_filtered_edge_cases(ctx, case):
    """filter_pinned on the keys only (values read in place through the
    original emission index, pinned identities appended after the stream):
    an empty stream, every slot pinned (A = identity), nothing pinned, and a
    random stream with duplicate keys touching pinned rows."""
    rng = np.random.default_rng(7)
    n = 40
    if case == "empty":
        keys, vals = np.zeros(0, np.uint64), np.zeros((0, 9))
    else:
        r = rng.integers(0, n, 3000)
        c = rng.integers(0, n, 3000)
        lo, hi = np.minimum(r, c), np.maximum(r, c)
        keys = ((lo.astype(np.uint64) << np.uint64(32)) | hi.astype(np.uint64)).astype(np.uint64)
        vals = rng.standard_normal((3000, 9))
    pinned = {"empty": rng.integers(0, 2, n), "all_pinned": np.ones(n), "none_pinned": np.zeros(n),
              "random": (rng.random(n) < 0.2)}[case].astype(np.uint8)
    ok, ov = O.filter_pinned(keys, vals, pinned)
    want = oracle_assemble(ok, ov, n)
    ctx.assemble_filtered(keys, vals, n, pinned)
    assert_bitwise(ctx.copy_matrix()[1:], want)


def test_dump_block_coo_from_device(ctx, tmp_path):
    """adipc_gpu_dump_block_coo (--dump-hessian, srbk_spmv.hpp:52-60) writes the
    device matrix as the same text as api.dump_block_coo, which the CPU suite
    checks byte for byte against the reference's own dump."""
    import io

    sc = scenes.CONFIGS["cfg1_soft_cube"]()
    fk, fv = ctx.filter_pinned(sc.keys, sc.vals, sc.pinned)
    ctx.assemble(fk, fv, sc.n_blocks)
    path = tmp_path / "hess.txt"
    ctx.dump_block_coo(path)
    n, rows, cols, blocks = ctx.copy_matrix()
    f = io.StringIO()
    P.dump_block_coo(P.SortedSymBlockCoo(n, rows, cols, blocks), f)
    assert path.read_text() == f.getvalue()
    with pytest.raises(InvalidArgument):
        ctx.dump_block_coo(tmp_path / "missing_dir" / "x.txt")


def test_assemble_filtered_pinned_host_overlap(ctx):
    """Host-pointer assembly from PINNED buffers: the values upload runs on
    the copy stream concurrently with the key filter and sort (only the
    reduction waits for it) — still bit-exact, and repeated calls reuse the
    upload buffers safely."""
    import torch

    sc = scenes.CONFIGS["stiff_beam"]()
    ok, ov = O.filter_pinned(sc.keys, sc.vals, sc.pinned)
    want = oracle_assemble(ok, ov, sc.n_blocks)
    hk = torch.from_numpy(sc.keys.view(np.int64)).pin_memory()
    hv = torch.from_numpy(sc.vals).pin_memory()
    hp = torch.from_numpy(sc.pinned).pin_memory()
    for _ in range(3):
        ctx.assemble_filtered(hk, hv, sc.n_blocks, hp)
        assert_bitwise(ctx.copy_matrix()[1:], want)


def test_dump_matrix_binary_round_trip(ctx, tmp_path):
    """adipc_gpu_dump_matrix_binary -> api.load_matrix_binary reproduces the
    device matrix bit for bit (the binary capture for offline oracle checks)."""
    sc = scenes.CONFIGS["cfg1_soft_cube"]()
    fk, fv = ctx.filter_pinned(sc.keys, sc.vals, sc.pinned)
    ctx.assemble(fk, fv, sc.n_blocks)
    ctx.dump_matrix_binary(tmp_path / "A.bin")
    A = P.load_matrix_binary(tmp_path / "A.bin")
    n, rows, cols, blocks = ctx.copy_matrix()
    assert A.n_block_rows == n
    assert_bitwise((A.rows, A.cols, A.blocks), (rows, cols, blocks))


@pytest.mark.parametrize("name,pin", [("cfg3_abd_stack", "none"), ("cfg3_abd_stack", "scene"),
                                      ("cfg4_hybrid", "scene"), ("cfg4_hybrid", "random")])
def test_assemble_contact_bitwise(ctx, name, pin):
    """adipc_gpu_assemble_contact: two_level_abd_reduce + stream_.append +
    filter_pinned + sort + reduce (incremental_potential.hpp:392-394,
    253-257) with the tiles kept on the device — bit-exact with the oracle's
    deterministic mode over the concatenated stream, host and device
    pointers."""
    import torch

    sc = scenes.CONFIGS[name]()
    pinned = {"none": np.zeros(sc.n_blocks, np.uint8), "scene": sc.pinned.copy(),
              "random": (np.random.default_rng(5).random(sc.n_blocks) < 0.05).astype(np.uint8)}[pin]
    args = (sc.node_keys, sc.node_vals, sc.n_fem, sc.n_bodies, sc.abd_body, sc.jac36)
    tk, tv = O.two_level_abd_reduce(*args, DET)
    keys, vals = O.filter_pinned(np.concatenate([sc.keys, tk]), np.concatenate([sc.vals, tv]), pinned)
    want = oracle_assemble(keys, vals, sc.n_blocks)
    U, nt = ctx.assemble_contact(sc.keys, sc.vals, sc.node_keys, sc.node_vals, sc.n_fem, sc.n_bodies, sc.abd_body,
                                 sc.jac36, sc.n_blocks, pinned)
    assert nt == len(tk) and U == len(want[0])
    assert_bitwise(ctx.copy_matrix()[1:], want)
    d = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    dk, dnk = d(sc.keys.view(np.int64)), d(sc.node_keys.view(np.int64))
    torch.cuda.synchronize()
    U2, nt2 = ctx.assemble_contact(dk, d(sc.vals), dnk, d(sc.node_vals), sc.n_fem, sc.n_bodies, d(sc.abd_body),
                                   d(sc.jac36), sc.n_blocks, d(pinned))
    assert (U2, nt2) == (U, nt)
    assert_bitwise(ctx.copy_matrix()[1:], want)
