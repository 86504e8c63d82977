"""CPU-only checks of the product library: the C-ABI .so loads and exports
every symbol include/adipc_gpu.h declares (no compute calls), and the native
host-side partition / hierarchy code (csrc/host_precond.cpp) is integer-exact
against the oracle restatement of precond/partition.hpp and hierarchy.hpp."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle_py as O
import paper_2411_06224_b200 as P
from paper_2411_06224_b200 import _lib
import scenegen as scenes
from helpers import sixteen_slot_graph_edges

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "adipc_gpu.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return set(re.findall(r"\b(adipc_\w+)\s*\(", hdr))


def test_header_symbols_exported_and_bound():
    syms = declared_symbols()
    assert len(syms) >= 30
    lib = ctypes.CDLL(_lib.GPU_LIB)
    for s in sorted(syms):
        assert hasattr(lib, s), f"{s} declared in adipc_gpu.h but not exported"
    assert syms == set(_lib.GPU_SIGNATURES), "ctypes binding out of sync with the header"


def test_library_is_sm100a_only():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {_lib.GPU_LIB} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_subdomain_count_and_chunk():
    for args in [(100, 16, 1), (100, 16, 0), (16, 16, 0), (17, 16, 0), (100, 32, 0), (1, 16, 0)]:
        assert P.subdomain_count(*args) == O.subdomain_count(*args)
    for v, cap in [(10, 4), (16, 4), (0, 4), (1000, 16)]:
        p = P.chunk_partition(v, cap)
        part, n = O.chunk_partition(v, cap)
        assert p.n_parts == n and np.array_equal(p.part_of, part)


def _random_graph(rng, v, m, clusters=False):
    a = rng.integers(0, v, m)
    if clusters:  # mostly local edges: mesh-like components
        b = np.clip(a + rng.integers(-6, 7, m), 0, v - 1)
    else:
        b = rng.integers(0, v, m)
    return np.stack([a, b], 1).astype(np.int32)


@pytest.mark.parametrize("seed", range(12))
def test_partition_matches_oracle_random(seed):
    rng = np.random.default_rng(seed)
    v = int(rng.integers(1, 400))
    e = _random_graph(rng, v, int(rng.integers(0, 3 * v)), clusters=seed % 2 == 0)
    for cap in (2, 4, 7, 16, 32):
        p = P.partition_block_graph(v, e, cap)
        part, n = O.partition_block_graph(v, e, cap)
        assert p.n_parts == n
        assert np.array_equal(p.part_of, part)


def _check_hierarchy(part, n_parts, cap, edges, max_levels):
    h = P.build_hierarchy(P.Partition(part, n_parts, cap), edges, max_levels)
    ho = O.Hierarchy(part, n_parts, cap, edges, max_levels)
    assert h.n_levels() == ho.n_levels()
    for a, b in zip(h.levels, ho.levels):
        assert a["n_nodes"] == b["n_nodes"] and a["n_parts"] == b["n_parts"]
        assert np.array_equal(a["part_of"], b["part_of"])
        assert np.array_equal(a["agg"], b["agg"])
    return h


def test_hierarchy_fixtures():  # test_precond.cpp:130-177 through the product library
    edges = sixteen_slot_graph_edges()
    c = P.chunk_partition(16, 4)
    h = _check_hierarchy(c.part_of, c.n_parts, 4, edges, 8)
    assert h.n_levels() == 3
    assert list(h.levels[1]["agg"]) == [0, 1, 2, 1, 3, 4, 5, 4, 6, 6, 6, 6, 7, 8, 7, 8]
    assert list(h.levels[2]["agg"]) == [0, 1, 0, 1, 2, 1, 2, 1, 3, 3, 3, 3, 2, 0, 2, 0]
    g = P.partition_block_graph(16, edges, 4)
    h = _check_hierarchy(g.part_of, g.n_parts, 4, edges, 8)
    assert h.n_levels() == 2 and h.levels[1]["n_parts"] == 1
    assert _check_hierarchy(c.part_of, c.n_parts, 4, edges, 2).n_levels() == 2
    assert _check_hierarchy(c.part_of, c.n_parts, 4, np.zeros((0, 2), np.int32), 8).n_levels() == 1


@pytest.mark.parametrize("seed", range(8))
def test_hierarchy_matches_oracle_random(seed):
    rng = np.random.default_rng(100 + seed)
    v = int(rng.integers(2, 600))
    e = _random_graph(rng, v, int(rng.integers(v, 4 * v)), clusters=True)
    cap = int(rng.choice([4, 8, 16]))
    part, n = O.partition_block_graph(v, e, cap)
    _check_hierarchy(part, n, cap, e, 4)
    part, n = O.chunk_partition(v, cap)
    _check_hierarchy(part, n, cap, e, 6)


@pytest.mark.parametrize("name", ["cfg1_soft_cube", "stiff_beam"])
def test_mesh_partition_and_hierarchy(name):
    """L0 CEMAS partition of the rest connectivity (newton.hpp:66-67) and the
    hierarchy over the pinned-filtered matrix pattern, as the solver builds it."""
    sc = scenes.CONFIGS[name]()
    l0 = P.partition_block_graph(sc.n_blocks, sc.rest_edges, 16)
    part, n = O.partition_block_graph(sc.n_blocks, sc.rest_edges, 16)
    assert l0.n_parts == n and np.array_equal(l0.part_of, part)
    fk, fv = O.filter_pinned(sc.keys, sc.vals, sc.pinned)
    sk, sv = O.sort_stream(fk, fv, O.ExecPolicy(deterministic=True))
    rows, cols, _ = O.fast_hash_reduction(sk, sv, sc.n_blocks, O.ExecPolicy(deterministic=True))
    be = O.block_edges(rows, cols)
    _check_hierarchy(l0.part_of, l0.n_parts, 16, be, 4)


def test_scene_sizes_match_reference_generators():
    """Counts of SURVEY.md Appendix B (reference generator connectivity)."""
    s = scenes.CONFIGS["cfg1_soft_cube"]()
    assert s.n_blocks == 1728 and len(s.keys) == 81588
    s = scenes.CONFIGS["stiff_beam"]()
    assert s.n_blocks == 5040 and len(s.keys) == 251880 and int(s.pinned.sum()) == 144


def test_load_matrix_binary_format(tmp_path):
    """api.load_matrix_binary: the ADIPCMAT layout (magic, version, n, U, rows,
    cols, column-major blocks) and its error on foreign files."""
    import numpy as np
    import pytest

    from paper_2411_06224_b200 import api as P

    rows = np.array([0, 0, 1], np.uint32)
    cols = np.array([0, 1, 1], np.uint32)
    blocks = np.arange(27, dtype=np.float64).reshape(3, 9)
    raw = (b"ADIPCMAT" + np.uint32(1).tobytes() + np.int32(2).tobytes() + np.int64(3).tobytes() + rows.tobytes()
           + cols.tobytes() + blocks.tobytes())
    (tmp_path / "m.bin").write_bytes(raw)
    A = P.load_matrix_binary(tmp_path / "m.bin")
    assert A.n_block_rows == 2 and np.array_equal(A.rows, rows) and np.array_equal(A.cols, cols)
    assert np.array_equal(A.blocks, blocks)
    (tmp_path / "bad.bin").write_bytes(b"NOTAMATRIX" + bytes(20))
    with pytest.raises(ValueError):
        P.load_matrix_binary(tmp_path / "bad.bin")
