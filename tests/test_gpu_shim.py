"""The drop-in boundary from C++ (INTEGRATION.md): tests/cpp/shim_driver.cpp
is built against the REFERENCE's own headers plus include/adipc_gpu.hpp
(`make -C oracle shim`, in the container that has /root/reference) and runs
the reference's CPU solve and the B200 solve through the shim in one process.
Parity: assembled matrix bitwise, MAS apply 1e-10, PCG iterations +-2 %,
solution 1e-5 relative L2."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DRIVER = os.path.join(ROOT, "oracle", "_ref", "shim_driver")


def test_shim_driver_built_against_product_library():
    if not os.path.exists(DRIVER):
        pytest.skip("oracle/_ref/shim_driver not built (needs /root/reference at build time)")
    out = subprocess.run(["ldd", DRIVER], capture_output=True, text=True).stdout
    assert "libadipc_gpu.so" in out and "paper_2411_06224_b200" in out


@pytest.mark.gpu
@pytest.mark.parametrize("grid", [8, 16])
def test_shim_driver_parity(grid):
    if not os.path.exists(DRIVER):
        pytest.skip("oracle/_ref/shim_driver not built (needs /root/reference at build time)")
    p = subprocess.run([DRIVER, str(grid)], capture_output=True, text=True, timeout=600)
    line = p.stdout.strip().splitlines()[-1]
    res = json.loads(line)
    assert res["assembly_bitwise"], res
    assert res["ok"] and p.returncode == 0, res
