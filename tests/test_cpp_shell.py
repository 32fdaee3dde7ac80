"""The C++ drop-in shell (include/tofsplat_b200/splat.hpp) runs the reference's
test_splat / test_trainer cases through libtsb.so on the GPU."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parent.parent / "paper_2505_05356_b200" / "build" / "test_splat_b200"


@pytest.mark.gpu
def test_cpp_dropin_shell():
    assert BIN.exists(), "build the C++ test with __graft_entry__.build()"
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


def test_cpp_shell_builds_and_links():
    assert BIN.exists()
    out = subprocess.run(["ldd", str(BIN)], capture_output=True, text=True).stdout
    assert "libtsb.so" in out and "not found" not in out.split("libtsb.so")[1].split("\n")[0]
