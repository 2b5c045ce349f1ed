"""The scheduler host mirror's id -> slot map (csrc/flat_idmap.hpp) against std::unordered_map
under a random operation mix (tests/cpp/flat_idmap_test.cpp; host-only, g++)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_flat_idmap_matches_unordered_map(tmp_path):
    exe = str(tmp_path / "flat_idmap_test")
    subprocess.run(["g++", "-O2", "-std=c++17", "-I",
                    os.path.join(ROOT, "paper_2604_00499_b200", "csrc"),
                    os.path.join(ROOT, "tests", "cpp", "flat_idmap_test.cpp"), "-o", exe],
                   check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
