"""Host sanitizers on the oracle (SURVEY §5 'race detection / sanitizers'):
every entry point, each strategy, dimension and data shape, built with
-fsanitize=address,undefined (compute-sanitizer is closed on the GPU pool)."""
import os
import shutil
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


@pytest.mark.skipif(shutil.which("gcc") is None, reason="gcc missing")
def test_oracle_under_asan_ubsan(tmp_path):
    exe = str(tmp_path / "oracle_san")
    subprocess.check_call(["gcc", "-O1", "-g", "-std=gnu11", "-fsanitize=address,undefined",
                           "-fno-sanitize-recover=all", "-ffp-contract=off",
                           "-I" + os.path.join(ROOT, "oracle"), os.path.join(HERE, "helpers", "oracle_san.c"),
                           os.path.join(ROOT, "oracle", "rt_oracle.c"), "-o", exe, "-lm"])
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, ASAN_OPTIONS="detect_leaks=1"))
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 errors" in r.stdout
