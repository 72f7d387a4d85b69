"""The C ABI driven from a plain C program (tests/c/abi_smoke.c): create ->
load_edges -> augment -> push -> train_episode -> get_* -> destroy on the
GPU, no Python in the loop."""
import subprocess

import pytest

from test_abi import build_c_smoke

pytestmark = pytest.mark.gpu


def test_plain_c_program_runs_on_the_gpu(tmp_path):
    exe = build_c_smoke(str(tmp_path))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, (r.returncode, r.stdout, r.stderr)
    assert "-> ok" in r.stdout
