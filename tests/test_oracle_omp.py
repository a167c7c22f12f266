"""The timing-only OpenMP build of the oracle (liboracle_omp.so, ORACLE_OMP=1; tools/config_sweep.py's
"oracle-omp" row) gives bitwise the plain build's FGMRES solution: its OMP_ROWS loops are row-independent and
every reduction stays sequential, so only the wall time may differ."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(omp, opts):
    env = dict(os.environ, ORACLE_OMP="1" if omp else "0", OMP_NUM_THREADS="4")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "oracle_run.py"), "C1", json.dumps(opts)],
                         env=env, capture_output=True, text=True, check=True, timeout=300).stdout
    return json.loads(out.strip().splitlines()[-1])


@pytest.mark.parametrize("opts", [{}, {"amg_smoother": 2}, {"local_sweeps": 2, "aps_mode": 1}])
def test_omp_build_is_bitwise_the_plain_oracle(opts):
    a, b = _run(False, opts), _run(True, opts)
    assert a["oracle_lib"].endswith("liboracle.so")
    assert b["oracle_lib"].endswith("liboracle_omp.so")
    assert a["iterations"] == b["iterations"]
    assert a["x_sha1"] == b["x_sha1"]
