"""Parity of the opt-in combine variants (environment-selected, read once per
process, so each runs the normal-mode parity cases in a fresh interpreter):

  EPB_COMBINE_MODE=stream             streamed push combine, TMA bulk-copy pushers
  EPB_COMBINE_MODE=stream, STREAM_TMA=0  streamed push, register pushers, one arrival word per row
  EPB_TMA=1                           bulk-copy (cp.async.bulk) reduce and dispatch copy path

Every variant must stay bit-exact against the oracle (tests/test_gpu_parity.py).
"""
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]

VARIANTS = {
    "stream_tma": {"EPB_COMBINE_MODE": "stream"},
    "stream_reg_row_flags": {"EPB_COMBINE_MODE": "stream", "EPB_COMBINE_STREAM_TMA": "0",
                             "EPB_COMBINE_FLAG_ROWS": "1", "EPB_COMBINE_PUSH_WARPS": "4"},
    "bulk_copy": {"EPB_TMA": "1"},
}


@pytest.mark.gpu
@pytest.mark.parametrize("variant", sorted(VARIANTS))
def test_combine_variant_parity(variant):
    env = dict(os.environ, **VARIANTS[variant])
    cmd = [sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
           str(ROOT / "tests" / "test_gpu_parity.py"), "-k",
           "test_dispatch_combine_emulated and nvlink or test_dispatch_fp8_tuple_emulated and nvlink"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert " passed" in r.stdout
