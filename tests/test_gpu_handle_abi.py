"""The handle-level C ABI (s2v_ctx / s2v_graph / s2v_state, library-owned
device memory) driven from plain ctypes in a process that never imports
torch: forward bits, a whole adaptive solve trajectory and a training step
against the reference's golden fixtures (tests/handle_abi_child.py)."""
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu


def test_handle_abi_without_torch():
    child = Path(__file__).resolve().parent / "handle_abi_child.py"
    r = subprocess.run([sys.executable, str(child)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert r.stdout.strip().startswith("OK")
