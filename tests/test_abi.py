"""CPU: libs2v.so loads and exports every function include/s2v.h declares
(no compute calls -- there is no GPU here)."""
import ctypes
import re
from pathlib import Path

import paper_2105_08764_b200 as P
from paper_2105_08764_b200 import _lib

HEADER = Path(__file__).resolve().parent.parent / "include" / "s2v.h"


def declared():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(s2v_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("s2v_embed_round", "s2v_score", "s2v_apply_phase1", "s2v_apply_phase2",
                 "s2v_layer_backward", "s2v_adam", "s2v_comm_allgather_slots"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    assert set(declared()) <= set(_lib.exported_symbols())


def test_version_string():
    assert b"sm_100a" in _lib.load().s2v_version()


def test_status_codes_map_to_reference_exceptions():
    import pytest
    with pytest.raises(P.InvalidActionError):
        raise_for(_lib.S2V_EACTION)
    with pytest.raises(P.CollectiveError):
        raise_for(_lib.S2V_ECOMM)
    with pytest.raises(ValueError):
        raise_for(_lib.S2V_EINVAL)


def raise_for(code):
    _lib.check(code, "test")


def test_library_loads_without_torch():
    """The C ABI is self-contained: a plain ctypes caller (the reference's
    own binding) loads libs2v.so and finds the handle-level
    API without torch in the process."""
    import subprocess
    import sys
    code = ("import ctypes, sys; lib = ctypes.CDLL(%r); "
            "[getattr(lib, n) for n in ('s2v_ctx_create', 's2v_graph_upload', "
            "'s2v_state_create', 's2v_embed', 's2v_score_topk', 's2v_apply', 's2v_loss_grad', "
            "'s2v_adam_update', 's2v_copy_out')]; assert 'torch' not in sys.modules; "
            "print('ok')" % str(_lib.LIB_PATH))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stderr
