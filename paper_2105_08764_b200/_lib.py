"""ctypes binding of libs2v.so (include/s2v.h) -- the only compute path.

There is no CPU fallback: importing a compute entry point without the built
extension, or without a CUDA device, raises immediately.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import CollectiveError, InvalidActionError

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libs2v.so"

S2V_OK, S2V_EINVAL, S2V_EACTION, S2V_ECOMM, S2V_ECUDA, S2V_ENONFINITE = range(6)
S2V_F32, S2V_F64 = 0, 1
KEY_BYTES = 16  # struct Key {uint64 s; uint64 inv;}
TOPK_MAX = 8
HUB_DEGREE = 4096  # include/s2v.h S2V_HUB_DEGREE


class s2v_eval_plan(ctypes.Structure):
    _fields_ = [("K", ctypes.c_int), ("L", ctypes.c_int), ("max_deg", ctypes.c_int),
                ("dmax", ctypes.c_int)] + [(f, ctypes.c_void_p) for f in (
                    "theta", "table", "h1_table", "h0", "h1", "colsum_ws")] + [
                ("colsum_ws_bytes", ctypes.c_size_t)] + [(f, ctypes.c_void_p) for f in (
                    "g", "u1", "scores", "block_keys", "out", "fracs", "ds")] + [
                ("nthr", ctypes.c_int), ("fallback", ctypes.c_int)] + [
                (f, ctypes.c_void_p) for f in (
                    "active", "picks", "evaluated", "error", "info", "applied", "removed",
                    "t_picks", "t_applied", "t_eval")]


class s2v_shard(ctypes.Structure):
    _fields_ = [
        ("num_nodes", ctypes.c_int64),
        ("batch", ctypes.c_int32),
        ("world", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("_pad", ctypes.c_int32),
        ("row_start", ctypes.c_int64),
        ("num_rows", ctypes.c_int64),
        ("rows_max", ctypes.c_int64),
        ("nnz", ctypes.c_int64),
        ("row_ptr", ctypes.c_void_p),
        ("cols", ctypes.c_void_p),
        ("col_ptr", ctypes.c_void_p),
        ("col_ent", ctypes.c_void_p),
        ("col_row", ctypes.c_void_p),
        ("rdeg", ctypes.c_void_p),
        ("sol", ctypes.c_void_p),
        ("cand", ctypes.c_void_p),
        ("residual", ctypes.c_void_p),
        ("order", ctypes.c_void_p),
        ("n_hub", ctypes.c_int64),
        ("active", ctypes.c_void_p),
        ("active_n", ctypes.c_void_p),
        ("active_ptr", ctypes.c_void_p),
        ("active_cols", ctypes.c_void_p),
        ("active_sol", ctypes.c_void_p),
    ]


_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_SZ = ctypes.c_size_t
_D = ctypes.c_double
_SH = ctypes.POINTER(s2v_shard)

_SIGNATURES = {
    "s2v_last_error": ([], ctypes.c_char_p),
    "s2v_version": ([], ctypes.c_char_p),
    "s2v_set_device": ([_I], _I),
    "s2v_shard_init": ([_SH, _P, _P, _P], _I),
    "s2v_segment_copy": ([_I, _P, _I, _I64, _P, _P], _I),
    "s2v_apply_phase1": ([_SH, _P, _I, _P, _I, _P, _P], _I),
    "s2v_apply_phase2": ([_SH, _P, _I, _P, _P, _P, _I, _P], _I),
    "s2v_e12_table": ([_I, _P, _P, _P, _I, _I, _P, _P], _I),
    "s2v_embed_round": ([_I, _SH, _P, _P, _I, _I, _P, _P, _P, _P], _I),
    "s2v_h1_table": ([_I, _P, _P, _I, _I, _P, _P], _I),
    "s2v_embed_round2_table": ([_I, _SH, _P, _P, _I, _I, _P, _P, _P, _P, _I, _P, _P], _I),
    "s2v_trow": ([_SH, _I, _P, _P], _I),
    "s2v_embed_round_peers": ([_I, _SH, _P, _P, _I, _I, _P, _P, _P, _I, _P, _P], _I),
    "s2v_colsum": ([_I, _SH, _I, _P, _P, _P, _SZ, _P], _I),
    "s2v_colsum_workspace": ([_SH, _I, _I], _SZ),
    "s2v_colsum_residual": ([_I, _SH, _I, _P, _P, _I, _P, _P, _SZ, _P, _I, _P, _P, _P, _P], _I),
    "s2v_colsum_residual_workspace": ([_SH, _I, _I], _SZ),
    "s2v_score_cached": ([_SH, _P, _P, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P], _I),
    "s2v_frontier_seed": ([_SH, _P, _I, _I, _P, _P, _P, _I64, _P], _I),
    "s2v_frontier_expand": ([_SH, _I, _P, _P, _P, _I64, _P, _P, _I64, _P], _I),
    "s2v_frontier_meta_size": ([_I], _I64),
    "s2v_frontier_bits_words": ([_SH], _I64),
    "s2v_frontier_bits_seed": ([_SH, _P, _I, _I, _P, _P, _P, _P], _I),
    "s2v_frontier_bits_expand": ([_SH, _P, _P, _P], _I),
    "s2v_frontier_bits_merge": ([_SH, _P, _P, _P, _I, _I, _P, _P, _P, _I64, _P, _P, _I64, _P], _I),
    "s2v_frontier_bits_nodes": ([_SH, _P, _P, _P, _P], _I),
    "s2v_active_compact": ([_SH, _P, _P, _P, _P, _I64, _P, _P, _P], _I),
    "s2v_sol_mark": ([_SH, _P, _P, _I, _P, _P], _I),
    "s2v_active_workspace": ([_I64], _I64),
    "s2v_score": ([_I, _SH, _I, _P, _P, _P, _P, _P, _I, _P, _P, _P, _P], _I),
    "s2v_score_blocks": ([_SH], _I),
    "s2v_topk_merge": ([_SH, _P, _I, _P, _P], _I),
    "s2v_score_keys": ([_SH, _P, _P, _I, _P, _P], _I),
    "s2v_score_keys_f64": ([_SH, _P, _P, _I, _P, _P], _I),
    "s2v_topk_below": ([_SH, _P, _P, _P, _P], _I),
    "s2v_u1": ([_I, _I, _I, _P, _P, _P, _P], _I),
    "s2v_u1_exact": ([_I, _I], _I),
    "s2v_merge_rank_keys": ([_I, _I, _I, _P, _P, _P], _I),
    "s2v_sum_ranks": ([_I, _I64, _P, _P, _P], _I),
    "s2v_sub_i64": ([_P, _P, _I, _P], _I),
    "s2v_eval_chain": ([_SH, ctypes.POINTER(s2v_eval_plan), _I, _P], _I),
    "s2v_select": ([_I, _I, _I64, _P, _P, _I, _I, _P, _P, _P, _P, _P, _P, _P], _I),
    "s2v_trace": ([_I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P], _I),
    "s2v_backward_blocks": ([_SH], _I),
    "s2v_grad_h_init": ([_I, _SH, _I, _P, _P, _P, _P, _P], _I),
    "s2v_layer_backward": ([_I, _SH, _I, _P, _P, _P, _P, _P, _P, _I, _P, _P], _I),
    "s2v_gather": ([_I, _SH, _I, _P, _P, _P], _I),
    "s2v_param_grads": ([_I, _SH, _I, _P, _P, _P, _P, _P, _P], _I),
    "s2v_theta2_terms_bytes": ([_I, _SH, _I], _SZ),
    "s2v_theta2_einsum": ([_I, _SH, _I, _P, _P, _P, _P], _I),
    "s2v_reduce_partials": ([_I, _P, _I, _I, _P, _P], _I),
    "s2v_head_backward": ([_I, _SH, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P], _I),
    "s2v_adam": ([_I, _P, _P, _P, _P, _I64, _D, _D, _D, _D, _D, _D, _D, _D, _P], _I),
    "s2v_adam_pack": ([_I, _P, _P, _P, _P, _I64, _D, _D, _D, _D, _D, _D, _D, _D, _P, _I, _P],
                      _I),
    "s2v_comm_unique_id": ([_P, _SZ], _I),
    "s2v_comm_init": ([_P, _I, _I, ctypes.POINTER(ctypes.c_void_p)], _I),
    "s2v_comm_destroy": ([_P], _I),
    "s2v_comm_allgather": ([_P, _P, _P, _SZ, _P], _I),
    "s2v_comm_allgather_slots": ([_P, _P, _SZ, _SZ, _I, _I, _P], _I),
    "s2v_comm_allreduce": ([_P, _P, _SZ, _I, _P], _I),
    "s2v_comm_allreduce_ordered": ([_P, _P, _SZ, _I, _P, _P], _I),
    "s2v_sum_ranks_typed": ([_I, _I, _I64, _P, _P, _P], _I),
    "s2v_enable_peer_access": ([_I], _I),
    "s2v_memcpy_async": ([_P, _P, _SZ, _P], _I),
    "s2v_ipc_export": ([_P, _P, ctypes.POINTER(ctypes.c_uint64)], _I),
    "s2v_ipc_import": ([_P, ctypes.POINTER(ctypes.c_void_p)], _I),
    "s2v_ipc_close": ([_P], _I),
    "s2v_stream_write_u32": ([_P, ctypes.c_uint32, _P], _I),
    "s2v_stream_wait_u32": ([_P, ctypes.c_uint32, _P], _I),
    "s2v_generate_ba": ([_I64, _I64, _P, _P], _I64),
    "s2v_generate_rmat": ([_I, _I64, _P, _D, _D, _D, _I64, _P], _I64),
    "s2v_build_csr": ([_I64, _P, _I64, _P, _P], _I),
    # handle-level API (library-owned memory; bound by plain-ctypes callers,
    # tests/handle_abi_child.py -- the Python mirror uses the entry points
    # above)
    "s2v_ctx_create": ([_I, _I, _I, _P, ctypes.POINTER(ctypes.c_void_p)], _I),
    "s2v_ctx_destroy": ([_P], _I),
    "s2v_group_create": ([_I, ctypes.POINTER(ctypes.c_void_p)], _I),
    "s2v_group_destroy": ([_P], _I),
    "s2v_ctx_create_in_group": ([_I, _I, _P, ctypes.POINTER(ctypes.c_void_p)], _I),
    "s2v_ctx_sync": ([_P], _I),
    "s2v_graph_upload": ([_P, _I64, _P, _P, ctypes.POINTER(ctypes.c_void_p)], _I),
    "s2v_graph_destroy": ([_P], _I),
    "s2v_state_create": ([_P, _P, _I, _P, ctypes.POINTER(ctypes.c_void_p)], _I),
    "s2v_state_destroy": ([_P], _I),
    "s2v_state_shard": ([_P, _SH], _I),
    "s2v_embed": ([_P, _P, _I, _P, _I, _I], _I),
    "s2v_global_sum": ([_P, _P, _P], _I),
    "s2v_score_topk": ([_P, _P, _I, _P, _P], _I),
    "s2v_apply": ([_P, _P, _P, _I, _P, _P], _I),
    "s2v_loss_grad": ([_P, _P, _I, _P, _I, _I, _P, _P, _P, ctypes.POINTER(ctypes.c_double)],
                      _I),
    "s2v_adam_update": ([_P, _I, _P, _P, _P, _P, _I64, _I, _D, _D, _D, _D], _I),
    "s2v_copy_out": ([_P, _P, _I, _P], _I),
    "s2v_shard_structure": ([_I64, _I, _I64, _I64, _P, _P, _I64, _P, _P, _P, _P, _P,
                             ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int32), _P],
                            _I),
}

_lib = None


def exported_symbols() -> list[str]:
    return sorted(_SIGNATURES)


def load() -> ctypes.CDLL:
    """Load libs2v.so (built by __graft_entry__.build()); fail loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    import torch  # noqa: F401  -- loads the CUDA runtime / NCCL torch was built with
    lib = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_GLOBAL if hasattr(os, "RTLD_GLOBAL") else 0)
    missing = [n for n in _SIGNATURES if not hasattr(lib, n)]
    if missing:
        raise RuntimeError(f"{LIB_PATH} is stale: missing symbols {missing}; rebuild it")
    for name, (args, res) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def check(rc: int, what: str = "") -> None:
    """Map an s2v_status onto the reference's exception types."""
    if rc == S2V_OK:
        return
    msg = load().s2v_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == S2V_EACTION:
        raise InvalidActionError(text)
    if rc == S2V_ECOMM:
        raise CollectiveError(text)
    if rc in (S2V_EINVAL, S2V_ENONFINITE):
        raise ValueError(text)
    raise RuntimeError(f"libs2v CUDA failure: {text}")


# kernels each entry point launches (for the bench's gpu_launches claim)
KERNELS_PER_CALL = {
    "s2v_shard_init": 2, "s2v_apply_phase1": 1, "s2v_apply_phase2": 2, "s2v_e12_table": 1,
    "s2v_embed_round": 1, "s2v_embed_round_peers": 1, "s2v_colsum": 2, "s2v_score": 1, "s2v_topk_merge": 1, "s2v_score_keys": 1, "s2v_score_keys_f64": 1,
    "s2v_topk_below": 1,
    "s2v_grad_h_init": 1, "s2v_layer_backward": 1, "s2v_gather": 1, "s2v_param_grads": 1,
    "s2v_reduce_partials": 1, "s2v_head_backward": 1, "s2v_adam": 1, "s2v_theta2_einsum": 2,
    "s2v_u1": 1, "s2v_select": 1, "s2v_trace": 1,
    "s2v_h1_table": 1, "s2v_embed_round2_table": 1, "s2v_trow": 1, "s2v_colsum_residual": 3,
    "s2v_active_compact": 3, "s2v_sol_mark": 1, "s2v_score_cached": 2, "s2v_frontier_seed": 3,
    "s2v_frontier_expand": 9, "s2v_frontier_bits_seed": 3, "s2v_frontier_bits_expand": 2,
    "s2v_frontier_bits_merge": 4, "s2v_frontier_bits_nodes": 1, "s2v_adam_pack": 2, "s2v_segment_copy": 1,
    "s2v_merge_rank_keys": 1, "s2v_sum_ranks": 1, "s2v_sub_i64": 1, "s2v_sum_ranks_typed": 1,
    "s2v_comm_allreduce_ordered": 1,
    "s2v_eval_chain": 14,  # L = 5: 4 rounds, colsum 2, u1, score, merge, select, apply 3, trace
}
launch_count = 0


def call(name: str, *args) -> None:
    global launch_count
    check(getattr(load(), name)(*args), name)
    launch_count += KERNELS_PER_CALL.get(name, 0)
