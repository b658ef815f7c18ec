"""CPU tests of the boundary: librnn.so loads and exports every symbol include/rnn.h declares,
and host-side argument checks reject bad calls without touching a GPU."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    with open(os.path.join(ROOT, "include", "rnn.h")) as f:
        src = f.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rnn_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2605_24207_b200 import build as b
    b.build()
    from paper_2605_24207_b200 import rnn
    return rnn.lib()


def test_every_declared_symbol_is_exported(lib):
    names = declared_functions()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n


def test_status_strings_and_version(lib):
    assert lib.rnn_abi_version() == 1
    assert lib.rnn_status_string(0) == b"RNN_OK"
    assert lib.rnn_status_string(4) == b"RNN_ERR_DUPLICATE_KEY"
    assert lib.rnn_status_string(99) == b"RNN_ERR_UNKNOWN"


def test_host_side_checks_without_gpu(lib):
    from paper_2605_24207_b200 import rnn
    # NULL index pointer -> invalid argument, detail in last error
    assert lib.rnn_join_aggregate_fwd(None, None, None, 0, C.c_float(0), None, None, 0, None) == 1
    assert b"required" in lib.rnn_last_error()
    # workspace size query is host-only
    idx = rnn.JoinIndexC()
    wsb = C.c_size_t(0)
    st = lib.rnn_build_join_index(C.c_void_p(16), C.c_void_p(16), 1000, C.c_void_p(16), 10, None,
                                  0, 0, 0, C.byref(idx), None, C.byref(wsb), None)
    assert st == 0 and wsb.value > 0
    # S given without the E column that joins it
    st = lib.rnn_build_join_index(None, C.c_void_p(16), 1000, C.c_void_p(16), 10, None, 0, 0, 0,
                                  C.byref(idx), None, C.byref(wsb), None)
    assert st == 1 and b"e_src_key" in lib.rnn_last_error()
    # bad projection shapes are rejected before any launch
    assert lib.rnn_project(C.c_void_p(16), 10, 10, 10, C.c_void_p(16), 9000, 10, None,
                           C.c_void_p(16), 9000, 0, None) == 5
    assert lib.rnn_hash_partition(None, 10, 0, 0, None, None) == 1


def test_round2_entry_points_host_checks(lib):
    """Host-side checks of the round-2 entry points: unknown precision, the fused ReLU backward
    without dX, an out-of-range L2 hit ratio -- all rejected before any device work."""
    v = C.c_void_p(16)
    # precision 3 does not exist (0 tf32, 1 3xtf32, 2 bf16)
    assert lib.rnn_project(v, 10, 8, 8, v, 8, 8, None, v, 8, 3, None) == 1
    assert b"precision" in lib.rnn_last_error()
    assert lib.rnn_project_bwd(v, 10, 8, 8, v, 8, 8, v, 8, v, 8, v, None, 3, v, 1 << 20, None) == 1
    # rnn_project_bwd_relu needs dX
    assert lib.rnn_project_bwd_relu(v, 10, 8, 8, v, 8, 8, v, 8, None, 8, v, None, None, 1, v,
                                    1 << 20, None) == 1
    assert b"dX" in lib.rnn_last_error()
    assert lib.rnn_stream_l2_window(None, v, 1024, C.c_float(1.5)) == 1
    assert lib.rnn_stream_l2_window(None, None, 1024, C.c_float(0.5)) == 1


def test_dhn_saved_entry_points_host_checks(lib):
    """rnn_dhn_fwd_save / rnn_dhn_bwd_saved reject a missing walk sum and unknown flags before
    any device work (an empty index has no groups, so no pointer is dereferenced)."""
    from paper_2605_24207_b200 import rnn
    idx = rnn.JoinIndexC()          # zeroed: n_groups = 0
    ops = (rnn.OperandC * 4)()
    # unknown flag bit
    st = lib.rnn_dhn_bwd_saved(C.byref(idx), 4, ops, None, 32, C.c_void_p(16), 32, None, 32,
                               C.c_uint32(2), None, 0, None)
    assert st == 1 and b"flags" in lib.rnn_last_error()
    assert lib.rnn_dhn_bwd_saved.argtypes is not None


def test_union_entry_points_host_checks(lib):
    """rnn_join_aggregate_fwd_union / rnn_join_aggregate_bwd_acc reject a beta outside {0, 1}
    and a MEAN union before any device work."""
    from paper_2605_24207_b200 import rnn
    idx = rnn.JoinIndexC()
    q = rnn.QueryC()
    v = C.c_void_p(16)
    assert lib.rnn_join_aggregate_fwd_union(C.byref(idx), C.byref(q), v, 128, v, v, 128,
                                            C.c_float(0.5), None, 0, None) == 1
    assert b"beta_acc" in lib.rnn_last_error()
    q.agg = rnn.AGG["mean"]
    assert lib.rnn_join_aggregate_fwd_union(C.byref(idx), C.byref(q), v, 128, v, v, 128,
                                            C.c_float(1.0), None, 0, None) != 0
    assert b"MEAN" in lib.rnn_last_error() or b"decomposable" in lib.rnn_last_error()
    assert lib.rnn_join_aggregate_bwd_acc(C.byref(idx), C.byref(q), None, 0, None, v, 128, None,
                                          None, None, v, C.c_float(2.0), None, 0, None) == 1
    assert b"beta_dst" in lib.rnn_last_error()
