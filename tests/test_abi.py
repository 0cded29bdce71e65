"""The C-ABI library builds for sm_100a, loads, and exports every symbol include/rnnt.h declares.
No compute calls (no GPU needed)."""
import ctypes
import os
import subprocess

import paper_2206_13236_b200 as R


def test_library_exports_header_symbols():
    lib = R.load_library()
    names = R.header_functions()
    assert {"rnnt_simple_loss", "rnnt_get_ranges", "rnnt_prune", "rnnt_pruned_loss",
            "rnnt_workspace_bytes", "rnnt_status_string"} <= set(names)
    for n in names:
        assert hasattr(lib, n), n
    assert "sm_100a" in R.rnnt_version()


def test_host_side_validation_and_workspace():
    """Host-only logic: argument validation returns synchronously without launching."""
    lib = R.load_library()
    d = R.make_dims(32, 500, 166, 500, 512, 5)
    ws = R.rnnt_workspace_bytes(d)
    assert ws > 0
    assert R.rnnt_workspace_bytes(R.make_dims(0, 5, 1, 5, 8, 2)) == 0        # N < 1
    assert R.rnnt_workspace_bytes(R.make_dims(2, 5, 1, 5, 12, 2)) == 0       # J % 8 != 0
    assert R.rnnt_workspace_bytes(R.make_dims(2, 5, 1, 5, 8, 33)) == 0       # S > 32
    # null pointers are rejected before any CUDA call
    rc = lib.rnnt_simple_loss(None, None, None, None, ctypes.byref(d), 0.5, None, None, None, None, None,
                              None, None, 0, None)
    assert rc == 1
    rc = lib.rnnt_get_ranges(None, None, None, ctypes.byref(d), None, None, None)
    assert rc == 1
    assert lib.rnnt_status_string(3) == b"RNNT_ERR_WORKSPACE"


def test_sass_is_sm100a():
    so = R.LIB_PATH
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_library_exports_only_the_c_abi():
    """The boundary is the C-ABI of include/rnnt.h and nothing else: every defined dynamic symbol of the
    shared library is a declared rnnt_* function (csrc/export.map keeps the C++ symbols local)."""
    out = subprocess.run(["nm", "-D", "--defined-only", R.LIB_PATH], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if len(ln.split()) >= 3 and ln.split()[-2] in "TtDdBb"}
    assert exported, "nm listed no symbols"
    assert exported == set(R.header_functions()), sorted(exported ^ set(R.header_functions()))
