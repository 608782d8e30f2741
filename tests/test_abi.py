"""Boundary checks that need no GPU: the C-ABI library builds, loads and exports
every symbol include/sflsqr.h declares; without a device it fails loudly."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sflsqr.h")


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(sflsqr_[a-z_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    from paper_2605_22281_b200._build import build_library
    path = build_library()
    return ctypes.CDLL(path), path


def test_header_declares_the_boundary():
    names = _declared()
    for need in ("sflsqr_create", "sflsqr_set_operator", "sflsqr_set_sketch", "sflsqr_set_precond",
                 "sflsqr_iterate", "sflsqr_get_x", "sflsqr_get_residual_norms", "sflsqr_destroy"):
        assert need in names


def test_library_exports_every_declared_symbol(lib):
    _, path = lib
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (sflsqr_\w+)", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    from paper_2605_22281_b200.sflsqr import EXPORTED
    assert sorted(EXPORTED) == _declared()


def test_library_is_sm100a(lib):
    _, path = lib
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_create_without_gpu(lib):
    import torch
    from paper_2605_22281_b200 import sflsqr as B
    L = B.load_library()
    assert L.sflsqr_version() == 5
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the -m gpu tests")
    with pytest.raises(B.SflsqrError) as ei:
        B.SFLSQR(method="sflsqr", window=2, maxit=5)
    assert ei.value.code == B.E_CUDA


def test_option_validation_precedes_device_use(lib):
    from paper_2605_22281_b200 import sflsqr as B
    bad = [dict(method="nope"), dict(window=0), dict(maxit=0), dict(tol=-1.0), dict(eta=0.5), dict(delta_e=-1.0),
           dict(knobs=1 << 20), dict(knobs=["res_main", "res_side"]), dict(knobs=["p2p_on", "p2p_off"])]
    for kw in bad:
        with pytest.raises(B.SflsqrError) as ei:
            B.SFLSQR(**kw)
        assert ei.value.code == B.E_INVALID, kw


def test_ctypes_structs_match_header_layout(lib):
    # the binding's ctypes mirrors of sflsqr_opts / sflsqr_info / sflsqr_profile must have the C sizes
    # (compiled here from include/sflsqr.h with gcc, no GPU needed)
    import ctypes
    import os
    import tempfile
    from paper_2605_22281_b200 import sflsqr as B
    inc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
    src = ('#include "sflsqr.h"\n#include <stdio.h>\nint main(void){printf("%zu %zu %zu\\n", sizeof(sflsqr_opts),'
           ' sizeof(sflsqr_info), sizeof(sflsqr_profile)); return 0;}\n')
    with tempfile.TemporaryDirectory() as d:
        c, exe = os.path.join(d, "s.c"), os.path.join(d, "s")
        open(c, "w").write(src)
        subprocess.run(["gcc", "-I" + inc, c, "-o", exe], check=True)
        sizes = [int(t) for t in subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()]
    assert sizes == [ctypes.sizeof(B.Opts), ctypes.sizeof(B.Info), ctypes.sizeof(B.Profile)]


def test_knob_names_match_header():
    # opts.knobs: the binding's names carry the header's bit values, and SFLSQR_KNOB_ALL covers them
    from paper_2605_22281_b200 import sflsqr as B
    txt = open(HEADER).read()
    bits = {m.group(1).lower(): int(m.group(2), 16) for m in re.finditer(r"#define SFLSQR_KNOB_(\w+) (0x[0-9a-f]+)", txt)}
    allbits = bits.pop("all")
    assert bits == B.KNOBS
    assert allbits == sum(bits.values())


def test_comm_kinds_match_header_and_are_validated(lib):
    from paper_2605_22281_b200 import sflsqr as B
    txt = open(HEADER).read()
    kinds = {m.group(1): int(m.group(2)) for m in re.finditer(r"#define SFLSQR_COMM_(\w+) (\d+)", txt)}
    assert kinds == {"NCCL": B.COMM_NCCL, "LOCAL": B.COMM_LOCAL, "IPC": B.COMM_IPC}
    # world > 1 needs its transport's argument (checked before any device or shared-memory use)
    o = B.Opts()
    o.method, o.window, o.maxit, o.world, o.rank = 0, 2, 5, 2, 0
    for kind in (B.COMM_NCCL, B.COMM_IPC, B.COMM_LOCAL, 7):
        o.comm_kind = kind
        h = ctypes.c_void_p()
        assert B.load_library().sflsqr_create(ctypes.byref(h), ctypes.byref(o)) == B.E_INVALID
