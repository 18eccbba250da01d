"""The C-ABI library loads and exports every symbol include/fek.h declares (CPU only).

No compute calls here: without a GPU only the pure-host entry points
(versions, status strings, error-key decoding, descriptor validation) run.
"""

import ctypes
import os
import subprocess

import pytest

from paper_1504_01023_b200 import _native
from paper_1504_01023_b200.csrc import gen_refconst

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_loads_from_the_package_directory():
    lib = _native.load()
    assert os.path.dirname(_native.LIB_PATH) == os.path.join(ROOT, "paper_1504_01023_b200")
    assert lib.fek_abi_version() == _native.ABI_VERSION


def test_every_header_function_is_exported_and_typed():
    declared = _native.header_functions()
    assert len(declared) >= 11
    lib = _native.load()
    for name in declared:
        assert hasattr(lib, name), name
        assert name in _native.SIGNATURES, f"{name} declared in fek.h but not bound in _native.py"
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(declared) <= exported


def test_sm100a_code_is_embedded():
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_decode():
    lib = _native.load()
    assert lib.fek_status_string(0) == b"ok"
    assert b"aligned" in lib.fek_status_string(_native.ERR_ALIGNMENT)

    def key(e, q, kind):
        blk, within = e >> 13, e & 8191
        return (blk << 24) | ((15 if q is None else q) << 20) | (within << 7) | kind

    for e, q, kind in ((0, 0, 1), (4, None, 2), (8200, 0, 2), (100, 4, 2), (2 ** 40 + 12345, 5, 1)):
        assert _native.decode_error(key(e, q, kind)) == (e, q, kind)
    # ordering = reference first-error rule: block, then point, then element
    assert key(100, 4, 2) < key(8200, 0, 2)
    assert key(7, 0, 2) < key(5, 3, 2)


def test_descriptor_validation_without_gpu():
    lib = _native.load()
    d = _native.BatchDesc()
    d.element, d.problem, d.variant, d.geometry_path = 1, 0, 0, 0  # geo_linear + prism: invalid
    d.layout, d.lane_width = 0, 1
    assert lib.fek_launch_config(ctypes.byref(d), None, None, None, None) == _native.ERR_ARGUMENT
    d.geometry_path = 1
    d.layout, d.lane_width = 1, 3
    assert lib.fek_launch_config(ctypes.byref(d), None, None, None, None) == _native.ERR_ARGUMENT
    d.lane_width = 8
    d.n_elements = 10
    d.geometry = 8  # misaligned pointer
    d.coefficients = d.stiffness = d.load = d.error_key = 16
    assert lib.fek_integrate(ctypes.byref(d), None) == _native.ERR_ALIGNMENT
    assert lib.fek_host_workspace_bytes(ctypes.byref(d), 3, 1024) > 3 * 1024 * (18 + 6 + 36 + 6) * 8


def test_jacobian_query_validated_without_gpu():
    """fek_jacobian / fek_error_detail reject bad element / point arguments before any launch."""
    lib = _native.load()
    d = _native.BatchDesc()
    d.element, d.problem, d.variant, d.geometry_path = 1, 0, 0, 1  # prism, generic
    d.layout, d.lane_width, d.n_elements = 0, 1, 4
    d.geometry = 256
    for fn in (lib.fek_jacobian, lib.fek_error_detail):
        assert fn(ctypes.byref(d), 0, 6, 512, None) == _native.ERR_ARGUMENT    # point out of range
        assert fn(ctypes.byref(d), 0, -1, 512, None) == _native.ERR_ARGUMENT   # affine query on a prism
        assert fn(ctypes.byref(d), 4, 0, 512, None) == _native.ERR_ARGUMENT    # element out of range
        assert fn(ctypes.byref(d), 0, 0, None, None) == _native.ERR_ARGUMENT   # no output


def test_v3_fields_validated_without_gpu():
    """ABI v3: misaligned tile-queue words and bad layout-conversion arguments are refused up front."""
    lib = _native.load()
    d = _native.BatchDesc()
    d.element, d.problem, d.variant, d.geometry_path = 0, 1, 0, 0
    d.layout, d.lane_width, d.n_elements = 0, 1, 10
    d.geometry = d.coefficients = d.stiffness = d.load = d.error_key = 256
    d.scheduler = 260  # not 8-byte aligned
    assert lib.fek_integrate(ctypes.byref(d), None) == _native.ERR_ALIGNMENT
    d.ctas_per_sm = -1
    assert lib.fek_integrate(ctypes.byref(d), None) == _native.ERR_ARGUMENT
    # fek_convert_layout: lane widths, row size, dtype, aliasing
    cv = lib.fek_convert_layout
    assert cv(256, 3, 512, 1, 10, 12, 0, 0.0, None) == _native.ERR_ARGUMENT
    assert cv(256, 1, 512, 128, 10, 12, 0, 0.0, None) == _native.ERR_ARGUMENT
    assert cv(256, 1, 512, 4, 10, 43, 0, 0.0, None) == _native.ERR_ARGUMENT
    assert cv(256, 1, 512, 4, 10, 12, 2, 0.0, None) == _native.ERR_ARGUMENT
    assert cv(256, 1, 256, 4, 10, 12, 0, 0.0, None) == _native.ERR_ARGUMENT
    assert cv(0, 1, 0, 4, 0, 12, 0, 0.0, None) == _native.OK  # empty: nothing to do


def test_refconst_header_is_current():
    path = os.path.join(ROOT, "paper_1504_01023_b200", "csrc", "refconst.h")
    assert open(path).read() == gen_refconst.render()


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_1504_01023_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(_native, "_lib", None)
    monkeypatch.setattr(_native, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(_native.NativeLibraryError):
        _native.load()


def test_integration_stub_struct_matches_the_library():
    """The ctypes stub in INTEGRATION.md lays out fek_batch_desc exactly as libfek does."""
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    start = text.index("class _Desc(ctypes.Structure)")
    block = text[start:text.index("\n\n", start)]
    ns = {"ctypes": ctypes}
    exec(block, ns)
    stub = ns["_Desc"]
    lib = _native.load()
    assert ctypes.sizeof(stub) == lib.fek_batch_desc_size() == ctypes.sizeof(_native.BatchDesc)
    ours = {name: getattr(_native.BatchDesc, name).offset for name, _ in _native.BatchDesc._fields_}
    assert {name: getattr(stub, name).offset for name, _ in stub._fields_} == ours
