"""CPU: the C-ABI library loads and exports every symbol include/holo_b200.h declares.
No compute calls: there is no GPU here."""
import ctypes

import pytest

from paper_1904_04884_b200 import _native as nat


def test_header_symbols_exported():
    lib = nat.load()
    declared = nat.header_functions()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    # the ctypes signature table covers the header exactly
    assert set(nat.SIGNATURES) == set(declared)


def test_version_and_shape_support():
    lib = nat.load()
    assert lib.holo_version() >= 1
    for n in (8, 64, 256, 1024, 2048, 4096):
        assert lib.holo_shape_supported(n, n) == 1
    assert lib.holo_shape_supported(1024, 256) == 1
    # general sides (mixed radix, gfft.cu): camera frames, odd ny
    for nx, ny in ((96, 64), (100, 100), (1280, 1024), (1000, 1000), (1920, 1080), (64, 99), (99, 64), (2 * 61, 64),
                   (2 * 67, 64), (4093, 8)):
        assert lib.holo_shape_supported(nx, ny) == 1, (nx, ny)
    for bad in (4, 7, 8192, 0, 4099):  # sides outside [8, 4096]
        assert lib.holo_shape_supported(bad, 64) == 0
    assert lib.holo_shape_supported(64, 5000) == 0


def test_invalid_arguments_are_status_codes_not_crashes():
    lib = nat.load()
    h = ctypes.c_void_p()
    assert lib.holo_create(None, 0, ctypes.byref(h)) == nat.HOLO_ERR_INVALID
    g = nat.Geometry(64, 64, 0, 1e-5, 1e-5, 5e-3, 632e-9)
    assert lib.holo_create(ctypes.byref(g), 0, ctypes.byref(h)) == nat.HOLO_ERR_INVALID
    assert "voxel counts" in nat.last_error()
    g = nat.Geometry(8192, 64, 4, 1e-5, 1e-5, 5e-3, 632e-9)
    assert lib.holo_create(ctypes.byref(g), 0, ctypes.byref(h)) == nat.HOLO_ERR_UNSUPPORTED
    with pytest.raises(ValueError):
        nat.check(nat.HOLO_ERR_UNSUPPORTED)
    assert lib.holo_destroy(None) == nat.HOLO_OK
    assert lib.holo_solve(None, None, None, None) == nat.HOLO_ERR_INVALID


def test_struct_layouts_match_header():
    # field order / sizes of the C structs (holo_geometry, holo_solver_config, holo_report)
    assert ctypes.sizeof(nat.Geometry) == 3 * 4 + 4 + 4 * 8  # int32 x3, pad, 4 doubles
    assert nat.Geometry.pitch.offset == 16
    assert nat.SolverConfig.step_size.offset == 32
    assert nat.SolverConfig.real_nonnegative.offset == 60 and ctypes.sizeof(nat.SolverConfig) == 64
    assert nat.Report.step_size.offset == 24
    assert nat.Report.nnz.offset == 56


def _header_struct_fields(name):
    """Field names of `typedef struct {...} name;` in include/holo_b200.h, in order."""
    import os
    import re
    hdr = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                            "holo_b200.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    m = re.search(r"typedef struct \{([^{}]*)\}\s*" + name + ";", hdr)
    assert m, name
    fields = []
    for decl in m.group(1).split(";"):
        decl = decl.strip()
        if not decl:
            continue
        names = decl.split(None, 1)[1]
        fields += [n.strip() for n in names.split(",")]
    return fields


@pytest.mark.parametrize("cname,pyname", [("holo_geometry", "Geometry"), ("holo_solver_config", "SolverConfig"),
                                          ("holo_report", "Report")])
def test_ctypes_structs_follow_the_header(cname, pyname):
    # the Python mirror of each ABI struct has the header's fields in the header's order
    py = [f[0] for f in getattr(nat, pyname)._fields_]
    assert py == _header_struct_fields(cname)
