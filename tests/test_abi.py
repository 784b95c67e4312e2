"""CPU-side checks of the C-ABI library: it builds, loads, and exports every symbol that
include/sc.h declares (no compute calls: there is no GPU here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2310_14712_b200.build import build
    build()
    import paper_2310_14712_b200 as pkg
    return pkg.load_library()


def _declared():
    hdr = open(os.path.join(ROOT, "include", "sc.h")).read()
    return sorted(set(re.findall(r"\b(sc_[a-z_]+)\s*\(", hdr)))


def test_header_declares_the_boundary():
    names = _declared()
    for n in ("sc_setup", "sc_step", "sc_read", "sc_sync", "sc_query", "sc_destroy",
              "sc_read_classification", "sc_set_state", "sc_last_error", "sc_dof_coords"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    for n in _declared():
        assert hasattr(lib, n), n
        assert isinstance(getattr(lib, n), ctypes._CFuncPtr)


def test_binding_mirrors_header(lib):
    import paper_2310_14712_b200 as pkg
    assert sorted(pkg.EXPORTS) == _declared()


def test_struct_layouts(tmp_path):
    """ctypes mirrors match the C layout: compile a probe against include/sc.h."""
    import subprocess
    import paper_2310_14712_b200 as pkg
    names = ["sc_grid", "sc_void", "sc_geometry", "sc_source", "sc_dist", "sc_info"]
    src = tmp_path / "probe.c"
    src.write_text('#include <stdio.h>\n#include "sc.h"\nint main(void){' +
                   "".join(f'printf("%zu\\n", sizeof({n}));' for n in names) + "return 0;}\n")
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    sizes = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    assert sizes == [ctypes.sizeof(getattr(pkg, n)) for n in names]


def test_null_context_is_rejected(lib):
    # argument validation happens before any device call
    assert lib.sc_step(None, 1) == 7
    assert lib.sc_sync(None) == 7
    lib.sc_destroy(None)
