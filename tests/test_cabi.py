"""CPU checks of the drop-in boundary: the CUDA library loads without a GPU and
exports every entry point declared in include/refusion_b200.h."""
import ctypes as C
import os
import re

import pytest

from paper_1905_02082_b200 import _lib
from paper_1905_02082_b200.build import LIB, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    text = open(os.path.join(ROOT, "include", "refusion_b200.h")).read()
    return sorted(set(re.findall(r"\b(rf_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        build()
    return C.CDLL(LIB)


def test_header_declares_expected_surface():
    names = declared_functions()
    assert set(names) == set(_lib.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing


def test_struct_layouts_match_header(tmp_path):
    # Compile a probe against the header and compare every struct size and
    # field offset with the ctypes mirror used by the Python layer and tests.
    structs = [_lib.rf_intrinsics, _lib.rf_volume_config, _lib.rf_registration_config, _lib.rf_mask_config,
               _lib.rf_pipeline_config, _lib.rf_frame, _lib.rf_frame_stats, _lib.rf_registration_result,
               _lib.rf_linearize_result, _lib.rf_frame_counters]
    lines = ['#include <stddef.h>', '#include <stdio.h>', '#include "refusion_b200.h"', "int main(void) {"]
    expect = []
    for s in structs:
        lines.append(f'printf("%zu\\n", sizeof({s.__name__}));')
        expect.append(C.sizeof(s))
        for name, _ in s._fields_:
            lines.append(f'printf("%zu\\n", offsetof({s.__name__}, {name}));')
            expect.append(getattr(s, name).offset)
    lines.append("return 0; }")
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    import subprocess
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    assert got == expect


def test_version_and_error_strings(lib):
    L = _lib.load()
    assert b"sm_100a" in L.rf_version()
    assert L.rf_last_error() is not None


def test_invalid_config_rejected_without_gpu():
    # Validation runs before any device work (VolumeConfig::Validate).
    from paper_1905_02082_b200 import api
    L = _lib.load()
    cfg = api.volume_config(truncation=0.001)
    h = C.c_void_p()
    assert L.rf_volume_create(C.byref(cfg), 0, C.byref(h)) == _lib.RF_INVALID_ARGUMENT
    cfg = api.volume_config(block_side=16)
    assert L.rf_volume_create(C.byref(cfg), 0, C.byref(h)) == _lib.RF_UNSUPPORTED
