"""C ABI checks that need no GPU: libpndf.so builds for sm_100a, loads, and exports every
symbol include/pndf.h declares; the binding has no compute fallback."""
import ctypes
import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pndf.h")


@pytest.fixture(scope="module")
def libpath():
    from paper_2109_14807_b200 import build
    if shutil.which("nvcc") is None and not os.path.exists(build.LIB):
        pytest.skip("nvcc unavailable and libpndf.so not built")
    return build.build()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pndf_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("pndf_load_factors", "pndf_query_batch", "pndf_sync"):  # BASELINE.json north_star's three calls
        assert must in names


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    for name in declared_functions():
        assert hasattr(lib, name), name
    nm = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    for name in declared_functions():
        assert re.search(rf"\bT {name}\b", nm), name


def test_calls_that_need_no_gpu(libpath):
    from paper_2109_14807_b200 import pndf
    assert pndf.lib().pndf_abi_version() == pndf.ABI_VERSION
    assert pndf.error_string(pndf.EQUERY).startswith("invalid query")
    assert pndf.error_string(pndf.OK) == "ok"
    assert pndf.lib().pndf_free(None) == 0
    # argument errors are returned synchronously, before any device work
    L = pndf.lib()
    assert L.pndf_query_batch(None, None, 0, None, 0, None) == pndf.EINVAL
    assert L.pndf_sample_batch(None, None, None, 0, None, 0, None) == pndf.EINVAL
    assert L.pndf_sample_tiles(None, None, None, 0, None, None, 0, None) == pndf.EINVAL
    assert L.pndf_sync(None, None) == pndf.EINVAL


def test_binding_matches_header_constants():
    from paper_2109_14807_b200 import pndf
    src = open(HEADER).read()
    for name, val in (("PNDF_WRAP", pndf.WRAP), ("PNDF_SUM", pndf.SUM), ("PNDF_BIN_ON", pndf.BIN_ON),
                      ("PNDF_BIN_OFF", pndf.BIN_OFF), ("PNDF_TIMING", pndf.TIMING),
                      ("PNDF_ABI_VERSION", pndf.ABI_VERSION)):
        m = re.search(rf"#define {name} (\d+)u", src)
        assert m and int(m.group(1)) == val, name
    assert set(pndf.EXPORTS) == set(declared_functions())


def test_sm100a_cubin_embedded(libpath):
    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump unavailable")
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    from paper_2109_14807_b200 import pndf
    monkeypatch.setattr(pndf, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(pndf, "_lib", None)
    with pytest.raises(RuntimeError, match="no fallback"):
        pndf.lib()
