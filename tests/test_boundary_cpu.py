"""CPU-side checks of the C-ABI boundary (no GPU needed, no compute calls)."""
import ast
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2510_15352_b200")
HEADER = os.path.join(ROOT, "include", "gg.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(gg_[a-z_0-9]+)\s*\(", src)
    return sorted(set(n for n in names if not n.startswith("gg_context")))


@pytest.fixture(scope="module")
def lib():
    so = os.path.join(PKG, "libgg.so")
    if not os.path.exists(so):
        subprocess.check_call(["sh", os.path.join(PKG, "build.sh")])
    import paper_2510_15352_b200 as gg
    return gg.load_library()


def test_header_declares_the_north_star_calls():
    fns = declared_functions()
    for must in ("gg_load_scene", "gg_render", "gg_create", "gg_destroy", "gg_debug_dump"):
        assert must in fns


def test_library_exports_every_declared_symbol(lib):
    import paper_2510_15352_b200 as gg
    fns = declared_functions()
    for f in fns:
        assert hasattr(lib, f), f"libgg.so does not export {f}"
    assert sorted(gg.EXPORTS) == fns


def test_nm_exports_are_c_linkage():
    so = os.path.join(PKG, "libgg.so")
    if not os.path.exists(so):
        pytest.skip("not built")
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    syms = {l.split()[-1] for l in out.splitlines() if l.strip()}
    for f in declared_functions():
        assert f in syms


def test_built_for_sm100a():
    so = os.path.join(PKG, "libgg.so")
    if not os.path.exists(so):
        pytest.skip("not built")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings_without_gpu(lib):
    import paper_2510_15352_b200 as gg
    assert gg.gg_status_string(gg.GG_E_BAD_SCENE) == "GG_E_BAD_SCENE"
    o = gg.default_opts()
    assert abs(o.near_plane - 0.01) < 1e-9 and o.sh_degree == -1 and o.debug_env == -1


def test_product_never_imports_oracle():
    """The product path shares no code with the oracle and has no CPU fallback."""
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            p = os.path.join(dirpath, f)
            if f.endswith(".py"):
                tree = ast.parse(open(p).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert not any(a.name.split(".")[0] == "oracle" for a in node.names), p
                    if isinstance(node, ast.ImportFrom):
                        assert (node.module or "").split(".")[0] != "oracle", p
            if f.endswith((".cu", ".cuh", ".h", ".cpp", ".sh")):
                txt = open(p).read()
                assert "gg_oracle" not in txt and "oracle/" not in txt, p


def test_missing_library_fails_loudly(tmp_path):
    import paper_2510_15352_b200 as gg
    saved = gg._lib
    gg._lib = None
    try:
        with pytest.raises(ImportError):
            gg.load_library(str(tmp_path / "nope.so"))
    finally:
        gg._lib = saved
