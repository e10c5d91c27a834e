"""The C-ABI library builds, loads and exports every symbol of
include/clothsim_b200.h; the ctypes descriptor matches the C layout; the
product fails loudly (no CPU fallback) when no device is present."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT, cuda_available
from paper_2507_11794_b200 import _native as N

HEADER = os.path.join(ROOT, "include", "clothsim_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|const char \*)\s*\**\s*(cs_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = N.load()
    syms = declared_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
        assert s in N.SIGNATURES, s
    assert lib.cs_abi_version() == N.ABI_VERSION


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout, out.stdout + out.stderr


def test_descriptor_layout_matches_c(tmp_path):
    src = tmp_path / "layout.c"
    fields = [f for f, _ in N.CsDesc._fields_]
    body = "\n".join(f'printf("{f} %zu\\n", offsetof(cs_desc, {f}));' for f in fields)
    src.write_text(
        "#include <stdio.h>\n#include <stddef.h>\n#include \"clothsim_b200.h\"\n"
        "int main(void){\n" + body + '\nprintf("sizeof %zu\\n", sizeof(cs_desc));'
        '\nprintf("stats %zu\\n", sizeof(cs_stats));'
        '\nprintf("peer %zu\\n", sizeof(cs_halo_peer));'
        '\nprintf("peer_flag %zu\\n", offsetof(cs_halo_peer, remote_flag));\nreturn 0;}\n')
    exe = tmp_path / "layout"
    cc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
    subprocess.run([cc, "-I", os.path.dirname(HEADER), str(src), "-o", str(exe)], check=True)
    out = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True,
                                                        text=True).stdout.splitlines())
    for f in fields:
        assert int(out[f]) == getattr(N.CsDesc, f).offset, f
    assert int(out["sizeof"]) == ctypes.sizeof(N.CsDesc)
    assert int(out["stats"]) == ctypes.sizeof(N.CsStats)
    assert int(out["peer"]) == ctypes.sizeof(N.CsHaloPeer)
    assert int(out["peer_flag"]) == N.CsHaloPeer.remote_flag.offset


def test_grid_descriptor_layout_matches_c(tmp_path):
    src = tmp_path / "glayout.c"
    fields = [f for f, _ in N.CsGridDesc._fields_]
    body = "\n".join(f'printf("{f} %zu\\n", offsetof(cs_grid_desc, {f}));' for f in fields)
    src.write_text(
        "#include <stdio.h>\n#include <stddef.h>\n#include \"clothsim_b200.h\"\n"
        "int main(void){\n" + body + '\nprintf("sizeof %zu\\n", sizeof(cs_grid_desc));\nreturn 0;}\n')
    exe = tmp_path / "glayout"
    cc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
    subprocess.run([cc, "-I", os.path.dirname(HEADER), str(src), "-o", str(exe)], check=True)
    out = dict(line.split() for line in subprocess.run([str(exe)], capture_output=True,
                                                        text=True).stdout.splitlines())
    for f in fields:
        assert int(out[f]) == getattr(N.CsGridDesc, f).offset, f
    assert int(out["sizeof"]) == ctypes.sizeof(N.CsGridDesc)


def test_adapter_none_is_refused(monkeypatch):
    from paper_2507_11794_b200 import AdapterUnavailable, get_adapter

    monkeypatch.setenv("CLOTHSIM_ADAPTER", "none")
    with pytest.raises(AdapterUnavailable):
        get_adapter()


@pytest.mark.skipif(cuda_available(), reason="host has a GPU")
def test_no_device_fails_loudly_instead_of_falling_back():
    import paper_2507_11794_b200 as P

    with pytest.raises(P.AdapterUnavailable):
        P.Engine(P.generate_cloth_grid(4, 4))
    # and the raw ABI reports it as CS_E_NODEVICE
    d = N.CsDesc()
    d.abi_version = N.ABI_VERSION
    h = ctypes.c_void_p()
    assert N.load().cs_create(ctypes.byref(d), ctypes.byref(h)) in (N.CS_E_INVALID, N.CS_E_NODEVICE)


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2507_11794_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in text.replace("oracles", ""), f
