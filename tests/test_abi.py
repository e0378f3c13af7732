"""The C ABI boundary without a GPU: the library loads, exports every symbol declared in
include/scalesim.h, the ctypes structs match the C layout, and the pure host entry points
validate their arguments (S:487 config errors -> SCALESIM_E_INVALID)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2601_21473_b200 import build
    build.build()
    from paper_2601_21473_b200 import _lib
    return _lib


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "scalesim.h")).read()
    return sorted(set(re.findall(r"\b(scalesim_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    lib = L.lib()
    decl = declared_symbols()
    assert set(decl) == set(L.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", L.SO_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(scalesim_[a-z_0-9]+)\b", out))
    for s in decl:
        assert s in exported, s
        assert hasattr(lib, s)


def test_struct_layout_matches_c(L, tmp_path):
    prog = tmp_path / "sz.c"
    prog.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "scalesim.h"\n'
                    'int main(){printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(scalesim_config), sizeof(scalesim_tables),'
                    ' sizeof(scalesim_plan_view), sizeof(scalesim_plan_host), offsetof(scalesim_config, page_bytes),'
                    ' offsetof(scalesim_tables, resident_init));}\n')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(prog), "-o", str(exe)])
    got = [int(x) for x in subprocess.check_output([str(exe)]).split()]
    exp = [C.sizeof(L.Config), C.sizeof(L.Tables), C.sizeof(L.PlanView), C.sizeof(L.PlanHost),
           L.Config.page_bytes.offset, L.Tables.resident_init.offset]
    assert got == exp


def _cfg(L, **kw):
    c = L.Config()
    c.abi_version = L.ABI_VERSION
    c.flags = kw.get("flags", 0)
    c.n_agents = kw.get("n", 100)
    c.shard_begin = 0
    c.shard_end = kw.get("shard_end", c.n_agents)
    c.n_kin = kw.get("n_kin", 0)
    c.budget_bytes = 1 << 20
    for k in range(3):
        c.theta[k] = kw.get("theta", 4.0)
    c.hop_scale = kw.get("hop_scale", 1.0)
    c.page_bytes = kw.get("page", 65536)
    c.rank, c.world = kw.get("rank", 0), kw.get("world", 1)
    return c


def test_workspace_bytes_and_validation(L):
    lib = L.lib()
    t = L.Tables()
    t.n_blocks = 100
    t.n_block_pages = 1600
    t.dev_bytes = 64 << 20
    good = lib.scalesim_workspace_bytes(C.byref(_cfg(L)), C.byref(t))
    assert good > 0 and good % 256 == 0
    bigger = lib.scalesim_workspace_bytes(C.byref(_cfg(L, n=10 ** 6)), C.byref(t))
    assert bigger > good
    for bad in (dict(theta=float("nan")), dict(theta=-1.0), dict(hop_scale=0.0), dict(page=1000),
                dict(shard_end=101), dict(world=0), dict(rank=2, world=2), dict(n_kin=5, world=2)):
        assert lib.scalesim_workspace_bytes(C.byref(_cfg(L, **bad)), C.byref(t)) == 0, bad
    ctx = C.c_void_p()
    assert lib.scalesim_init(None, C.byref(t), C.byref(ctx)) == L.E_INVALID
    assert lib.scalesim_init(C.byref(_cfg(L, theta=-2.0)), C.byref(t), C.byref(ctx)) == L.E_INVALID
    assert ctx.value is None
    assert lib.scalesim_score(None, 0, None) == L.E_INVALID
    assert lib.scalesim_plan(None, None) == L.E_INVALID
    assert lib.scalesim_sync(None, None) == L.E_INVALID
    lib.scalesim_destroy(None)
    assert L.strerror(L.E_INSUFFICIENT).startswith("insufficient")


def test_no_oracle_in_product():
    """The product path never imports, includes or links the oracle."""
    pkg = os.path.join(ROOT, "paper_2601_21473_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in txt.lower(), f
    assert "oracle" not in open(os.path.join(ROOT, "include", "scalesim.h")).read().lower()
