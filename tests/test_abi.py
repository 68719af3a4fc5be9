"""CPU: the C-ABI library loads, exports exactly what include/cdx_c.h declares, and the
Python binding table matches; without a GPU every compute entry fails loudly."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "cdx_c.h")


def declared():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cdx_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2412_20993_b200 import _abi
    if not os.path.exists(_abi.LIB_PATH):
        subprocess.run(["make", "-C", ROOT, "-j8", "lib"], check=True)
    return _abi.load()


def test_library_exports_every_declared_symbol(lib):
    from paper_2412_20993_b200 import _abi
    out = subprocess.run(["nm", "-D", "--defined-only", _abi.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (cdx_[a-z0-9_]+)$", out, flags=re.M))
    missing = [s for s in declared() if s not in exported]
    assert not missing, f"declared in cdx_c.h but not exported: {missing}"


def test_binding_table_covers_header():
    from paper_2412_20993_b200 import _abi
    assert sorted(_abi.SIGNATURES) == declared()


def test_abi_version(lib):
    assert lib.cdx_abi_version() == 4


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2412_20993_b200 import CdxCudaError, Context
    with pytest.raises(CdxCudaError):
        Context(0)


def test_struct_layouts_match_header():
    """Compile a tiny C program against cdx_c.h and compare sizeof/offsetof with ctypes."""
    import ctypes as C

    from paper_2412_20993_b200 import _abi
    prog = r"""
#include <stdio.h>
#include <stddef.h>
#include "cdx_c.h"
int main(void){
 printf("%zu %zu %zu %zu %zu %zu\n", sizeof(cdx_threshold), sizeof(cdx_alloc_policy), sizeof(cdx_probe_cfg),
        sizeof(cdx_inter_policy), sizeof(cdx_prog_soa), sizeof(cdx_gen_params));
 printf("%zu %zu %zu %zu\n", offsetof(cdx_alloc_policy, tokens_per_unit), offsetof(cdx_gen_params, noise_level),
        offsetof(cdx_gen_params, reward_jitter_k), offsetof(cdx_prog_soa, id_base));
 return 0; }
"""
    import tempfile
    d = tempfile.mkdtemp()
    with open(os.path.join(d, "t.c"), "w") as f:
        f.write(prog)
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-o", os.path.join(d, "t"), os.path.join(d, "t.c")],
                   check=True)
    out = subprocess.run([os.path.join(d, "t")], capture_output=True, text=True).stdout.split()
    sizes = [C.sizeof(t) for t in (_abi.Threshold, _abi.AllocPolicy, _abi.ProbeCfg, _abi.InterPolicy, _abi.ProgSoA,
                                   _abi.GenParams)]
    offs = [_abi.AllocPolicy.tokens_per_unit.offset, _abi.GenParams.noise_level.offset,
            _abi.GenParams.reward_jitter_k.offset, _abi.ProgSoA.id_base.offset]
    assert [int(x) for x in out] == sizes + offs
