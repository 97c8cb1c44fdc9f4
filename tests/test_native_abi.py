"""The C-ABI library loads without a GPU and exports every function that
include/hm_page.h declares; the ctypes table covers exactly that set."""
import ctypes
import ctypes as C
import re
from pathlib import Path

from conftest import ROOT
from paper_2303_02868_b200 import _native as N


def declared_functions():
    text = (ROOT / "include" / "hm_page.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = set(re.findall(r"\b(hm_[a-z0-9_]+)\s*\(", text))
    return names


def test_library_exports_header():
    lib = ctypes.CDLL(str(N.LIB_PATH))
    names = declared_functions()
    assert len(names) >= 20
    for name in sorted(names):
        assert hasattr(lib, name), f"{name} declared in include/hm_page.h but not exported"
    assert names == set(N.SIGNATURES), names ^ set(N.SIGNATURES)


def test_abi_constants():
    lib = N.lib()
    assert lib.hm_abi_version() == 2
    assert lib.hm_device_chunk_elems() == 4096


def test_struct_layouts_match_header():
    text = (ROOT / "include" / "hm_page.h").read_text()
    assert "#define HM_ADAM_CHUNK 4096" in text
    assert N.ADAM_CHUNK.names == ("g_off", "s_off", "p_off", "n", "slot")
    assert N.GROUP_LAUNCH.names == ("g_shift", "p_shift", "group", "flag")
    assert N.SEG_CHUNK.names == ("src_off", "dst_off", "n", "slot")
    assert ctypes.sizeof(N.AdamHyperC) == 32
    assert ctypes.sizeof(N.LaunchOpts) == 24 and "typedef struct hm_launch_opts" in text


def test_kernels_do_not_spill():
    """Every data-path kernel in the library keeps its working set in
    registers: no local memory / stack (a spill or a runtime-indexed peer
    table turns into extra HBM traffic — it once cost the update+AG kernel
    2 GB per step)."""
    import shutil
    import subprocess
    import pytest
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    lib = ROOT / "paper_2303_02868_b200" / "libhm_page.so"
    if not lib.exists() or not Path(tool).exists():
        pytest.skip("needs the built library and cuobjdump")
    out = subprocess.run([tool, "-res-usage", str(lib)], capture_output=True, text=True, check=True).stdout
    funcs = re.findall(r"Function (\S+):\s*\n\s*REG:(\d+) STACK:(\d+) SHARED:\d+ LOCAL:(\d+)", out)
    assert len(funcs) > 20
    bad = [(f, stack, local) for f, _, stack, local in funcs if int(stack) or int(local)]
    assert not bad, bad


def test_null_pointers_rejected_before_launch():
    """Argument validation happens on the host, before any CUDA call, so it
    runs here without a GPU: a null buffer with work to do is HM_ERR_INVALID
    (never a kernel fault), and an empty launch is a no-op."""
    lib = N.lib()
    INVALID = 7
    acc = lambda *a: lib.hm_accumulate(*a, None, None, None, None)
    assert acc(None, 2, None, 2, None, 1, 0, None, None, None) == INVALID
    assert b"null pointer" in lib.hm_last_error()
    assert lib.hm_cast(None, 3, None, 2, None, 5, None) == INVALID
    assert lib.hm_reduce_stats(None, 2, None, 3, None, None, None, None) == INVALID
    assert lib.hm_copy_runs(None, None, None, 2, None) == INVALID
    assert acc(None, 2, None, 2, None, 0, 0, None, None, None) == 0
    assert lib.hm_cast(None, 3, None, 2, None, 0, None) == 0
    assert acc(None, 9, None, 2, None, 1, 0, None, None, None) == INVALID
    assert lib.hm_stats_take(None, 3, None, None, None, None, None) == INVALID
    assert lib.hm_stats_take(None, 0, None, None, None, None, None) == 0
    # a ledger delta row without the running sums it telescopes against
    assert lib.hm_accumulate(None, 2, None, 2, None, 1, 0, None, None, None, None, C.c_void_p(8),
                             None, None) == INVALID
    assert lib.hm_set_dp_reduce_ctas(-1) == INVALID and lib.hm_set_dp_reduce_ctas(0) == 0
    assert lib.hm_set_ag_publish(3) == INVALID and lib.hm_set_ag_publish(0) == 0
    assert lib.hm_set_adam_threads(300) == INVALID
    # per-launch options are validated like the process defaults
    hc = N.AdamHyperC(0.01, 0.9, 0.1, 0.999, 0.001, 1e-8, 1.0, 0.0)
    assert lib.hm_adam_main(None, 1, None, C.c_void_p(8), None, 2, None, None, None, None, 0, C.byref(hc),
                            C.byref(N.LaunchOpts(adam_threads=300)), None) == INVALID
    assert lib.hm_adam_main(None, 1, None, C.c_void_p(8), None, 2, None, None, None, None, 0, C.byref(hc),
                            C.byref(N.LaunchOpts(adam_variant=5)), None) == INVALID


def test_cpulist_parser():
    from paper_2303_02868_b200._device import _parse_cpulist
    assert _parse_cpulist("0-3,8,10-11\n") == {0, 1, 2, 3, 8, 10, 11}
    assert _parse_cpulist("") == set()


def test_ctypes_arity_matches_header():
    """Every prototype's parameter count equals the ctypes argtypes length (a
    missing argument would shift every later one at the call site)."""
    text = re.sub(r"/\*.*?\*/", "", (ROOT / "include" / "hm_page.h").read_text(), flags=re.S)
    protos = re.findall(r"\b(?:int|int64_t|const char\s*\*|void|uint32_t)\s+\**\s*(hm_[a-z0-9_]+)\s*\(([^;{]*?)\)\s*;",
                        text, flags=re.S)
    assert {p[0] for p in protos} == declared_functions()
    for name, params in protos:
        params = params.strip()
        n = 0 if params in ("", "void") else params.count(",") + 1
        assert n == len(N.SIGNATURES[name][1]), f"{name}: header {n} params, ctypes {len(N.SIGNATURES[name][1])}"


def test_package_exports_resolve():
    """Every name the package re-exports resolves (the reference's names for
    the path plus the build's own entry points); importing needs no GPU."""
    import paper_2303_02868_b200 as P
    for name in P._LAZY:
        assert getattr(P, name) is not None, name
    for name in ("PageManager", "TierPool", "pool_init", "TensorSpec", "ConfigError"):
        assert hasattr(P, name)
