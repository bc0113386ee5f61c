"""The C-ABI library loads and exports every symbol include/pw_b200.h declares
(no compute calls: runs without a GPU)."""

import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared_functions():
    text = (ROOT / "include" / "pw_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w]+\s*\*?\s*(pw_\w+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    names = declared_functions()
    for must in ("pw_shard_create", "pw_search_one", "pw_search_stage", "pw_run", "pw_reduce_topk"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2507_17094_b200 import _abi

    assert _abi.LIB_PATH.exists(), "libpwb200.so not built (run __graft_entry__.build())"
    lib = ctypes.CDLL(str(_abi.LIB_PATH))
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert set(declared_functions()) == set(_abi.EXPORTS)


def test_version_string():
    from paper_2507_17094_b200 import _abi

    lib = _abi.load(require_device=False)
    assert b"sm_100a" in lib.pw_version()


def test_sass_is_sm100a():
    import shutil
    import subprocess

    from paper_2507_17094_b200 import _abi

    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump not on PATH")
    out = subprocess.run(["cuobjdump", "--list-elf", str(_abi.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("device present")
    import numpy as np

    import paper_2507_17094_b200 as pw
    from paper_2507_17094_b200.rng import stream

    ctx = pw.ShardContext(vectors=np.zeros((4, 2), np.float32), adj=np.zeros((4, 1), np.int32),
                          global_ids=np.arange(4, dtype=np.int32))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        pw.search(np.zeros(2, np.float32), ctx, pw.SearchParams(k=1, l=4, m=4, r=1), rng=stream(0, 4, 0, 0))


def test_no_fused_multiply_add_in_distance_code():
    """Bit-exact L2 (numpy pairwise order, separately rounded sub/mul/add):
    ptxas contracts packed mul.rn.f32x2 + add.rn.f32x2 into FFMA2, so the
    kernels must contain no FFMA2 at all (and FMUL2 feeds scalar FADDs)."""
    import shutil
    import subprocess

    from paper_2507_17094_b200 import _abi

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(tool).exists():
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([tool, "-sass", str(_abi.LIB_PATH)], capture_output=True, text=True).stdout
    assert "beam_search_kernel" in sass
    assert "FFMA2" not in sass


def test_no_odd_uniform_memory_descriptors():
    """Memory descriptors are 64-bit uniform register pairs.  ptxas 12.9 once
    emitted `LDGSTS ... desc[UR1]` for the uint8-row K1 instances with an L2
    cache-hint copy, which faults at run time as an illegal instruction; the
    library must contain no odd descriptor register."""
    import shutil
    import subprocess

    from paper_2507_17094_b200 import _abi

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(tool).exists():
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([tool, "-sass", str(_abi.LIB_PATH)], capture_output=True, text=True).stdout
    # memory descriptors only (`desc[URn]`); tcgen05's instruction / matrix
    # descriptors (`idesc[..]`, `gdesc[..]`) are other operand kinds
    odd = sorted(set(re.findall(r"(?<![a-z])desc\[UR\d*[13579]\]", sass)))
    assert not odd, odd


def test_result_block_layout():
    """_abi.result_block follows include/pw_b200.h's result block: the six
    arrays in order, each at the previous start + its size rounded up to 256
    bytes, with the documented shapes and dtypes."""
    import numpy as np

    from paper_2507_17094_b200 import _abi
    for q, n, k in ((10000, 1, 10), (1537, 3, 16), (1, 2, 100)):
        b = _abi.result_block(q, n, k)
        names = ("shard_ids", "shard_dists", "final_ids", "final_dists", "s32", "s64")
        shapes = ((q, n, k), (q, n, k), (q, k), (q, k), (n, 4, q), (n, 6, q))
        dts = (np.int32, np.float32, np.int32, np.float32, np.int32, np.int64)
        addr = b["shard_ids"].ctypes.data
        for name, shape, dt in zip(names, shapes, dts):
            a = b[name]
            assert a.shape == shape and a.dtype == dt and a.flags.c_contiguous, name
            assert a.ctypes.data == addr, name
            addr += (a.nbytes + 255) // 256 * 256
