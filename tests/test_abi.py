"""CPU-side checks of the C-ABI library: it builds, loads, exports every symbol include/tcl.h
declares, and its host-only logic (dims validation, weight counts, error reporting) is right.
No compute call is made here (no GPU in this container)."""
import ctypes
import os
import re

import numpy as np
import pytest

import inputs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2604_12891_b200 import build, tcl
    build.build()
    return tcl.load()


def _declared():
    src = open(os.path.join(ROOT, "include", "tcl.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tcl_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    names = _declared()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n
    from paper_2604_12891_b200 import tcl
    assert sorted(tcl.EXPORTS) == names


def test_built_for_sm100a_only():
    import subprocess
    from paper_2604_12891_b200 import tcl
    out = subprocess.run(["cuobjdump", "--list-elf", tcl.LIB_PATH], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


@pytest.mark.parametrize("name", list(inputs.CONFIGS))
def test_weights_count_matches_blob_layout(lib, name):
    from paper_2604_12891_b200 import tcl
    d = inputs.config(name)["dims"]
    assert tcl.tcl_weights_count(d) == inputs.weights_count(d)


@pytest.mark.parametrize("bad", [dict(d_model=48), dict(d_state=32), dict(enc_dims=(32, 64, 32)),
                                 dict(dec_dims=(32, 16, 2)), dict(max_len=0), dict(d_in=40),
                                 dict(dt_rank=6), dict(precision=7), dict(disc=3)])
def test_dims_validation(lib, bad):
    from paper_2604_12891_b200 import tcl
    d = inputs.config("tiny")["dims"].replace(**bad)
    assert tcl.tcl_weights_count(d) == 0
    assert len(lib.tcl_last_error()) > 0


def test_create_rejects_bad_args_before_touching_cuda(lib):
    from paper_2604_12891_b200 import tcl
    d = inputs.config("tiny")["dims"]
    w = np.zeros(inputs.weights_count(d) - 1, np.float32)
    h = ctypes.c_void_p()
    rc = lib.tcl_model_create(w.ctypes.data, w.size, ctypes.byref(tcl.tcl_dims.of(d)), 0, ctypes.byref(h))
    assert rc == -2 and h.value is None          # TCL_ESHAPE: wrong blob size
    rc = lib.tcl_model_create(None, 10, ctypes.byref(tcl.tcl_dims.of(d)), 0, ctypes.byref(h))
    assert rc == -1                               # TCL_EINVAL: null weights
    with pytest.raises(tcl.TclError):
        tcl.Model(np.zeros(3, np.float32), d)
    # null-model calls are rejected on the host
    assert lib.tcl_score(None, None, None, 0, None, None) == -1
    assert lib.tcl_topk(None, None, 0, 1, 0, None, None, None) == -1
    assert lib.tcl_launch_count(None) == 0


def test_no_gpu_means_loud_failure(lib):
    """Without a CUDA device the product path fails loudly (no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2604_12891_b200 import tcl
    d = inputs.config("tiny")["dims"]
    w = inputs.make_weights(d, 1)
    with pytest.raises(tcl.TclError) as e:
        tcl.Model(w, d)
    assert e.value.code == -4                    # TCL_ECUDA


def test_product_never_imports_oracle():
    """The CUDA path and the oracle share no code (③)."""
    pkg = os.path.join(ROOT, "paper_2604_12891_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", txt).lower() or f == "build.py", f
