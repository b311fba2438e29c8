"""Thin ctypes binding of libtcl.so (include/tcl.h).  Argument marshalling only.

Every step of the scoring path runs in libtcl's CUDA kernels; this module converts torch
tensors / numpy arrays into pointers and status codes into exceptions.  There is no CPU
fallback: if libtcl.so is missing or no CUDA device is present the calls raise.
PyTorch is used only for device memory, streams and (in bench.py) process groups.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TCL_LIB") or os.path.join(HERE, "libtcl.so")  # TCL_LIB: A/B builds only

STATUS = {0: "TCL_OK", -1: "TCL_EINVAL", -2: "TCL_ESHAPE", -3: "TCL_ELEN", -4: "TCL_ECUDA",
          -5: "TCL_ENOMEM", -6: "TCL_ENCCL", -7: "TCL_ESTATE"}
TCL_PREC_FP32, TCL_PREC_BF16_PROJ = 0, 1
TCL_DISC_ZOH, TCL_DISC_EULER_B = 0, 1


class TclError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class tcl_dims(ctypes.Structure):
    _fields_ = [("d_in", ctypes.c_int32), ("max_len", ctypes.c_int32), ("d_model", ctypes.c_int32),
                ("n_layer", ctypes.c_int32), ("d_state", ctypes.c_int32), ("d_conv", ctypes.c_int32),
                ("expand", ctypes.c_int32), ("dt_rank", ctypes.c_int32),
                ("enc_dims", ctypes.c_int32 * 3), ("dec_dims", ctypes.c_int32 * 3),
                ("ln_eps", ctypes.c_float), ("dropout_p", ctypes.c_float),
                ("precision", ctypes.c_int32), ("disc", ctypes.c_int32)]

    @classmethod
    def of(cls, d) -> "tcl_dims":
        return cls(d.d_in, d.max_len, d.d_model, d.n_layer, d.d_state, d.d_conv, d.expand, d.dt_rank,
                   (ctypes.c_int32 * 3)(*d.enc_dims), (ctypes.c_int32 * 3)(*d.dec_dims),
                   d.ln_eps, d.dropout_p, d.precision, d.disc)


EXPORTS = ["tcl_weights_count", "tcl_model_create", "tcl_model_destroy", "tcl_reserve", "tcl_score",
           "tcl_score_mc", "tcl_topk", "tcl_comm_unique_id", "tcl_comm_init", "tcl_topk_global",
           "tcl_score_host", "tcl_sync_error", "tcl_launch_count", "tcl_last_error", "tcl_build_info",
           "tcl_profile_enable", "tcl_profile_read", "tcl_profile_name", "tcl_debug_read", "tcl_rdu_select",
           "tcl_topk_score", "tcl_adapters_count", "tcl_model_create_kbac", "tcl_train_init", "tcl_train_step",
           "tcl_train_read", "tcl_set_option", "tcl_topk_local_keys", "tcl_topk_merge_keys", "tcl_shard_range",
           "tcl_topk_key"]
TCL_OPT_GRAPHS, TCL_OPT_SCAN = 1, 2
SCAN_MODES = {"auto": 0, "sequential": 1, "chunked": 2}
PROF_KINDS = ["pack", "encoder", "layernorm", "in_proj", "conv", "x_proj", "dt_proj", "scan", "out_proj",
              "head", "topk", "mixer", "allgather", "mc", "lateral", "xdt"]

_lib: Optional[ctypes.CDLL] = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libtcl.so (import torch first so its NCCL is the one the library binds to)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: build it with `python -m paper_2604_12891_b200.build` "
                           "(there is no CPU fallback)")
    try:
        import torch  # noqa: F401  (loads libnccl.so.2 / the CUDA driver first)
    except Exception:
        pass
    L = ctypes.CDLL(path)
    P, vp = ctypes.POINTER, ctypes.c_void_p
    i32, i64, u64, sz = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_size_t
    L.tcl_weights_count.restype = sz
    L.tcl_weights_count.argtypes = [P(tcl_dims)]
    L.tcl_model_create.argtypes = [vp, sz, P(tcl_dims), ctypes.c_int, P(vp)]
    L.tcl_model_create_kbac.argtypes = [vp, vp, sz, vp, sz, i32, P(tcl_dims), ctypes.c_int, P(vp)]
    L.tcl_train_init.argtypes = [vp, i64, ctypes.c_float, ctypes.c_float, ctypes.c_float, ctypes.c_float,
                                 ctypes.c_float]
    L.tcl_train_step.argtypes = [vp, vp, vp, i64, vp, vp, i64, i32, i32, vp, vp]
    L.tcl_train_read.argtypes = [vp, i32, vp, i64]
    L.tcl_adapters_count.restype = sz
    L.tcl_adapters_count.argtypes = [P(tcl_dims), i32]
    L.tcl_model_destroy.argtypes = [vp]
    L.tcl_reserve.argtypes = [vp, i64, i32]
    L.tcl_score.argtypes = [vp, vp, vp, i64, vp, vp]
    L.tcl_score_mc.argtypes = [vp, vp, vp, i64, i32, u64, i64, vp, vp, vp]
    L.tcl_topk.argtypes = [vp, vp, i64, i32, i64, vp, vp, vp]
    L.tcl_comm_unique_id.argtypes = [vp]
    L.tcl_comm_init.argtypes = [vp, vp, i32, i32]
    L.tcl_topk_global.argtypes = [vp, vp, i64, i64, i32, vp, vp, vp]
    L.tcl_score_host.argtypes = [vp, vp, vp, i64, i64, vp, i32, vp, vp, vp]
    L.tcl_sync_error.argtypes = [vp, vp]
    L.tcl_launch_count.restype = i64
    L.tcl_launch_count.argtypes = [vp]
    L.tcl_last_error.restype = ctypes.c_char_p
    L.tcl_last_error.argtypes = []
    L.tcl_build_info.restype = ctypes.c_char_p
    L.tcl_build_info.argtypes = []
    L.tcl_profile_enable.argtypes = [vp, ctypes.c_int]
    L.tcl_profile_read.argtypes = [vp, P(ctypes.c_double), P(i64), ctypes.c_int]
    L.tcl_debug_read.argtypes = [vp, ctypes.c_char_p, vp, i64, i64]
    L.tcl_rdu_select.argtypes = [vp, vp, vp, i64, vp, i64, i32, i32, vp, vp, vp]
    L.tcl_topk_score.argtypes = [vp, vp, vp, vp, vp, i64, i32, vp, i32, vp, vp]
    L.tcl_set_option.argtypes = [vp, i32, i64]
    L.tcl_topk_local_keys.argtypes = [vp, vp, i64, i64, i32, vp, vp]
    L.tcl_topk_merge_keys.argtypes = [vp, vp, i64, i32, vp, vp, vp]
    L.tcl_shard_range.argtypes = [i64, i32, i32, P(i64), P(i64)]
    L.tcl_topk_key.restype = u64
    L.tcl_topk_key.argtypes = [ctypes.c_float, i64]
    L.tcl_profile_name.restype = ctypes.c_char_p
    L.tcl_profile_name.argtypes = [ctypes.c_int]
    for fn in ("tcl_model_create", "tcl_model_destroy", "tcl_reserve", "tcl_score", "tcl_score_mc",
               "tcl_topk", "tcl_comm_unique_id", "tcl_comm_init", "tcl_topk_global",
               "tcl_score_host", "tcl_sync_error", "tcl_profile_enable", "tcl_profile_read", "tcl_debug_read", "tcl_rdu_select",
               "tcl_topk_score", "tcl_model_create_kbac", "tcl_train_init", "tcl_train_step", "tcl_train_read",
               "tcl_set_option", "tcl_topk_local_keys", "tcl_topk_merge_keys", "tcl_shard_range"):
        getattr(L, fn).restype = ctypes.c_int
    _lib = L
    return L


def _check(code: int):
    if code != 0:
        raise TclError(code, load().tcl_last_error().decode())


def _ptr(t) -> int:
    """Device/host address of a torch tensor or numpy array (no copy, must be contiguous)."""
    if isinstance(t, np.ndarray):
        if not t.flags["C_CONTIGUOUS"]:
            raise TclError(-1, "array must be C-contiguous")
        return t.ctypes.data
    if not t.is_contiguous():
        raise TclError(-1, "tensor must be contiguous")
    return t.data_ptr()


_NP = {"f32": np.float32, "f64": np.float64, "i32": np.int32, "i64": np.int64}


def _arg(t, kind: str, count: int, name: str, device: bool = True) -> int:
    """Validated pointer of argument `name`: dtype `kind`, >= `count` elements, contiguous, on a
    CUDA device (device=True: a torch CUDA tensor) or in host memory (device=False: a numpy array
    or a CPU tensor).  Raises TclError(TCL_EINVAL) instead of passing a bad pointer to the C ABI."""
    if t is None:
        raise TclError(-1, f"{name} is None")
    if isinstance(t, np.ndarray):
        if device:
            raise TclError(-1, f"{name}: a CUDA tensor is required, got a numpy array")
        dt, size = t.dtype, t.size
        ok = dt == np.dtype(_NP[kind])
    else:
        if bool(t.is_cuda) != device:
            raise TclError(-1, f"{name}: expected a {'CUDA' if device else 'host'} tensor")
        dt, size = t.dtype, t.numel()
        ok = str(dt) == "torch." + {"f32": "float32", "f64": "float64", "i32": "int32", "i64": "int64"}[kind]
    if not ok:
        raise TclError(-1, f"{name}: dtype {dt} where {np.dtype(_NP[kind])} is required")
    if size < count:
        raise TclError(-1, f"{name}: {size} elements where {count} are required")
    return _ptr(t)


def _stream(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def shard_range(n_global: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous candidate shard of `rank` (libtcl's tcl_shard_range): [start,
    start + count), start = rank * ceil(n / world); global index of local candidate i = start + i."""
    st, cnt = ctypes.c_int64(), ctypes.c_int64()
    _check(load().tcl_shard_range(n_global, world, rank, ctypes.byref(st), ctypes.byref(cnt)))
    return st.value, cnt.value


def topk_key(score: float, global_index: int) -> int:
    """The packed (score desc, index asc) key of the device top-k (libtcl's tcl_topk_key)."""
    return int(load().tcl_topk_key(score, global_index))


def tcl_weights_count(dims) -> int:
    return int(load().tcl_weights_count(ctypes.byref(tcl_dims.of(dims))))


def tcl_comm_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(load().tcl_comm_unique_id(buf))
    return bytes(buf)


class Model:
    """Owns one tcl_model handle (weights on one device + workspace)."""

    def __init__(self, weights: np.ndarray, dims, device: int = 0):
        w = np.ascontiguousarray(weights, dtype=np.float32)
        self.dims = dims
        self.device = device
        h = ctypes.c_void_p()
        _check(load().tcl_model_create(w.ctypes.data, w.size, ctypes.byref(tcl_dims.of(dims)), device,
                                       ctypes.byref(h)))
        self._h = h

    @classmethod
    def kbac(cls, kb_weights: np.ndarray, ac_weights: np.ndarray, adapters: np.ndarray, adapter_rank: int, dims,
             device: int = 0) -> "Model":
        """KB + AC two-column model (Eq. 7 lateral adapters); scores are the AC column's output."""
        kb = np.ascontiguousarray(kb_weights, dtype=np.float32)
        ac = np.ascontiguousarray(ac_weights, dtype=np.float32)
        ad = np.ascontiguousarray(adapters, dtype=np.float32)
        if kb.size != ac.size:
            raise ValueError("KB and AC weight blobs differ in size")
        self = cls.__new__(cls)
        self.dims = dims
        self.device = device
        h = ctypes.c_void_p()
        _check(load().tcl_model_create_kbac(kb.ctypes.data, ac.ctypes.data, ac.size, ad.ctypes.data, ad.size,
                                            adapter_rank, ctypes.byref(tcl_dims.of(dims)), device, ctypes.byref(h)))
        self._h = h
        return self

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            load().tcl_model_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def set_option(self, option: int, value: int):
        _check(load().tcl_set_option(self._h, option, value))

    def use_graphs(self, on: bool = True):
        """CUDA-graph replay of repeated calls (TCL_OPT_GRAPHS, default on)."""
        self.set_option(TCL_OPT_GRAPHS, 1 if on else 0)

    def scan_mode(self, mode: str):
        """fp32 path recurrence: "auto" (by dims), "sequential", or "chunked" (warp-shuffle across L)."""
        self.set_option(TCL_OPT_SCAN, SCAN_MODES[mode])

    def reserve(self, n_max: int, mc_passes_max: int = 0):
        _check(load().tcl_reserve(self._h, n_max, mc_passes_max))

    # -- device-buffer calls (torch CUDA tensors) --------------------------------------------
    def _feats(self, feats, lens, device=True):
        n = lens.shape[0]
        row = self.dims.max_len * self.dims.d_in
        return n, _arg(feats, "f32", n * row, "feats", device), _arg(lens, "i32", n, "lens", device)

    def tcl_score(self, feats, lens, scores, stream=None):
        n, pf, pl = self._feats(feats, lens)
        _check(load().tcl_score(self._h, pf, pl, n, _arg(scores, "f32", n, "scores"), _stream(stream)))

    def tcl_score_mc(self, feats, lens, n_passes: int, seed: int, index_base: int, mean, var, stream=None):
        n, pf, pl = self._feats(feats, lens)
        _check(load().tcl_score_mc(self._h, pf, pl, n, n_passes, seed, index_base,
                                   _arg(mean, "f32", n, "mean"), _arg(var, "f32", n, "var"), _stream(stream)))

    def tcl_topk(self, scores, k: int, index_base: int, idx, top, n: Optional[int] = None, stream=None):
        n = scores.shape[0] if n is None else n
        _check(load().tcl_topk(self._h, _arg(scores, "f32", n, "scores"), n, k, index_base,
                               _arg(idx, "i64", k, "idx"), _arg(top, "f32", k, "top"), _stream(stream)))

    def tcl_comm_init(self, uid: bytes, nranks: int, rank: int):
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        _check(load().tcl_comm_init(self._h, buf, nranks, rank))

    def tcl_topk_global(self, scores, index_base: int, k: int, idx, top, stream=None):
        n = scores.shape[0]
        _check(load().tcl_topk_global(self._h, _arg(scores, "f32", n, "scores"), n, index_base, k,
                                      _arg(idx, "i64", k, "idx"), _arg(top, "f32", k, "top"), _stream(stream)))

    def tcl_topk_local_keys(self, scores, index_base: int, k: int, keys, stream=None):
        """This shard's best k as packed uint64 keys (device int64 tensor [k]), sorted descending."""
        n = scores.shape[0]
        _check(load().tcl_topk_local_keys(self._h, _arg(scores, "f32", n, "scores") if n else None, n, index_base, k,
                                          _arg(keys, "i64", k, "keys"), _stream(stream)))

    def tcl_topk_merge_keys(self, keys, k: int, idx, top, stream=None):
        """Best k of gathered packed keys (device int64 tensor) -> (idx, score) [k]."""
        cnt = keys.shape[0]
        _check(load().tcl_topk_merge_keys(self._h, _arg(keys, "i64", cnt, "keys"), cnt, k, _arg(idx, "i64", k, "idx"),
                                          _arg(top, "f32", k, "top"), _stream(stream)))

    def tcl_topk_score(self, scores, latency, task_offsets, task_weights, max_task_len: int, ks, result,
                       stream=None):
        """Eq. 12 Top-k score over CSR tasks (device tensors); result [3*len(ks)] fp64 = score|num|den."""
        kk = np.ascontiguousarray(ks, dtype=np.int32)
        nt = task_offsets.shape[0] - 1
        n = scores.shape[0]
        _check(load().tcl_topk_score(self._h, _arg(scores, "f32", n, "scores"), _arg(latency, "f32", n, "latency"),
                                     _arg(task_offsets, "i64", nt + 1, "task_offsets"),
                                     _arg(task_weights, "f32", nt, "task_weights"), nt, max_task_len,
                                     kk.ctypes.data, kk.size, _arg(result, "f64", 3 * kk.size, "result"),
                                     _stream(stream)))

    # -- training (fp32 models) ------------------------------------------------------------------
    def tcl_train_init(self, n_max: int, lr: float = 7e-4, beta1: float = 0.9, beta2: float = 0.999,
                       eps: float = 1e-8, sigma_rank: float = 1.0):
        _check(load().tcl_train_init(self._h, n_max, lr, beta1, beta2, eps, sigma_rank))

    def tcl_train_step(self, feats, lens, latency, group_offsets, max_group: int, apply_update: bool = True,
                       loss=None, stream=None):
        """One LambdaRank + Adam step on device tensors; loss (fp32 [1] device tensor) optional."""
        n, pf, pl = self._feats(feats, lens)
        ng = group_offsets.shape[0] - 1
        _check(load().tcl_train_step(self._h, pf, pl, n, _arg(latency, "f32", n, "latency"),
                                     _arg(group_offsets, "i64", ng + 1, "group_offsets"), ng, max_group,
                                     1 if apply_update else 0, _arg(loss, "f32", 1, "loss") if loss is not None else None,
                                     _stream(stream)))

    def tcl_train_read(self, what: str, count: int) -> np.ndarray:
        code = {"weights": 0, "grads": 1, "dscores": 2, "scores": 3}[what]
        out = np.empty(count, np.float32)
        _check(load().tcl_train_read(self._h, code, out.ctypes.data, count))
        return out

    def tcl_rdu_select(self, pool_scores, pool_ops, labeled_scores, n_ops: int, budget_total: int,
                       selected, n_selected, stream=None):
        """RDU acquisition round (Alg. 1 lines 16-31): device tensors in, picks in `selected`."""
        n, nl = pool_scores.shape[0], labeled_scores.shape[0]
        _check(load().tcl_rdu_select(self._h, _arg(pool_scores, "f32", n, "pool_scores"),
                                     _arg(pool_ops, "i32", n, "pool_ops"),
                                     n, _arg(labeled_scores, "f32", nl, "labeled_scores") if nl else None,
                                     nl, n_ops, budget_total, _arg(selected, "i64", budget_total, "selected"),
                                     _arg(n_selected, "i32", 1, "n_selected"), _stream(stream)))

    def tcl_sync_error(self, stream=None):
        _check(load().tcl_sync_error(self._h, _stream(stream)))

    def launch_count(self) -> int:
        return int(load().tcl_launch_count(self._h))

    def debug_read(self, name: str, rows: int, cols: int) -> np.ndarray:
        out = np.empty((rows, cols), np.float32)
        _check(load().tcl_debug_read(self._h, name.encode(), out.ctypes.data, rows, cols))
        return out

    def profile_enable(self, on: bool = True):
        _check(load().tcl_profile_enable(self._h, 1 if on else 0))

    def profile_read(self, reset: bool = True) -> dict:
        """{stage: (total_ms, launches)} accumulated since the last reset (synchronises)."""
        n = len(PROF_KINDS)
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_int64 * n)()
        _check(load().tcl_profile_read(self._h, ms, cnt, 1 if reset else 0))
        return {load().tcl_profile_name(i).decode(): (ms[i], cnt[i]) for i in range(n) if cnt[i] > 0}

    # -- host-buffer call (end to end) -----------------------------------------------------------
    def tcl_score_host(self, feats: np.ndarray, lens: np.ndarray, k: int = 0, index_base: int = 0,
                       scores: np.ndarray = None, idx: np.ndarray = None, top: np.ndarray = None,
                       stream=None) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        n, pf, pl = self._feats(feats, lens, device=False)
        scores = np.empty(n, np.float32) if scores is None else scores
        idx = np.empty(max(k, 1), np.int64) if idx is None else idx
        top = np.empty(max(k, 1), np.float32) if top is None else top
        _check(load().tcl_score_host(self._h, pf, pl, n, index_base, _arg(scores, "f32", n, "scores", False), k,
                                     _arg(idx, "i64", k, "idx", False), _arg(top, "f32", k, "top", False),
                                     _stream(stream)))
        return scores, idx[:k], top[:k]
