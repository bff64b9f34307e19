"""paper_2605_06057_b200 -- thin Python binding of liblcma.so (include/lcma.h).

Argument marshalling only: every step of C = A*B (Combine A/B, the tcgen05
sub-GEMMs, Combine H) runs in the CUDA kernels behind the C ABI.  There is no
CPU or PyTorch fallback -- if the extension is missing, import fails loudly.
PyTorch is used for device memory and streams only.
"""
from __future__ import annotations

import ctypes
import os

__all__ = ["lib", "Plan", "decide", "scheme_get", "scheme_register_file", "scheme_register",
           "LcmaError", "BF16", "FP16", "TF32", "FP32", "FP8", "ALGO", "VARIANT"]

_HERE = os.path.dirname(os.path.abspath(__file__))
# LCMA_LIB: an alternative build of the same library (tuning experiments)
_LIB_PATH = os.environ.get("LCMA_LIB") or os.path.join(_HERE, "liblcma.so")

BF16, FP16, TF32, FP32, FP8 = 0, 1, 2, 3, 4   # FP8: bf16 in, E4M3 1x128-scaled MMA
ALGO = {"auto": 0, "classical": 1, "strassen": 2, "strassen2": 3, "laderman": 4, "scheme": 5}
VARIANT = {"auto": 0, "unfused": 1, "fused_h": 2, "producer": 3, "two_level": 4}
STATUS = {0: "LCMA_OK", 1: "LCMA_ERR_INVALID_VALUE", 2: "LCMA_ERR_NOT_SUPPORTED",
          3: "LCMA_ERR_MISALIGNED", 4: "LCMA_ERR_SCHEME_INVALID", 5: "LCMA_ERR_COEFF_RANGE",
          6: "LCMA_ERR_PARSE", 7: "LCMA_ERR_WORKSPACE", 8: "LCMA_ERR_CUDA"}


class LcmaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class HwProfile(ctypes.Structure):
    _fields_ = [("flops_mul", ctypes.c_double), ("flops_add", ctypes.c_double),
                ("beta_elems", ctypes.c_double), ("workers", ctypes.c_int32)]


class PlanDesc(ctypes.Structure):
    _fields_ = [("M", ctypes.c_int64), ("N", ctypes.c_int64), ("K", ctypes.c_int64),
                ("dtype", ctypes.c_int), ("out_dtype", ctypes.c_int), ("algo", ctypes.c_int),
                ("scheme_id", ctypes.c_int32), ("b_layout", ctypes.c_int32),
                ("b_static", ctypes.c_int32), ("variant", ctypes.c_int32),
                ("schedule", ctypes.c_int32), ("num_ctas", ctypes.c_int32),
                ("hw", ctypes.POINTER(HwProfile)), ("decision_model", ctypes.c_int32),
                ("raster_rows", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("algo", ctypes.c_int), ("variant", ctypes.c_int32),
                ("m", ctypes.c_int32), ("k", ctypes.c_int32), ("n", ctypes.c_int32),
                ("R", ctypes.c_int32), ("depth", ctypes.c_int32), ("scheme", ctypes.c_char * 64),
                ("Mb", ctypes.c_int64), ("Nb", ctypes.c_int64), ("Kb", ctypes.c_int64),
                ("BM", ctypes.c_int32), ("BN", ctypes.c_int32), ("BK", ctypes.c_int32),
                ("cta_group", ctypes.c_int32), ("groups", ctypes.c_int32), ("tiles", ctypes.c_int32), ("ctas", ctypes.c_int32),
                ("waves", ctypes.c_int32), ("group_waves", ctypes.c_int32),
                ("split_groups", ctypes.c_int32),
                ("t_pred_classical", ctypes.c_double), ("t_pred_choice", ctypes.c_double),
                ("speedup_pred", ctypes.c_double), ("memory_bound", ctypes.c_int32),
                ("lcma_condition", ctypes.c_int32), ("fused_condition", ctypes.c_int32),
                ("workspace_bytes", ctypes.c_size_t), ("btilde_bytes", ctypes.c_size_t),
                ("partial_slots", ctypes.c_int32)]

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_}
        d["scheme"] = self.scheme.decode()
        return d


_lib = None


def lib():
    """Load liblcma.so (built in-tree by build.py / __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} missing: run `python -m paper_2605_06057_b200.build` "
                          "(no CPU fallback exists)")
    L = ctypes.CDLL(_LIB_PATH)
    P, I32, I64, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    plan_p = ctypes.POINTER(ctypes.c_void_p)
    L.lcma_plan.argtypes = [I64, I64, I64, ctypes.c_int, ctypes.c_int, plan_p]
    L.lcma_plan_ex.argtypes = [ctypes.POINTER(PlanDesc), plan_p]
    L.lcma_free.argtypes = [P]
    L.lcma_free.restype = None
    L.lcma_plan_get_info.argtypes = [P, ctypes.POINTER(PlanInfo)]
    L.lcma_workspace_size.argtypes = [P, ctypes.POINTER(SZ)]
    L.lcma_btilde_size.argtypes = [P, ctypes.POINTER(SZ)]
    L.lcma_workspace_region.argtypes = [P, ctypes.c_int32, ctypes.POINTER(SZ)]
    L.lcma_gemm.argtypes = [P, P, P, P, P, SZ, P]
    L.lcma_precombine_b.argtypes = [P, P, P, P]
    L.lcma_gemm_precombined.argtypes = [P, P, P, P, P, SZ, P]
    L.lcma_decide.argtypes = [I64, I64, I64, ctypes.c_int, ctypes.POINTER(HwProfile), I32,
                              ctypes.POINTER(PlanInfo)]
    L.lcma_scheme_register_file.argtypes = [ctypes.c_char_p, ctypes.POINTER(I32)]
    L.lcma_scheme_register.argtypes = [I32, I32, I32, I32, P, P, P, ctypes.c_char_p,
                                       ctypes.POINTER(I32)]
    L.lcma_scheme_get.argtypes = [I32, ctypes.POINTER(I32), P, P, P]
    L.lcma_plan_schedule.argtypes = [P, I32, ctypes.POINTER(I32), I32, ctypes.POINTER(I32)]
    L.lcma_last_error.restype = ctypes.c_char_p
    L.lcma_last_error.argtypes = []
    L.lcma_last_launch_count.restype = I32
    L.lcma_last_launch_count.argtypes = []
    L.lcma_set_kernel_events.argtypes = [P, P]
    L.lcma_set_kernel_events.restype = None
    L.lcma_debug_stats.argtypes = [P, ctypes.c_int]
    L.lcma_debug_stats.restype = ctypes.c_int
    for name in ("lcma_plan", "lcma_plan_ex", "lcma_plan_get_info", "lcma_workspace_size",
                 "lcma_btilde_size", "lcma_gemm", "lcma_precombine_b", "lcma_gemm_precombined",
                 "lcma_decide", "lcma_scheme_register_file", "lcma_scheme_register",
                 "lcma_scheme_get", "lcma_plan_schedule", "lcma_workspace_region"):
        getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def _check(st: int):
    if st != 0:
        raise LcmaError(st, lib().lcma_last_error().decode())


def _profile(hw):
    if hw is None:
        return None
    if isinstance(hw, dict):
        hw = HwProfile(hw["flops_mul"], hw["flops_add"], hw["beta_elems"], hw.get("workers", 0))
    return ctypes.pointer(hw)


_DT_TORCH = None


def _torch_dtype(code):
    import torch
    return {BF16: torch.bfloat16, FP16: torch.float16, TF32: torch.float32, FP32: torch.float32,
            FP8: torch.bfloat16}[code]


class Plan:
    """lcma_plan_ex wrapper.  gemm() takes CUDA torch tensors (row-major,
    contiguous, on one device, of the plan's dtype and shape); the call is
    enqueued on that device's current stream (or `stream`)."""

    def __init__(self, M, N, K, dtype=BF16, algo="auto", out_dtype=None, b_layout=0,
                 variant="auto", b_static=False, schedule=0, num_ctas=0, scheme_id=0, hw=None,
                 decision_model=0, raster_rows=0):
        L = lib()
        if out_dtype is None:
            out_dtype = FP32 if dtype == TF32 else (BF16 if dtype == FP8 else dtype)
        self._hw = _profile(hw)
        d = PlanDesc(M, N, K, dtype, out_dtype, ALGO[algo] if isinstance(algo, str) else algo,
                     scheme_id, b_layout, int(b_static),
                     VARIANT[variant] if isinstance(variant, str) else variant,
                     schedule, num_ctas, self._hw, decision_model, raster_rows, 0)
        h = ctypes.c_void_p()
        _check(L.lcma_plan_ex(ctypes.byref(d), ctypes.byref(h)))
        self._h = h
        self.M, self.N, self.K = M, N, K
        self.dtype, self.out_dtype, self.b_layout = dtype, out_dtype, b_layout
        info = PlanInfo()
        _check(L.lcma_plan_get_info(h, ctypes.byref(info)))
        self.info = info.as_dict()
        self.workspace_bytes = self.info["workspace_bytes"]
        self.btilde_bytes = self.info["btilde_bytes"]
        self._ws = {}

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.lcma_free(h)
            self._h = None

    def workspace(self, device=None, stream=None):
        """Zero-initialised workspace (the library keeps its counters and flags
        zero afterwards).  Cached per (device, stream): a workspace must not be
        used by two in-flight calls at once (include/lcma.h)."""
        import torch
        dev = torch.device(device if device is not None else "cuda")
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        key = (dev.index, self._stream(stream, dev).value or 0)
        ws = self._ws.get(key)
        if ws is None:
            ws = torch.zeros(max(self.workspace_bytes, 16), dtype=torch.uint8, device=dev)
            self._ws[key] = ws
        return ws

    @staticmethod
    def _stream(stream, device=None):
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(device)
        return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))

    def empty_c(self, device="cuda"):
        import torch
        return torch.empty((self.M, self.N), dtype=_torch_dtype(self.out_dtype), device=device)

    # -- argument checks (the C ABI sees raw pointers and cannot check sizes)
    def _check_t(self, t, name, dtype, numel, dev):
        import torch
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise LcmaError(1, f"{name} must be a CUDA tensor")
        if t.device != dev:
            raise LcmaError(1, f"{name} is on {t.device}, A on {dev}")
        if not t.is_contiguous():
            raise LcmaError(1, f"{name} must be contiguous (row-major)")
        if dtype is not None and t.dtype != dtype:
            raise LcmaError(1, f"{name} has dtype {t.dtype}, the plan needs {dtype}")
        if t.numel() * t.element_size() < numel:
            raise LcmaError(1, f"{name} holds {t.numel() * t.element_size()} bytes, needs {numel}")

    def _check_args(self, A, B, Bt, C, ws):
        import torch
        dt = _torch_dtype(self.dtype)
        e = torch.empty((), dtype=dt).element_size()
        self._check_t(A, "A", dt, 0, A.device if isinstance(A, torch.Tensor) else None)
        dev = A.device
        if tuple(A.shape) != (self.M, self.K):
            raise LcmaError(1, f"A is {tuple(A.shape)}, the plan needs {(self.M, self.K)}")
        if B is not None:
            self._check_t(B, "B", dt, 0, dev)
            want = (self.K, self.N) if self.b_layout == 0 else (self.N, self.K)
            if tuple(B.shape) != want:
                raise LcmaError(1, f"B is {tuple(B.shape)}, the plan needs {want}")
        if Bt is not None:
            self._check_t(Bt, "Bt", None, self.btilde_bytes, dev)
        self._check_t(C, "C", _torch_dtype(self.out_dtype), 0, dev)
        if tuple(C.shape) != (self.M, self.N):
            raise LcmaError(1, f"C is {tuple(C.shape)}, the plan needs {(self.M, self.N)}")
        self._check_t(ws, "workspace", None, self.workspace_bytes, dev)
        return dev

    def gemm(self, A, B, C=None, workspace=None, stream=None):
        import torch
        if C is None:
            C = self.empty_c(A.device)
        ws = workspace if workspace is not None else self.workspace(A.device, stream)
        dev = self._check_args(A, B, None, C, ws)
        with torch.cuda.device(dev):
            _check(lib().lcma_gemm(self._h, A.data_ptr(), B.data_ptr(), C.data_ptr(),
                                   ws.data_ptr(), ws.numel() * ws.element_size(), self._stream(stream, dev)))
        return C

    def precombine_b(self, B, Bt=None, stream=None):
        import torch
        self._check_t(B, "B", _torch_dtype(self.dtype), 0, B.device if isinstance(B, torch.Tensor) else None)
        if Bt is None:
            Bt = torch.empty(max(self.btilde_bytes, 16), dtype=torch.uint8, device=B.device)
        self._check_t(Bt, "Bt", None, self.btilde_bytes, B.device)
        with torch.cuda.device(B.device):
            _check(lib().lcma_precombine_b(self._h, B.data_ptr(), Bt.data_ptr(), self._stream(stream, B.device)))
        return Bt

    def gemm_precombined(self, A, Bt, C=None, workspace=None, stream=None):
        import torch
        if C is None:
            C = self.empty_c(A.device)
        ws = workspace if workspace is not None else self.workspace(A.device, stream)
        if self.info["algo"] == ALGO["classical"] and self.dtype != FP8:
            dev = self._check_args(A, Bt, None, C, ws)     # classical: Bt is B itself
        else:
            dev = self._check_args(A, None, Bt, C, ws)
        with torch.cuda.device(dev):
            _check(lib().lcma_gemm_precombined(self._h, A.data_ptr(), Bt.data_ptr(), C.data_ptr(),
                                               ws.data_ptr(), ws.numel() * ws.element_size(),
                                               self._stream(stream, dev)))
        return C

    def workspace_region(self, which):
        """Byte offset of the A~ (0) / B~ (1) region of the workspace."""
        off = ctypes.c_size_t()
        _check(lib().lcma_workspace_region(self._h, which, ctypes.byref(off)))
        return off.value

    def schedule(self, cta):
        cap = 4096
        buf = (ctypes.c_int32 * (4 * cap))()
        n = ctypes.c_int32()
        _check(lib().lcma_plan_schedule(self._h, cta, buf, cap, ctypes.byref(n)))
        return [tuple(buf[4 * i:4 * i + 4]) for i in range(min(n.value, cap))]

    @staticmethod
    def last_launch_count():
        return int(lib().lcma_last_launch_count())


def set_kernel_events(start=None, end=None):
    """Record torch.cuda.Event `start`/`end` around the tcgen05 GEMM of later calls."""
    lib().lcma_set_kernel_events(start.cuda_event if start is not None else None,
                                 end.cuda_event if end is not None else None)


def decide(M, N, K, dtype=BF16, hw=None, fused=True):
    info = PlanInfo()
    _check(lib().lcma_decide(M, N, K, dtype, _profile(hw), int(fused), ctypes.byref(info)))
    return info.as_dict()


def scheme_get(scheme_id):
    import numpy as np
    mknR = (ctypes.c_int32 * 4)()
    _check(lib().lcma_scheme_get(scheme_id, mknR, None, None, None))
    m, k, n, R = list(mknR)
    U = np.zeros((R, m, k), np.int8)
    V = np.zeros((R, k, n), np.int8)
    W = np.zeros((R, m, n), np.int8)
    _check(lib().lcma_scheme_get(scheme_id, mknR, U.ctypes.data, V.ctypes.data, W.ctypes.data))
    return m, k, n, R, U, V, W


def scheme_register_file(path):
    sid = ctypes.c_int32()
    _check(lib().lcma_scheme_register_file(os.fsencode(path), ctypes.byref(sid)))
    return sid.value


def scheme_register(U, V, W, name="registered"):
    import numpy as np
    U = np.ascontiguousarray(U, np.int8)
    V = np.ascontiguousarray(V, np.int8)
    W = np.ascontiguousarray(W, np.int8)
    R, m, k = U.shape
    n = V.shape[2]
    sid = ctypes.c_int32()
    _check(lib().lcma_scheme_register(m, k, n, R, U.ctypes.data, V.ctypes.data, W.ctypes.data,
                                      name.encode(), ctypes.byref(sid)))
    return sid.value
