"""ctypes front end of the test-only oracles (oracle/cpu_ref.c, oracle/ref_shim.cpp).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs, always as the checker or
the timed CPU baseline, never as the product path.  The product package
(``paper_2407_02327_b200``) does not import this module.

Two libraries:
  * ``CpuRef``   -- the CPU restatement (always present once ``make -f
    oracle/Makefile`` ran).
  * ``RefLib``   -- the unmodified reference library (oracle/_ref/libqsync_ref.so),
    built from /root/reference/proj/src when the tree exists.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")

_i64 = C.c_int64
_u64 = C.c_uint64
_f32 = C.c_float
_p = C.c_void_p


def build() -> None:
    """Compile the oracle libraries (the reference one only if its tree exists)."""
    subprocess.run(["make", "-s", "-f", os.path.join(HERE, "Makefile"), "all", "acceptance"], check=True)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_p) if a is not None else None


class CpuRef:
    """The CPU restatement (cpu_ref.c)."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(REF_DIR, "libqsync_cpuref.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        self.L = L
        L.ref_mt64_draws.argtypes = [_u64, _i64, _p]
        L.ref_stochastic_round.argtypes = [_p, _i64, C.c_double, C.c_double, _u64, _p, _p]
        L.ref_stochastic_round.restype = C.c_int
        L.ref_stochastic_round_float.argtypes = [_p, _i64, C.c_int, C.c_int, _u64, _p]
        L.ref_stochastic_round_float.restype = C.c_int
        L.ref_absmax_f32.argtypes = [_p, _i64]
        L.ref_absmax_f32.restype = _f32
        L.ref_scale_from_absmax.argtypes = [_f32]
        L.ref_scale_from_absmax.restype = _f32
        L.ref_quantize_per_tensor.argtypes = [_p, _i64, _p, _p]
        L.ref_quantize_per_channel.argtypes = [_p, _i64, _i64, _p, _p]
        L.ref_quantize_sr_per_tensor.argtypes = [_p, _i64, _f32, _u64, _p]
        L.ref_dequantize_per_tensor.argtypes = [_p, _i64, _f32, _p]
        L.ref_dequantize_per_channel.argtypes = [_p, _i64, _i64, _p, _p]
        L.ref_cast_f32_f16.argtypes = [_p, _i64, _p]
        L.ref_gemm_s8_tn.argtypes = [_p, _p, _i64, _i64, _i64, _p]
        L.ref_dequant_epilogue.argtypes = [_p, _i64, _i64, _f32, _p, _p, _p]
        L.ref_gemm_f16_tn.argtypes = [_p, _p, _i64, _i64, _i64, _f32, _p]
        L.ref_gemm_f32_tn.argtypes = [_p, _p, _i64, _i64, _i64, _p]
        L.ref_tensor_stats_f32.argtypes = [_p, _i64, _p]
        L.ref_qlinear_int8_fwd_bwd.argtypes = [_p] * 4 + [_i64] * 3 + [_p] * 9
        L.ref_qlinear_f16_fwd_bwd.argtypes = [_p] * 4 + [_i64] * 3 + [_p] * 4
        L.ref_im2col.argtypes = [_p, C.c_int] + [_i64] * 4 + [C.c_int] * 8 + [_i64] * 3 + [_p]
        L.ref_col2im.argtypes = [_p] + [_i64] * 4 + [C.c_int] * 8 + [_i64] * 3 + [_p]
        L.ref_num_threads.restype = C.c_int

    # -- RNG / SR ----------------------------------------------------------
    def mt64_draws(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, np.uint64)
        self.L.ref_mt64_draws(seed, n, _ptr(out))
        return out

    def stochastic_round(self, x, q: float, zp: float, seed: int):
        x = np.ascontiguousarray(x, np.float64)
        r = np.empty(x.size, np.int64)
        d = np.empty(x.size, np.float64)
        rc = self.L.ref_stochastic_round(_ptr(x), x.size, q, zp, seed, _ptr(r), _ptr(d))
        if rc:
            raise ValueError("domain: stochastic rounding needs a scaling factor > 0")
        return r, d

    def stochastic_round_float(self, x, e: int, k: int, seed: int) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        d = np.empty(x.size, np.float64)
        if self.L.ref_stochastic_round_float(_ptr(x), x.size, e, k, seed, _ptr(d)):
            raise ValueError("domain: mantissa bit count must be at least 1")
        return d

    # -- quantization ------------------------------------------------------
    def absmax(self, x) -> float:
        x = np.ascontiguousarray(x, np.float32)
        return float(self.L.ref_absmax_f32(_ptr(x), x.size))

    def scale_from_absmax(self, a: float) -> np.float32:
        return np.float32(self.L.ref_scale_from_absmax(a))

    def quantize_per_tensor(self, x):
        x = np.ascontiguousarray(x, np.float32)
        q = np.empty(x.shape, np.int8)
        s = np.zeros(1, np.float32)
        self.L.ref_quantize_per_tensor(_ptr(x), x.size, _ptr(q), _ptr(s))
        return q, s[0]

    def quantize_per_channel(self, w):
        w = np.ascontiguousarray(w, np.float32)
        rows, cols = w.shape
        q = np.empty(w.shape, np.int8)
        s = np.empty(rows, np.float32)
        self.L.ref_quantize_per_channel(_ptr(w), rows, cols, _ptr(q), _ptr(s))
        return q, s

    def quantize_sr_per_tensor(self, x, scale: float, seed: int) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        q = np.empty(x.shape, np.int8)
        self.L.ref_quantize_sr_per_tensor(_ptr(x), x.size, np.float32(scale), seed, _ptr(q))
        return q

    def dequantize_per_tensor(self, q, scale: float) -> np.ndarray:
        q = np.ascontiguousarray(q, np.int8)
        out = np.empty(q.shape, np.float32)
        self.L.ref_dequantize_per_tensor(_ptr(q), q.size, np.float32(scale), _ptr(out))
        return out

    def dequantize_per_channel(self, q, scales) -> np.ndarray:
        q = np.ascontiguousarray(q, np.int8)
        scales = np.ascontiguousarray(scales, np.float32)
        out = np.empty(q.shape, np.float32)
        self.L.ref_dequantize_per_channel(_ptr(q), q.shape[0], q.shape[1], _ptr(scales), _ptr(out))
        return out

    def cast_f32_f16(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty(x.shape, np.uint16)
        self.L.ref_cast_f32_f16(_ptr(x), x.size, _ptr(out))
        return out.view(np.float16)

    # -- GEMM --------------------------------------------------------------
    def gemm_s8_tn(self, a, b) -> np.ndarray:
        a = np.ascontiguousarray(a, np.int8)
        b = np.ascontiguousarray(b, np.int8)
        M, K = a.shape
        N = b.shape[0]
        c = np.empty((M, N), np.int32)
        self.L.ref_gemm_s8_tn(_ptr(a), _ptr(b), M, N, K, _ptr(c))
        return c

    def dequant_epilogue(self, acc, s_a: float, s_w, bias=None) -> np.ndarray:
        acc = np.ascontiguousarray(acc, np.int32)
        s_w = np.ascontiguousarray(s_w, np.float32)
        M, N = acc.shape
        y = np.empty((M, N), np.float32)
        b = np.ascontiguousarray(bias, np.float32) if bias is not None else None
        self.L.ref_dequant_epilogue(_ptr(acc), M, N, np.float32(s_a), _ptr(s_w), _ptr(b), _ptr(y))
        return y

    def gemm_f16_tn(self, a, b, alpha: float = 1.0) -> np.ndarray:
        a = np.ascontiguousarray(a, np.float16).view(np.uint16)
        b = np.ascontiguousarray(b, np.float16).view(np.uint16)
        M, K = a.shape
        N = b.shape[0]
        c = np.empty((M, N), np.float32)
        self.L.ref_gemm_f16_tn(_ptr(a), _ptr(b), M, N, K, np.float32(alpha), _ptr(c))
        return c

    def gemm_f32_tn(self, a, b) -> np.ndarray:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        M, K = a.shape
        N = b.shape[0]
        c = np.empty((M, N), np.float32)
        self.L.ref_gemm_f32_tn(_ptr(a), _ptr(b), M, N, K, _ptr(c))
        return c

    def tensor_stats(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty(5, np.float64)
        self.L.ref_tensor_stats_f32(_ptr(x), x.size, _ptr(out))
        return out

    def qlinear_int8(self, x, w, bias, dy):
        """Forward + backward of one INT8 Linear (cpu_ref.c ref_qlinear_int8_fwd_bwd)."""
        x = np.ascontiguousarray(x, np.float32)
        w = np.ascontiguousarray(w, np.float32)
        M, K = x.shape
        N = w.shape[0]
        b = np.ascontiguousarray(bias, np.float32) if bias is not None else None
        g = np.ascontiguousarray(dy, np.float32) if dy is not None else None
        xq = np.empty((M, K), np.int8)
        wq = np.empty((N, K), np.int8)
        sx = np.empty(1, np.float32)
        sw = np.empty(N, np.float32)
        acc = np.empty((M, N), np.int32)
        y = np.empty((M, N), np.float32)
        dx = np.empty((M, K), np.float32)
        dw = np.empty((N, K), np.float32)
        db = np.empty(N, np.float32)
        self.L.ref_qlinear_int8_fwd_bwd(_ptr(x), _ptr(w), _ptr(b), _ptr(g), M, N, K, _ptr(xq),
                                        _ptr(wq), _ptr(sx), _ptr(sw), _ptr(acc), _ptr(y),
                                        _ptr(dx), _ptr(dw), _ptr(db))
        return dict(xq=xq, wq=wq, s_x=sx[0], s_w=sw, acc=acc, y=y, dx=dx, dw=dw, db=db)

    def qlinear_f16(self, x, w, bias, dy):
        """Forward + backward of one FP16 Linear (cpu_ref.c ref_qlinear_f16_fwd_bwd)."""
        x = np.ascontiguousarray(x, np.float32)
        w = np.ascontiguousarray(w, np.float32)
        M, K = x.shape
        N = w.shape[0]
        b = np.ascontiguousarray(bias, np.float32) if bias is not None else None
        g = np.ascontiguousarray(dy, np.float32) if dy is not None else None
        y = np.empty((M, N), np.float32)
        dx = np.empty((M, K), np.float32)
        dw = np.empty((N, K), np.float32)
        db = np.empty(N, np.float32)
        self.L.ref_qlinear_f16_fwd_bwd(_ptr(x), _ptr(w), _ptr(b), _ptr(g), M, N, K, _ptr(y),
                                       _ptr(dx), _ptr(dw), _ptr(db))
        return dict(y=y, dx=dx, dw=dw, db=db)

    @staticmethod
    def conv_out(H, W, R, S, stride, pad, dil=(1, 1)):
        P = (H + 2 * pad[0] - dil[0] * (R - 1) - 1) // stride[0] + 1
        Q = (W + 2 * pad[1] - dil[1] * (S - 1) - 1) // stride[1] + 1
        return P, Q

    def im2col(self, x, R, S, stride, pad, dil=(1, 1), ld=None):
        x = np.ascontiguousarray(x)
        N, H, W, Cc = x.shape
        P, Q = self.conv_out(H, W, R, S, stride, pad, dil)
        K = R * S * Cc
        ld = ld or K
        out = np.empty((N * P * Q, ld), x.dtype)
        self.L.ref_im2col(_ptr(x), x.itemsize, N, H, W, Cc, R, S, stride[0], stride[1], pad[0],
                          pad[1], dil[0], dil[1], P, Q, ld, _ptr(out))
        return out, (P, Q)

    def col2im(self, dcol, xshape, R, S, stride, pad, dil=(1, 1)):
        dcol = np.ascontiguousarray(dcol, np.float32)
        N, H, W, Cc = xshape
        P, Q = self.conv_out(H, W, R, S, stride, pad, dil)
        dx = np.empty((N, H, W, Cc), np.float32)
        self.L.ref_col2im(_ptr(dcol), N, H, W, Cc, R, S, stride[0], stride[1], pad[0], pad[1],
                          dil[0], dil[1], P, Q, dcol.shape[1], _ptr(dx))
        return dx

    def num_threads(self) -> int:
        return int(self.L.ref_num_threads())


class RefLib:
    """The unmodified reference (oracle/_ref/libqsync_ref.so)."""

    PATH = os.path.join(REF_DIR, "libqsync_ref.so")

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(cls.PATH)

    def __init__(self):
        L = C.CDLL(self.PATH)
        self.L = L
        L.qref_last_error.restype = C.c_char_p
        L.qref_stochastic_round.argtypes = [_p, _i64, C.c_double, C.c_double, _u64, _p, _p]
        L.qref_stochastic_round_float.argtypes = [_p, _i64, C.c_int, C.c_int, _u64, _p]
        L.qref_mt64_draws.argtypes = [_u64, _i64, _p]
        L.qref_uniform01.argtypes = [_u64, _i64, _p]
        L.qref_sigma.argtypes = [C.c_int, _p, C.c_uint32, C.c_int, C.c_int, C.c_int, _p]
        L.qref_omega.argtypes = [_p, C.c_uint32, C.c_int, C.c_int, C.c_int, C.c_int, _i64,
                                 C.c_int, C.c_int, _p]
        L.qref_reduce_stats.argtypes = [_p, _p, C.c_int, C.c_int, _p, _p]
        L.qref_score_bundle.argtypes = [C.c_char_p, C.c_int, _i64, C.c_int, C.c_char_p, _i64]
        L.qref_score_bundle.restype = _i64
        L.qref_plan_bundle.argtypes = [C.c_char_p, C.c_int, _i64, C.c_int, C.c_char_p, _i64,
                                       C.c_int, C.c_char_p, _i64]
        L.qref_plan_bundle.restype = _i64
        L.qref_replay_bundle.argtypes = [C.c_char_p, C.c_char_p]
        L.qref_replay_bundle.restype = _i64
        L.qref_replay_trace.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, _i64]
        L.qref_replay_trace.restype = _i64

    def _err(self, rc):
        if rc:
            raise RuntimeError(self.L.qref_last_error().decode())

    def stochastic_round(self, x, q, zp, seed):
        x = np.ascontiguousarray(x, np.float64)
        r = np.empty(x.size, np.int64)
        d = np.empty(x.size, np.float64)
        self._err(self.L.qref_stochastic_round(_ptr(x), x.size, q, zp, seed, _ptr(r), _ptr(d)))
        return r, d

    def stochastic_round_float(self, x, e, k, seed):
        x = np.ascontiguousarray(x, np.float64)
        d = np.empty(x.size, np.float64)
        self._err(self.L.qref_stochastic_round_float(_ptr(x), x.size, e, k, seed, _ptr(d)))
        return d

    def mt64_draws(self, seed, n):
        out = np.empty(n, np.uint64)
        self.L.qref_mt64_draws(seed, n, _ptr(out))
        return out

    def uniform01(self, seed, n):
        out = np.empty(n, np.float64)
        self.L.qref_uniform01(seed, n, _ptr(out))
        return out

    def sigma(self, which, values, mask, precision, parameter_free, k=9):
        v = np.ascontiguousarray(values, np.float64)
        out = np.zeros(1, np.float64)
        self._err(self.L.qref_sigma(which, _ptr(v), mask, precision, int(parameter_free), k,
                                    _ptr(out)))
        return float(out[0])

    def omega(self, values, mask, has_weight, depth, d_l, loss_kind, loss_n, precision, k=9):
        v = np.ascontiguousarray(values, np.float64)
        out = np.zeros(1, np.float64)
        self._err(self.L.qref_omega(_ptr(v), mask, int(has_weight), depth, d_l, loss_kind, loss_n,
                                    precision, k, _ptr(out)))
        return float(out[0])

    def reduce_stats(self, values, masks, window):
        v = np.ascontiguousarray(values, np.float64)
        m = np.ascontiguousarray(masks, np.uint32)
        out = np.zeros(12, np.float64)
        om = np.zeros(1, np.uint32)
        self._err(self.L.qref_reduce_stats(_ptr(v), _ptr(m), len(m), window, _ptr(out), _ptr(om)))
        return out, int(om[0])

    def plan_bundle(self, path, loss_kind=0, loss_n=1, window=50, cap_device="", cap_bytes=0,
                    b_max=8) -> dict:
        """The reference planner (cli.cpp:116-136) on a bundle: the solve_report JSON."""
        import json as _json
        buf = C.create_string_buffer(8 << 20)
        n = self.L.qref_plan_bundle(path.encode(), loss_kind, loss_n, window, cap_device.encode(),
                                    cap_bytes, b_max, buf, 8 << 20)
        if n < 0:
            raise RuntimeError(self.L.qref_last_error().decode())
        return _json.loads(buf.raw[:n].decode())

    def replay_bundle(self, path, plan: dict) -> int:
        """The reference replayer's makespan (ns) for a plan (cli.cpp:90-114)."""
        import json as _json
        n = self.L.qref_replay_bundle(path.encode(), _json.dumps(plan).encode())
        if n < 0:
            raise RuntimeError(self.L.qref_last_error().decode())
        return int(n)

    def replay_trace(self, path, plan: dict) -> dict:
        """The replayer's Chrome trace of one simulated iteration (replayer.cpp:126-148)."""
        import json as _json
        buf = C.create_string_buffer(16 << 20)
        n = self.L.qref_replay_trace(path.encode(), _json.dumps(plan).encode(), buf, 16 << 20)
        if n < 0:
            raise RuntimeError(self.L.qref_last_error().decode())
        return _json.loads(buf.raw[:n].decode())

    def score_bundle(self, path, loss_kind, loss_n, window=50):
        buf = C.create_string_buffer(1 << 20)
        n = self.L.qref_score_bundle(path.encode(), loss_kind, loss_n, window, buf, 1 << 20)
        if n < 0:
            raise RuntimeError(self.L.qref_last_error().decode())
        rows = []
        for line in buf.raw[:n].decode().splitlines():
            op, p, w = line.split("\t")
            rows.append((op, p, float(w)))
        return rows
