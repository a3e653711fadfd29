"""ctypes binding of include/quantc_cuda.h — the kernel-level C ABI — taking
torch CUDA tensors (torch is only the device-memory/stream plumbing here).
Fails loudly when the extension is missing: there is no fallback."""
from __future__ import annotations

import ctypes as C

import torch

from . import quantc as Q

_P = C.c_void_p


class CudaOps:
    def __init__(self, lib: C.CDLL):
        self.lib = lib
        L = lib
        L.qcu_last_error.restype = C.c_char_p
        L.qcu_sim_quant.argtypes = [_P, _P, C.c_int64, C.POINTER(Q.QParams), _P]
        L.qcu_minmax.argtypes = [_P, C.c_int64, _P, _P]
        L.qcu_histogram.argtypes = [_P, C.c_int64, C.c_double, C.c_int, _P, _P]
        L.qcu_kl_sweep.argtypes = [_P, C.c_int, C.c_int, C.c_int, _P, _P, _P]
        L.qcu_conv2d_f64acc.argtypes = [_P, _P, _P, _P] + [C.c_int] * 11 + [_P]
        L.qcu_conv2d_grouped_f64acc.argtypes = [_P, _P, _P, _P] + [C.c_int] * 12 + [_P]
        L.qcu_avg_pool2d_f32.argtypes = [_P, _P] + [C.c_int] * 10 + [_P]
        L.qcu_conv2d_int.argtypes = ([_P, _P, _P, _P] + [C.c_int] * 11 + [C.c_int64, C.c_int64]
                                     + [C.c_int, C.c_int, C.POINTER(C.c_int64), _P])
        L.qcu_requantize.argtypes = [_P, _P, C.c_int64, C.c_int64, C.c_int, C.c_int64,
                                     C.c_int64, C.c_int64, C.c_int64, _P]
        L.qcu_gemm_s8.argtypes = [_P, _P, C.c_int, C.c_int, C.c_int, C.c_double, _P, _P, C.c_int,
                                  _P]
        L.qcu_argmax_rows.argtypes = [_P, C.c_int, C.c_int64, C.c_int, _P, _P]
        L.qcu_synchronize.argtypes = [_P]
        L.qcu_set_engine_mode.argtypes = [C.c_int]
        L.qcu_counters.argtypes = [C.POINTER(C.c_int64)] * 4
        L.qcu_simt_int_convs.argtypes = [C.POINTER(C.c_int64)]

    def _ok(self, rc):
        if rc != 0:
            raise Q.DeviceError(self.lib.qcu_last_error().decode())

    @staticmethod
    def _s():
        # torch's default stream has handle 0, which the ABI reserves for the
        # engine stream; pass cudaStreamLegacy (0x1) so kernels order with it
        h = torch.cuda.current_stream().cuda_stream
        return C.c_void_p(h if h else 1)

    @staticmethod
    def _p(t):
        return None if t is None else C.c_void_p(t.data_ptr())

    def sim_quant(self, x: torch.Tensor, p: Q.QParams, out=None) -> torch.Tensor:
        y = torch.empty_like(x) if out is None else out
        self._ok(self.lib.qcu_sim_quant(self._p(x), self._p(y), x.numel(), C.byref(p), self._s()))
        return y

    def minmax(self, x):
        out = torch.empty(2, dtype=torch.float64, device=x.device)
        self._ok(self.lib.qcu_minmax(self._p(x), x.numel(), self._p(out), self._s()))
        return out

    def histogram(self, x, absmax, bins, counts=None):
        c = torch.zeros(bins, dtype=torch.int64, device=x.device) if counts is None else counts
        self._ok(self.lib.qcu_histogram(self._p(x), x.numel(), absmax, bins, self._p(c), self._s()))
        return c

    def kl_sweep(self, counts: torch.Tensor, target_bit: int):
        e, bins = counts.shape
        bi = torch.empty(e, dtype=torch.int32, device=counts.device)
        bk = torch.empty(e, dtype=torch.float64, device=counts.device)
        self._ok(self.lib.qcu_kl_sweep(self._p(counts), e, bins, target_bit, self._p(bi),
                                       self._p(bk), self._s()))
        return bi, bk

    def conv2d_f64acc(self, x, w, bias, stride=(1, 1), pad=(0, 0)):
        N, Cc, H, W = x.shape
        O, _, KH, KW = w.shape
        OH = (H + 2 * pad[0] - KH) // stride[0] + 1
        OW = (W + 2 * pad[1] - KW) // stride[1] + 1
        y = torch.empty((N, O, OH, OW), dtype=torch.float32, device=x.device)
        self._ok(self.lib.qcu_conv2d_f64acc(self._p(x), self._p(w), self._p(bias), self._p(y),
                                            N, Cc, H, W, O, KH, KW, stride[0], stride[1], pad[0],
                                            pad[1], self._s()))
        return y

    def conv2d_grouped_f64acc(self, x, w, bias, stride=(1, 1), pad=(0, 0), groups=1):
        N, Cc, H, W = x.shape
        O, _, KH, KW = w.shape
        OH = (H + 2 * pad[0] - KH) // stride[0] + 1
        OW = (W + 2 * pad[1] - KW) // stride[1] + 1
        y = torch.empty((N, O, OH, OW), dtype=torch.float32, device=x.device)
        self._ok(self.lib.qcu_conv2d_grouped_f64acc(self._p(x), self._p(w), self._p(bias),
                                                    self._p(y), N, Cc, H, W, O, KH, KW, stride[0],
                                                    stride[1], pad[0], pad[1], groups, self._s()))
        return y

    def avg_pool2d(self, x, k, stride, pad):
        N, Cc, H, W = x.shape
        OH = (H + 2 * pad[0] - k[0]) // stride[0] + 1
        OW = (W + 2 * pad[1] - k[1]) // stride[1] + 1
        y = torch.empty((N, Cc, OH, OW), dtype=torch.float32, device=x.device)
        self._ok(self.lib.qcu_avg_pool2d_f32(self._p(x), self._p(y), N, Cc, H, W, k[0], k[1],
                                             stride[0], stride[1], pad[0], pad[1], self._s()))
        return y

    def conv2d_int(self, x, w, bias, stride, pad, zp0, zp1, acc_dtype, trap=False):
        N, Cc, H, W = x.shape
        O, _, KH, KW = w.shape
        OH = (H + 2 * pad[0] - KH) // stride[0] + 1
        OW = (W + 2 * pad[1] - KW) // stride[1] + 1
        y = torch.empty((N, O, OH, OW), dtype=torch.int32, device=x.device)
        flat = C.c_int64(-1)
        self._ok(self.lib.qcu_conv2d_int(self._p(x), self._p(w), self._p(bias), self._p(y), N, Cc,
                                         H, W, O, KH, KW, stride[0], stride[1], pad[0], pad[1],
                                         zp0, zp1, acc_dtype, int(trap), C.byref(flat),
                                         self._s()))
        return y, flat.value

    def requantize(self, x, mult, shift, in_zp, out_zp, qmin, qmax):
        y = torch.empty_like(x)
        self._ok(self.lib.qcu_requantize(self._p(x), self._p(y), x.numel(), mult, shift, in_zp,
                                         out_zp, qmin, qmax, self._s()))
        return y

    def argmax_rows(self, x, grouped=0):
        out = torch.empty(x.shape[0], dtype=torch.int64, device=x.device)
        self._ok(self.lib.qcu_argmax_rows(self._p(x), x.shape[0], x.shape[1], grouped,
                                          self._p(out), self._s()))
        return out

    def gemm_s8(self, A, B, scale=1.0, bias=None, ohw=1):
        M, K = A.shape
        N = B.shape[0]
        y = torch.empty((M // ohw, N, ohw), dtype=torch.float32, device=A.device)
        self._ok(self.lib.qcu_gemm_s8(self._p(A), self._p(B), M, N, K, scale, self._p(bias),
                                      self._p(y), ohw, self._s()))
        return y

    def synchronize(self):
        self._ok(self.lib.qcu_synchronize(None))

    def tcgen05_available(self) -> bool:
        return bool(self.lib.qcu_tcgen05_available())

    def set_engine_mode(self, mode: str):
        self._ok(self.lib.qcu_set_engine_mode({"exact": 0, "fast": 1, "auto": 2}[mode]))

    def counters(self):
        v = [C.c_int64() for _ in range(4)]
        self.lib.qcu_counters(*[C.byref(x) for x in v])
        s = C.c_int64()
        self.lib.qcu_simt_int_convs(C.byref(s))
        return {"steps": v[0].value, "tcgen05_gemms": v[1].value, "f64_convs": v[2].value,
                "fused_batches": v[3].value, "simt_int_convs": s.value}


_ops = None


def load() -> CudaOps:
    global _ops
    if _ops is None:
        _ops = CudaOps(Q.load_b200().lib)
    return _ops
