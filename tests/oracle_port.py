"""ctypes view of the plain-C oracle restatement (oracle/quantc_oracle.c).
TEST INFRASTRUCTURE: a checker, never the thing measured."""
import ctypes as C

import numpy as np

_F = C.POINTER(C.c_float)
_I32 = C.POINTER(C.c_int32)
_I64 = C.POINTER(C.c_int64)


class Port:
    def __init__(self, path):
        L = self.lib = C.CDLL(path)
        L.orc_sim_quant.restype = C.c_float
        L.orc_sim_quant.argtypes = [C.c_float, C.c_double, C.c_int, C.c_int, C.c_int64, C.c_int,
                                    C.c_int, C.c_double, C.c_double]
        L.orc_sim_quant_array.argtypes = [_F, _F, C.c_int64, C.c_double, C.c_int, C.c_int,
                                          C.c_int64, C.c_int, C.c_int, C.c_double, C.c_double]
        L.orc_histogram.argtypes = [_F, C.c_int64, C.c_double, C.c_int, _I64]
        L.orc_threshold_quantile.restype = C.c_double
        L.orc_threshold_quantile.argtypes = [_I64, C.c_int, C.c_double, C.c_double]
        L.orc_kl_best_index.restype = C.c_int
        L.orc_kl_best_index.argtypes = [_I64, C.c_int, C.c_int, C.POINTER(C.c_double)]
        L.orc_conv2d_f64acc.argtypes = [_F, _F, _F, _F] + [C.c_int] * 11
        L.orc_conv2d_grouped_f64acc.argtypes = [_F, _F, _F, _F] + [C.c_int] * 12
        L.orc_avg_pool2d.argtypes = [_F, _F] + [C.c_int] * 10
        L.orc_global_avg_pool2d.argtypes = [_F, _F, C.c_int, C.c_int]
        L.orc_conv2d_int.restype = C.c_int64
        L.orc_conv2d_int.argtypes = [_I32, _I32, _I32, _I32] + [C.c_int] * 11 + [C.c_int64] * 4
        L.orc_requantize.argtypes = [_I32, _I32, C.c_int64, C.c_int64, C.c_int, C.c_int64,
                                     C.c_int64, C.c_int64, C.c_int64]

    def sim_quant(self, x, threshold, bit, sign=1, zero_point=0, passthrough=False,
                  acc=None):
        x = np.ascontiguousarray(x, np.float32)
        y = np.empty_like(x)
        lo, hi = acc if acc is not None else (0.0, 0.0)
        self.lib.orc_sim_quant_array(x.ctypes.data_as(_F), y.ctypes.data_as(_F), x.size,
                                     threshold, bit, sign, zero_point, int(passthrough),
                                     int(acc is not None), lo, hi)
        return y

    def histogram(self, x, absmax, bins):
        x = np.ascontiguousarray(x, np.float32)
        c = np.zeros(bins, np.int64)
        self.lib.orc_histogram(x.ctypes.data_as(_F), x.size, absmax, bins, c.ctypes.data_as(_I64))
        return c

    def kl_best_index(self, counts, target_bit):
        c = np.ascontiguousarray(counts, np.int64)
        kl = C.c_double()
        i = self.lib.orc_kl_best_index(c.ctypes.data_as(_I64), len(c), target_bit, C.byref(kl))
        return i, kl.value

    def quantile(self, counts, absmax, q):
        c = np.ascontiguousarray(counts, np.int64)
        return self.lib.orc_threshold_quantile(c.ctypes.data_as(_I64), len(c), absmax, q)

    def conv2d(self, x, w, bias, stride=(1, 1), pad=(0, 0), groups=1):
        x = np.ascontiguousarray(x, np.float32)
        w = np.ascontiguousarray(w, np.float32)
        N, Cc, H, W = x.shape
        O, _, KH, KW = w.shape
        OH = (H + 2 * pad[0] - KH) // stride[0] + 1
        OW = (W + 2 * pad[1] - KW) // stride[1] + 1
        y = np.empty((N, O, OH, OW), np.float32)
        b = None if bias is None else np.ascontiguousarray(bias, np.float32)
        self.lib.orc_conv2d_grouped_f64acc(x.ctypes.data_as(_F), w.ctypes.data_as(_F),
                                           None if b is None else b.ctypes.data_as(_F),
                                           y.ctypes.data_as(_F), N, Cc, H, W, O, KH, KW,
                                           stride[0], stride[1], pad[0], pad[1], groups)
        return y

    def avg_pool2d(self, x, k, stride, pad):
        x = np.ascontiguousarray(x, np.float32)
        N, Cc, H, W = x.shape
        OH = (H + 2 * pad[0] - k[0]) // stride[0] + 1
        OW = (W + 2 * pad[1] - k[1]) // stride[1] + 1
        y = np.empty((N, Cc, OH, OW), np.float32)
        self.lib.orc_avg_pool2d(x.ctypes.data_as(_F), y.ctypes.data_as(_F), N, Cc, H, W, k[0], k[1],
                                stride[0], stride[1], pad[0], pad[1])
        return y

    def global_avg_pool2d(self, x):
        x = np.ascontiguousarray(x, np.float32)
        N, Cc, H, W = x.shape
        y = np.empty((N, Cc, 1, 1), np.float32)
        self.lib.orc_global_avg_pool2d(x.ctypes.data_as(_F), y.ctypes.data_as(_F), N * Cc, H * W)
        return y

    def conv2d_int(self, x, w, bias, stride, pad, zp0, zp1, acc_min, acc_max):
        x = np.ascontiguousarray(x, np.int32)
        w = np.ascontiguousarray(w, np.int32)
        N, Cc, H, W = x.shape
        O, _, KH, KW = w.shape
        OH = (H + 2 * pad[0] - KH) // stride[0] + 1
        OW = (W + 2 * pad[1] - KW) // stride[1] + 1
        y = np.empty((N, O, OH, OW), np.int32)
        b = None if bias is None else np.ascontiguousarray(bias, np.int32)
        first = self.lib.orc_conv2d_int(x.ctypes.data_as(_I32), w.ctypes.data_as(_I32),
                                        None if b is None else b.ctypes.data_as(_I32),
                                        y.ctypes.data_as(_I32), N, Cc, H, W, O, KH, KW,
                                        stride[0], stride[1], pad[0], pad[1], zp0, zp1,
                                        acc_min, acc_max)
        return y, first

    def requantize(self, x, mult, shift, in_zp, out_zp, qmin, qmax):
        x = np.ascontiguousarray(x, np.int32)
        y = np.empty_like(x)
        self.lib.orc_requantize(x.ctypes.data_as(_I32), y.ctypes.data_as(_I32), x.size, mult,
                                shift, in_zp, out_zp, qmin, qmax)
        return y


def load(path):
    return Port(path)
