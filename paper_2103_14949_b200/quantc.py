"""Python mirror of the quantc calibrate-and-search API over the C-ABI.

Each class/function wraps one entry point of include/quantc_capi.h, which in
turn maps 1:1 onto the reference C++ API (/root/reference/proj/include/quantc,
cited per function).  The same wrapper drives two shared libraries:

  * ``load_b200()``       -> libquantc_b200.so   (this repo: C++ host + sm_100a kernels)
  * ``Quantc(path)``      -> any library exporting the same C ABI, e.g. the
                             reference compiled as a test oracle.

Errors come back as the Python analogues of the reference exception types
(SURVEY.md §5); ``OverflowError_`` carries (node, flat_index, value) like
interpreter.hpp:32-38.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence

import numpy as np

# ---- dtype codes (include/quantc_capi.h; reference dtype.hpp:13-19) --------
F32, I8, U8, I16, I32, NONE = 0, 1, 2, 3, 4, -1
DTYPE_NAMES = {F32: "float32", I8: "int8", U8: "uint8", I16: "int16", I32: "int32"}
DTYPE_CODES = {v: k for k, v in DTYPE_NAMES.items()}


class QuantcError(RuntimeError):
    pass


class InvalidArgument(QuantcError, ValueError):
    pass


class GraphError(QuantcError):
    pass


class SpecError(QuantcError):
    pass


class TopologyError(QuantcError):
    pass


class CalibrationError(QuantcError):
    pass


class SearchError(QuantcError):
    pass


class EvalError(QuantcError):
    pass


class OverflowError_(EvalError):
    def __init__(self, msg, node, flat_index, value):
        super().__init__(msg)
        self.node, self.flat_index, self.value = node, flat_index, value


class DeviceError(QuantcError):
    pass


class BufferError_(QuantcError):
    pass


_ERRORS = {1: InvalidArgument, 2: GraphError, 3: SpecError, 4: TopologyError,
           5: CalibrationError, 6: SearchError, 7: EvalError, 9: DeviceError,
           10: BufferError_, 11: QuantcError}


class QParams(C.Structure):
    """quantc::QParams (reference simulate.hpp:33-45) as the C-ABI POD."""
    _fields_ = [("threshold", C.c_double), ("bit", C.c_int32), ("sign", C.c_int32),
                ("in_dtype", C.c_int32), ("out_dtype", C.c_int32),
                ("zero_point", C.c_int64), ("passthrough", C.c_int32),
                ("acc_dtype", C.c_int32), ("acc_scale", C.c_double)]

    @staticmethod
    def make(threshold=0.0, bit=8, sign=1, in_dtype=I8, out_dtype=None, zero_point=0,
             passthrough=False, acc_dtype=NONE, acc_scale=0.0) -> "QParams":
        return QParams(threshold, bit, sign, in_dtype,
                       in_dtype if out_dtype is None else out_dtype, zero_point,
                       1 if passthrough else 0, acc_dtype, acc_scale)

    @staticmethod
    def symmetric(threshold, bit, storage=I8) -> "QParams":
        """QParams::symmetric (reference simulate.cpp:27-35)."""
        return QParams.make(threshold, bit, 1, storage, storage)

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class SearchParams(C.Structure):
    _fields_ = [("rounds", C.c_int32), ("tol", C.c_double), ("steps", C.c_int32),
                ("t0", C.c_double), ("decay", C.c_double), ("seed", C.c_uint64),
                ("n", C.c_int32), ("cap", C.c_int64)]


LOSS_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_int), C.c_size_t, C.c_void_p,
                      C.POINTER(C.c_double))
BATCH_LOSS_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_int), C.c_size_t, C.c_size_t, C.c_void_p,
                            C.POINTER(C.c_double))
COMM_SUM_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_int64), C.c_size_t, C.c_void_p)
COMM_F64_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_double), C.c_size_t, C.c_int, C.c_void_p)
COMM_GATHER_FN = C.CFUNCTYPE(C.c_int, C.POINTER(C.c_double), C.c_size_t,
                             C.POINTER(C.c_double), C.c_void_p)

_P = C.c_void_p
_SZ = C.c_size_t
_PI = C.POINTER(C.c_int)
_PI64 = C.POINTER(C.c_int64)
_PD = C.POINTER(C.c_double)
_PF = C.POINTER(C.c_float)
_PSZ = C.POINTER(C.c_size_t)
_PSTR = C.POINTER(C.c_void_p)

_SIGNATURES = {
    "qc_last_error": (C.c_char_p, []),
    "qc_last_overflow": (None, [_PI64, _PI64, _PI64]),
    "qc_impl_name": (C.c_char_p, []),
    "qc_free": (None, [_P]),
    "qc_graph_from_json": (C.c_int, [C.c_char_p, _P, _SZ, C.POINTER(_P)]),
    "qc_graph_to_json": (C.c_int, [_P, _PSTR]),
    "qc_graph_free": (None, [_P]),
    "qc_graph_num_nodes": (C.c_int, [_P, _PSZ]),
    "qc_validate_graph": (C.c_int, [_P, _PSTR]),
    "qc_traversal_order": (C.c_int, [_P, _PI64, _SZ, _PSZ]),
    "qc_edge_order": (C.c_int, [_P, _PI64, _SZ, _PSZ]),
    "qc_spec_parse": (C.c_int, [C.c_char_p, C.POINTER(_P)]),
    "qc_spec_free": (None, [_P]),
    "qc_spec_serialize": (C.c_int, [_P, _PSTR]),
    "qc_classify_op": (C.c_int, [_P, C.c_char_p, _PI]),
    "qc_candidate_dtypes": (C.c_int, [_P, C.c_char_p, C.c_int, _PI, _SZ, _PSZ]),
    "qc_match_signature": (C.c_int, [_P, C.c_char_p, _PI, _PI, _SZ, _PI, _PI, _PI]),
    "qc_generate_topology": (C.c_int, [_P, _P, C.POINTER(_P)]),
    "qc_topology_free": (None, [_P]),
    "qc_dump_topology": (C.c_int, [_P, _P, _PSTR]),
    "qc_topology_qv": (C.c_int, [_P, _PI64, _SZ, _PSZ]),
    "qc_insert_simulated_quantize": (C.c_int, [_P, _P, C.POINTER(_P)]),
    "qc_searchable_edge_indices": (C.c_int, [_P, _PI, _SZ, _PSZ]),
    "qc_simulated_edge_indices": (C.c_int, [_P, _P, _PI, _SZ, _PSZ]),
    "qc_dataset_create": (C.c_int, [_PF, C.c_int64, _PI64, C.c_int, _PI64, C.POINTER(_P)]),
    "qc_dataset_free": (None, [_P]),
    "qc_compute_scale": (C.c_int, [C.c_double, C.c_int, C.c_int, _PD]),
    "qc_quant_bounds": (C.c_int, [C.c_int, C.c_int, _PI64, _PI64]),
    "qc_simulated_quantize_value": (C.c_int, [C.c_float, C.POINTER(QParams), _PF]),
    "qc_simulated_quantize": (C.c_int, [_PF, C.c_int64, C.POINTER(QParams), _PF]),
    "qc_asymmetric_zero_point": (C.c_int, [C.c_double, C.c_double, C.c_int, _PI64]),
    "qc_noop_params": (C.c_int, [C.POINTER(QParams)]),
    "qc_collect_stats": (C.c_int, [_P, _P, C.c_int, _PI, _SZ, C.c_int, C.POINTER(_P)]),
    "qc_stats_create": (C.c_int, [C.POINTER(_P)]),
    "qc_stats_set_edge": (C.c_int, [_P, C.c_int, C.c_double, C.c_double, C.c_double,
                                    C.c_int64, _PI64, _SZ]),
    "qc_stats_free": (None, [_P]),
    "qc_stats_edges": (C.c_int, [_P, _PI, _SZ, _PSZ]),
    "qc_stats_get": (C.c_int, [_P, C.c_int, _PD, _PD, _PD, _PI64, _PI64, _SZ, _PSZ]),
    "qc_estimate_thresholds": (C.c_int, [_P, C.c_int, C.c_double, C.c_int, C.c_int, _PI,
                                         _PD, _SZ, _PSZ]),
    "qc_threshold_max": (C.c_int, [C.c_double, _PD]),
    "qc_threshold_quantile": (C.c_int, [_PI64, _SZ, C.c_double, C.c_double, _PD]),
    "qc_threshold_kl": (C.c_int, [_PI64, _SZ, C.c_double, C.c_int, _PD]),
    "qc_round_pow2": (C.c_int, [C.c_double, _PD]),
    "qc_eval_fp32": (C.c_int, [_P, _PF, _PI64, C.c_int, _PI64, C.POINTER(QParams), _SZ,
                               _PF, _SZ, _PSZ, _PI64, _PI]),
    "qc_eval_fp32_values": (C.c_int, [_P, _PF, _PI64, C.c_int, _PI64, _SZ, _PF, _SZ,
                                      _PSZ]),
    "qc_eval_int": (C.c_int, [_P, _PF, _PI64, C.c_int, C.c_int, C.POINTER(C.c_int32),
                              _SZ, _PSZ, _PI]),
    "qc_predict_top1": (C.c_int, [_P, _P, C.c_int, _PI64, C.POINTER(QParams), _SZ, _PI64,
                                  _SZ, _PSZ]),
    "qc_evaluator_create": (C.c_int, [_P, _P, _P, _PI, _PD, _SZ, _P, _P, C.c_int, C.c_int,
                                      C.POINTER(_P)]),
    "qc_evaluator_free": (None, [_P]),
    "qc_evaluator_space": (C.c_int, [_P, _PI, _PI, _PI, _SZ, _PSZ]),
    "qc_evaluator_refs": (C.c_int, [_P, _PI64, _SZ, _PSZ]),
    "qc_evaluator_bind": (C.c_int, [_P, _PI, _SZ, _PI64, C.POINTER(QParams), _SZ, _PSZ]),
    "qc_evaluator_loss": (C.c_int, [_P, _PI, _SZ, _PD]),
    "qc_evaluator_losses": (C.c_int, [_P, _PI, _SZ, _SZ, _PD]),
    "qc_evaluator_strategy": (C.c_int, [_P, _PI, _SZ, _PSTR]),
    "qc_evaluator_evaluations": (C.c_int, [_P, _PI64]),
    "qc_search": (C.c_int, [C.c_int, _PI, _PI, _PI, _SZ, LOSS_FN, _P, _P,
                            C.POINTER(SearchParams), _PI, _PD, _PI64, _PSTR]),
    "qc_space_size": (C.c_int, [_PI, _PI, _SZ, _PSTR]),
}


def _arr(a, ctype):
    """numpy array -> (contiguous array kept alive, ctypes pointer)."""
    np_t = {C.c_int: np.int32, C.c_int32: np.int32, C.c_int64: np.int64,
            C.c_double: np.float64, C.c_float: np.float32}[ctype]
    a = np.ascontiguousarray(np.asarray(a, dtype=np_t))
    return a, a.ctypes.data_as(C.POINTER(ctype))


class Quantc:
    """One loaded implementation of the quantc C ABI."""

    def __init__(self, path: str):
        self.path = path
        self.lib = C.CDLL(path)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(self.lib, name)
            fn.restype = res
            fn.argtypes = args
        self.name = self.lib.qc_impl_name().decode()

    # -- plumbing --------------------------------------------------------
    def check(self, rc: int):
        if rc == 0:
            return
        msg = self.lib.qc_last_error().decode(errors="replace")
        if rc == 8:
            node, flat, val = C.c_int64(), C.c_int64(), C.c_int64()
            self.lib.qc_last_overflow(C.byref(node), C.byref(flat), C.byref(val))
            raise OverflowError_(msg, node.value, flat.value, val.value)
        raise _ERRORS.get(rc, QuantcError)(msg)

    def _take_string(self, p: C.c_void_p) -> str:
        s = C.cast(p, C.c_char_p).value.decode()
        self.lib.qc_free(p)
        return s

    def _vec(self, fn, args, ctype, first_cap=256):
        n = C.c_size_t(0)
        cap = first_cap
        while True:
            buf, ptr = _arr(np.zeros(cap), ctype)
            rc = fn(*args, ptr, cap, C.byref(n))
            if rc == 10 and n.value > cap:
                cap = n.value
                continue
            self.check(rc)
            return buf[: n.value].copy()

    # -- graph (graph.hpp) ----------------------------------------------
    def graph(self, doc: dict, blob: bytes = b"") -> "Graph":
        h = C.c_void_p()
        buf = C.create_string_buffer(blob, len(blob)) if blob else None
        self.check(self.lib.qc_graph_from_json(json.dumps(doc).encode(), buf, len(blob),
                                               C.byref(h)))
        return Graph(self, h)

    def _bind(self, name, res, args):
        """Bind an entry point the reference build may not export (the
        serialize.hpp files are B200-library only)."""
        fn = getattr(self.lib, name)
        fn.restype, fn.argtypes = res, args
        return fn

    # -- files (serialize.hpp) ------------------------------------------
    def load_graph(self, path) -> "Graph":
        h = C.c_void_p()
        fn = self._bind("qc_graph_load", C.c_int, [C.c_char_p, C.POINTER(_P)])
        self.check(fn(str(path).encode(), C.byref(h)))
        return Graph(self, h)

    def load_dataset(self, path) -> "Dataset":
        h, n = C.c_void_p(), C.c_int64()
        fn = self._bind("qc_dataset_load", C.c_int, [C.c_char_p, C.POINTER(_P), C.POINTER(C.c_int64)])
        self.check(fn(str(path).encode(), C.byref(h), C.byref(n)))
        return Dataset(self, h, n.value)

    def fixtures_write_all(self, directory):
        """quantc::fixtures::write_all (fixtures.hpp; B200 library)."""
        fn = self._bind("qc_fixtures_write_all", C.c_int, [C.c_char_p])
        self.check(fn(str(directory).encode()))

    def fixtures_verify_committed(self, directory):
        """quantc::fixtures::verify_committed: raises on any byte mismatch."""
        fn = self._bind("qc_fixtures_verify_committed", C.c_int, [C.c_char_p])
        self.check(fn(str(directory).encode()))

    def load_stats(self, path) -> "CalibrationStats":
        h = C.c_void_p()
        fn = self._bind("qc_stats_load", C.c_int, [C.c_char_p, C.POINTER(_P)])
        self.check(fn(str(path).encode(), C.byref(h)))
        return CalibrationStats(self, h)

    def fnv1a64(self, data: bytes, seed: int = 1469598103934665603) -> int:
        out = C.c_uint64()
        fn = self._bind("qc_fnv1a64", C.c_int, [C.c_char_p, _SZ, C.c_uint64,
                                                 C.POINTER(C.c_uint64)])
        self.check(fn(data, len(data), seed, C.byref(out)))
        return out.value

    def parse_spec(self, text) -> "HardwareSpec":
        if isinstance(text, dict):
            text = json.dumps(text)
        h = C.c_void_p()
        self.check(self.lib.qc_spec_parse(text.encode(), C.byref(h)))
        return HardwareSpec(self, h)

    def generate_topology(self, g: "Graph", spec: "HardwareSpec") -> "Topology":
        h = C.c_void_p()
        self.check(self.lib.qc_generate_topology(g.h, spec.h, C.byref(h)))
        return Topology(self, h, g)

    def insert_simulated_quantize(self, g: "Graph", t: "Topology") -> "Graph":
        h = C.c_void_p()
        self.check(self.lib.qc_insert_simulated_quantize(g.h, t.h, C.byref(h)))
        return Graph(self, h)

    def simulated_edge_indices(self, g: "Graph", t: "Topology") -> List[int]:
        return self._vec(self.lib.qc_simulated_edge_indices, (g.h, t.h), C.c_int).tolist()

    def searchable_edge_indices(self, t: "Topology") -> List[int]:
        return self._vec(self.lib.qc_searchable_edge_indices, (t.h,), C.c_int).tolist()

    def dataset(self, samples: np.ndarray, labels=None) -> "Dataset":
        """samples: [N, *sample_shape] float32 (one graph input per sample)."""
        x = np.ascontiguousarray(samples, dtype=np.float32)
        shape, sp = _arr(x.shape[1:], C.c_int64)
        lab, lp = (None, None) if labels is None else _arr(labels, C.c_int64)
        h = C.c_void_p()
        self.check(self.lib.qc_dataset_create(x.ctypes.data_as(_PF), x.shape[0], sp,
                                              len(x.shape) - 1, lp, C.byref(h)))
        return Dataset(self, h, x.shape[0])

    # -- simulate (simulate.hpp) ----------------------------------------
    def compute_scale(self, threshold, bit, sign) -> float:
        out = C.c_double()
        self.check(self.lib.qc_compute_scale(threshold, bit, sign, C.byref(out)))
        return out.value

    def quant_bounds(self, bit, sign):
        lo, hi = C.c_int64(), C.c_int64()
        self.check(self.lib.qc_quant_bounds(bit, sign, C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    def simulated_quantize_value(self, x: float, p: QParams) -> float:
        out = C.c_float()
        self.check(self.lib.qc_simulated_quantize_value(x, C.byref(p), C.byref(out)))
        return out.value

    def simulated_quantize(self, x: np.ndarray, p: QParams) -> np.ndarray:
        a = np.ascontiguousarray(x, dtype=np.float32)
        out = np.empty_like(a)
        self.check(self.lib.qc_simulated_quantize(a.ctypes.data_as(_PF), a.size, C.byref(p),
                                                  out.ctypes.data_as(_PF)))
        return out

    def asymmetric_zero_point(self, min_value, range_threshold, bit) -> int:
        out = C.c_int64()
        self.check(self.lib.qc_asymmetric_zero_point(min_value, range_threshold, bit,
                                                     C.byref(out)))
        return out.value

    def noop_params(self) -> QParams:
        p = QParams()
        self.check(self.lib.qc_noop_params(C.byref(p)))
        return p

    # -- calibration (calibration.hpp) ----------------------------------
    def collect_stats(self, g: "Graph", d: "Dataset", bins=2048, edges=(), workers=0):
        e, ep = _arr(list(edges) or [0], C.c_int)
        h = C.c_void_p()
        self.check(self.lib.qc_collect_stats(g.h, d.h, bins, ep, len(edges), workers,
                                             C.byref(h)))
        return CalibrationStats(self, h)

    def make_stats(self, per_edge: Dict[int, dict]) -> "CalibrationStats":
        h = C.c_void_p()
        self.check(self.lib.qc_stats_create(C.byref(h)))
        st = CalibrationStats(self, h)
        for k, e in per_edge.items():
            c, cp = _arr(e["counts"], C.c_int64)
            self.check(self.lib.qc_stats_set_edge(h, k, e["min"], e["max"], e["absmax"],
                                                  e.get("sample_count", 1), cp, len(c)))
        return st

    def threshold_max(self, absmax) -> float:
        out = C.c_double()
        self.check(self.lib.qc_threshold_max(absmax, C.byref(out)))
        return out.value

    def threshold_quantile(self, counts, absmax, q) -> float:
        c, cp = _arr(counts, C.c_int64)
        out = C.c_double()
        self.check(self.lib.qc_threshold_quantile(cp, len(c), absmax, q, C.byref(out)))
        return out.value

    def threshold_kl(self, counts, absmax, target_bit) -> float:
        c, cp = _arr(counts, C.c_int64)
        out = C.c_double()
        self.check(self.lib.qc_threshold_kl(cp, len(c), absmax, target_bit, C.byref(out)))
        return out.value

    def round_pow2(self, t) -> float:
        out = C.c_double()
        self.check(self.lib.qc_round_pow2(t, C.byref(out)))
        return out.value

    # -- interpreter (interpreter.hpp) ----------------------------------
    @staticmethod
    def _binding(binding):
        if not binding:
            return None, None, 0, None
        ids = np.array(list(binding.keys()), dtype=np.int64)
        params = (QParams * len(binding))(*binding.values())
        return ids, params, len(binding), ids.ctypes.data_as(_PI64)

    def eval_fp32(self, g: "Graph", x: np.ndarray, binding=None) -> np.ndarray:
        a = np.ascontiguousarray(x, dtype=np.float32)
        sh, shp = _arr(a.shape, C.c_int64)
        ids, params, nb, idp = self._binding(binding)
        cap = 1 << 16
        while True:
            out = np.empty(cap, np.float32)
            n = C.c_size_t()
            oshape = np.zeros(8, np.int64)
            ond = C.c_int()
            rc = self.lib.qc_eval_fp32(g.h, a.ctypes.data_as(_PF), shp, a.ndim, idp, params, nb,
                                       out.ctypes.data_as(_PF), cap, C.byref(n),
                                       oshape.ctypes.data_as(_PI64), C.byref(ond))
            if rc == 10 and n.value > cap:
                cap = n.value
                continue
            self.check(rc)
            return out[: n.value].reshape(oshape[: ond.value]).copy()

    def eval_fp32_values(self, g: "Graph", x: np.ndarray, nodes: Sequence[int]) -> np.ndarray:
        a = np.ascontiguousarray(x, dtype=np.float32)
        sh, shp = _arr(a.shape, C.c_int64)
        nd, ndp = _arr(nodes, C.c_int64)
        return self._vec(self.lib.qc_eval_fp32_values,
                         (g.h, a.ctypes.data_as(_PF), shp, a.ndim, ndp, len(nd)), C.c_float,
                         first_cap=1 << 20)

    def eval_int(self, g: "Graph", x: np.ndarray, trap=False):
        a = np.ascontiguousarray(x, dtype=np.float32)
        sh, shp = _arr(a.shape, C.c_int64)
        cap = 1 << 16
        while True:
            out = np.empty(cap, np.int32)
            n = C.c_size_t()
            dt = C.c_int()
            rc = self.lib.qc_eval_int(g.h, a.ctypes.data_as(_PF), shp, a.ndim, 1 if trap else 0,
                                      out.ctypes.data_as(C.POINTER(C.c_int32)), cap,
                                      C.byref(n), C.byref(dt))
            if rc == 10 and n.value > cap:
                cap = n.value
                continue
            self.check(rc)
            r = out[: n.value].copy()
            return (r.view(np.float32) if dt.value == F32 else r), dt.value

    def predict_top1(self, g: "Graph", d: "Dataset", workers=0, binding=None) -> np.ndarray:
        ids, params, nb, idp = self._binding(binding)
        return self._vec(self.lib.qc_predict_top1, (g.h, d.h, workers, idp, params, nb),
                         C.c_int64, first_cap=max(1, d.n))

    def fused_status(self, g: "Graph", binding=None) -> str:
        """'' when the fused int8 tcgen05 engine runs g under `binding`, else
        the reason (B200 extension)."""
        ids, params, nb, idp = self._binding(binding)
        s = C.c_void_p()
        fn = self._bind("qc_fused_status", C.c_int,
                        [_P, _PI64, C.POINTER(QParams), _SZ, _PSTR])
        self.check(fn(g.h, idp, params, nb, C.byref(s)))
        return self._take_string(s)

    def predict_scores(self, g: "Graph", d: "Dataset", binding=None) -> np.ndarray:
        """B200 extension (quantc/device.hpp): the fp32 output rows behind
        predict_top1 under the active engine mode, shape [samples, per]."""
        fn = self.lib.qc_predict_scores
        fn.restype = C.c_int
        fn.argtypes = [_P, _P, _PI64, C.POINTER(QParams), _SZ, C.POINTER(C.c_float), _SZ, _PSZ,
                       _PI64]
        ids, params, nb, idp = self._binding(binding)
        per = C.c_int64(0)
        n = C.c_size_t(0)
        cap = max(1, d.n) * 1024
        while True:
            buf = np.zeros(cap, np.float32)
            rc = fn(g.h, d.h, idp, params, nb, buf.ctypes.data_as(C.POINTER(C.c_float)), cap,
                    C.byref(n), C.byref(per))
            if rc == 10 and n.value > cap:
                cap = n.value
                continue
            self.check(rc)
            return buf[: n.value].reshape(d.n, -1)

    def realize(self, sim_g: "Graph", strategy: dict, spec) -> "Graph":
        """B200 extension: realize() (SPEC.md realize module) of sim_g under a
        strategy (CandidateEvaluator.strategy_for's dict)."""
        fn = self.lib.qc_realize
        fn.restype = C.c_int
        fn.argtypes = [_P, C.c_char_p, _P, C.POINTER(_P)]
        h = _P()
        doc = json.dumps({str(k): v for k, v in strategy.items()}).encode()
        self.check(fn(sim_g.h, doc, spec.h, C.byref(h)))
        return Graph(self, h)

    def requantize_params(self, s_in: float, s_out: float):
        m, sh = C.c_int32(), C.c_int()
        fn = self._bind("qc_requantize_params", C.c_int,
                        [C.c_double, C.c_double, C.POINTER(C.c_int32), C.POINTER(C.c_int)])
        self.check(fn(s_in, s_out, C.byref(m), C.byref(sh)))
        return m.value, sh.value

    def choose_storage_dtype(self, bit: int, candidates: Sequence[str], sign: int = 1) -> str:
        buf = C.create_string_buffer(32)
        fn = self._bind("qc_choose_storage_dtype", C.c_int,
                        [C.c_int, C.c_char_p, C.c_int, C.c_char_p, C.c_size_t])
        self.check(fn(bit, ",".join(candidates).encode(), sign, buf, 32))
        return buf.value.decode()

    def rewrite_clip(self, min_f, max_f, s_out, zero_point, storage="int8"):
        lo, hi = C.c_int64(), C.c_int64()
        fn = self._bind("qc_rewrite_clip", C.c_int,
                        [C.c_double, C.c_double, C.c_double, C.c_int64, C.c_char_p,
                         C.POINTER(C.c_int64), C.POINTER(C.c_int64)])
        self.check(fn(min_f, max_f, s_out, zero_point, storage.encode(), C.byref(lo),
                      C.byref(hi)))
        return lo.value, hi.value

    # -- search (search.hpp) --------------------------------------------
    def evaluator(self, sim_g, spec, topo, thresholds: Dict[int, float], stats, calib,
                  min_bit=4, workers=0) -> "CandidateEvaluator":
        ks, kp = _arr(list(thresholds.keys()), C.c_int)
        vs, vp = _arr(list(thresholds.values()), C.c_double)
        h = C.c_void_p()
        self.check(self.lib.qc_evaluator_create(sim_g.h, spec.h, topo.h, kp, vp, len(ks),
                                                stats.h, calib.h, min_bit, workers,
                                                C.byref(h)))
        return CandidateEvaluator(self, h, keep=(sim_g, spec, topo, stats, calib))

    def search(self, method: str, space: "SearchSpace",
               loss: Optional[Callable[[List[int]], float]] = None,
               evaluator: Optional["CandidateEvaluator"] = None, **kw) -> "SearchResult":
        code = {"greedy": 0, "anneal": 1, "random": 2, "exhaustive": 3}[method]
        p = SearchParams(kw.get("rounds", 1), kw.get("tol", 0.0), kw.get("steps", 1),
                         kw.get("t0", 0.1), kw.get("decay", 0.995), kw.get("seed", 0),
                         kw.get("n", 1), kw.get("cap", 100000))
        e, ep = _arr(space.edges or [0], C.c_int)
        lo, lop = _arr(space.lo or [0], C.c_int)
        hi, hip = _arr(space.hi or [0], C.c_int)
        n = len(space.edges)
        errors: List[BaseException] = []

        def _cb(cand, ns, user, out):
            try:
                out[0] = float(loss([cand[i] for i in range(ns)]))
                return 0
            except BaseException as ex:  # surfaced after the call
                errors.append(ex)
                return 1

        cb = LOSS_FN(_cb) if loss is not None else LOSS_FN()
        best = np.zeros(max(n, 1), np.int32)
        bl = C.c_double()
        ne = C.c_int64()
        tr = C.c_void_p()
        rc = self.lib.qc_search(code, ep, lop, hip, n, cb, None,
                                evaluator.h if evaluator is not None else None, C.byref(p),
                                best.ctypes.data_as(_PI), C.byref(bl), C.byref(ne),
                                C.byref(tr))
        if errors:
            raise errors[0]
        self.check(rc)
        trace = json.loads(self._take_string(tr))
        return SearchResult(best[:n].tolist(), bl.value, ne.value, trace)

    def search_batched(self, method: str, space: "SearchSpace",
                       losses: Optional[Callable[[List[List[int]]], Sequence[float]]] = None,
                       evaluator: Optional["CandidateEvaluator"] = None,
                       comm: Optional["Comm"] = None, mode: str = "local", width: int = 4,
                       **kw) -> "SearchResult":
        """search.hpp *_batched (B200 extension): the speculative batched
        searches.  Results and traces equal search(); `losses` is a batch
        callable, else the evaluator is used with mode "local", "samples"
        (counts all-reduced over comm) or "candidates" (batches split over
        comm's ranks).  Returns a SearchResult with .speculation =
        (batches, evaluated, committed)."""
        code = {"greedy": 0, "anneal": 1, "random": 2, "exhaustive": 3}[method]
        lmode = {"local": 0, "samples": 1, "candidates": 2}[mode]
        p = SearchParams(kw.get("rounds", 1), kw.get("tol", 0.0), kw.get("steps", 1),
                         kw.get("t0", 0.1), kw.get("decay", 0.995), kw.get("seed", 0),
                         kw.get("n", 1), kw.get("cap", 100000))
        e, ep = _arr(space.edges or [0], C.c_int)
        lo, lop = _arr(space.lo or [0], C.c_int)
        hi, hip = _arr(space.hi or [0], C.c_int)
        n = len(space.edges)
        errors: List[BaseException] = []

        def _cb(cands, nc, ns, user, out):
            try:
                a = np.ctypeslib.as_array(cands, shape=(nc * ns,)).reshape(nc, ns) if nc * ns \
                    else np.zeros((nc, ns), np.int32)
                v = [float(x) for x in losses(a.tolist())]
                if len(v) != nc:
                    raise ValueError("batch loss returned the wrong count")
                for i, x in enumerate(v):
                    out[i] = x
                return 0
            except BaseException as ex:  # surfaced after the call
                errors.append(ex)
                return 1

        fn = self._bind("qc_search_batched", C.c_int,
                        [C.c_int, _PI, _PI, _PI, _SZ, BATCH_LOSS_FN, _P, _P, _P, C.c_int,
                         C.POINTER(SearchParams), C.c_int, _PI, _PD, _PI64, _PSTR, _PI64])
        cb = BATCH_LOSS_FN(_cb) if losses is not None else BATCH_LOSS_FN()
        best = np.zeros(max(n, 1), np.int32)
        bl = C.c_double()
        ne = C.c_int64()
        tr = C.c_void_p()
        st = np.zeros(3, np.int64)
        rc = fn(code, ep, lop, hip, n, cb, None,
                evaluator.h if evaluator is not None else None,
                comm.h if comm is not None else None, lmode, C.byref(p), width,
                best.ctypes.data_as(_PI), C.byref(bl), C.byref(ne), C.byref(tr),
                st.ctypes.data_as(_PI64))
        if errors:
            raise errors[0]
        self.check(rc)
        trace = json.loads(self._take_string(tr))
        r = SearchResult(best[:n].tolist(), bl.value, ne.value, trace)
        r.speculation = tuple(int(x) for x in st)
        return r

    # -- communicators (comm.hpp; B200 extension) -------------------------
    def comm_local(self) -> "Comm":
        h = C.c_void_p()
        self.check(self._bind("qc_comm_local", C.c_int, [C.POINTER(_P)])(C.byref(h)))
        return Comm(self, h)

    def nccl_unique_id(self) -> bytes:
        buf = C.create_string_buffer(128)
        self.check(self._bind("qc_comm_nccl_unique_id", C.c_int, [C.c_char_p])(buf))
        return buf.raw

    def comm_nccl(self, rank: int, world: int, uid: bytes) -> "Comm":
        h = C.c_void_p()
        fn = self._bind("qc_comm_nccl", C.c_int, [C.c_int, C.c_int, C.c_char_p, C.POINTER(_P)])
        self.check(fn(rank, world, C.create_string_buffer(uid, 128), C.byref(h)))
        return Comm(self, h)

    def comm_torch(self, group=None) -> "Comm":
        """A communicator whose collectives are torch.distributed calls on
        `group` (any backend; gloo in the CPU tests)."""
        import torch
        import torch.distributed as dist
        dev = (torch.device("cuda", torch.cuda.current_device())
               if dist.get_backend(group) == "nccl" else torch.device("cpu"))
        world = dist.get_world_size(group)

        def sum_i64(data, n, user):
            try:
                t = torch.from_numpy(np.ctypeslib.as_array(data, shape=(n,)).copy()).to(dev)
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
                np.ctypeslib.as_array(data, shape=(n,))[:] = t.cpu().numpy()
                return 0
            except BaseException:
                return 1

        def minmax(data, n, op, user):
            try:
                t = torch.from_numpy(np.ctypeslib.as_array(data, shape=(n,)).copy()).to(dev)
                dist.all_reduce(t, op=dist.ReduceOp.MIN if op == 0 else dist.ReduceOp.MAX,
                                group=group)
                np.ctypeslib.as_array(data, shape=(n,))[:] = t.cpu().numpy()
                return 0
            except BaseException:
                return 1

        def gather(send, n, recv, user):
            try:
                t = torch.from_numpy(np.ctypeslib.as_array(send, shape=(n,)).copy()).to(dev)
                outs = [torch.empty_like(t) for _ in range(world)]
                dist.all_gather(outs, t, group=group)
                np.ctypeslib.as_array(recv, shape=(n * world,))[:] = \
                    torch.cat(outs).cpu().numpy()
                return 0
            except BaseException:
                return 1

        cbs = (COMM_SUM_FN(sum_i64), COMM_F64_FN(minmax), COMM_GATHER_FN(gather))
        fn = self._bind("qc_comm_callbacks", C.c_int,
                        [C.c_int, C.c_int, COMM_SUM_FN, COMM_F64_FN, COMM_GATHER_FN, _P,
                         C.POINTER(_P)])
        h = C.c_void_p()
        self.check(fn(dist.get_rank(group), world, *cbs, None, C.byref(h)))
        return Comm(self, h, keep=cbs)

    def collect_stats_dist(self, g: "Graph", shard: "Dataset", comm: "Comm", bins=2048,
                           edges=()) -> "CalibrationStats":
        """distributed.hpp collect_stats: this rank's shard, merged over comm."""
        e, ep = _arr(list(edges) or [0], C.c_int)
        h = C.c_void_p()
        fn = self._bind("qc_collect_stats_dist", C.c_int,
                        [_P, _P, _P, C.c_int, _PI, _SZ, C.POINTER(_P)])
        self.check(fn(g.h, shard.h, comm.h, bins, ep, len(edges), C.byref(h)))
        return CalibrationStats(self, h)

    def space_size(self, space: "SearchSpace") -> int:
        lo, lop = _arr(space.lo or [0], C.c_int)
        hi, hip = _arr(space.hi or [0], C.c_int)
        s = C.c_void_p()
        self.check(self.lib.qc_space_size(lop, hip, len(space.lo), C.byref(s)))
        return int(self._take_string(s))


class _Handle:
    _free = ""

    def __init__(self, q: Quantc, h):
        self.q, self.h = q, h

    def __del__(self):
        try:
            if self.h:
                getattr(self.q.lib, self._free)(self.h)
                self.h = None
        except Exception:
            pass


class Graph(_Handle):
    _free = "qc_graph_free"

    def to_json(self) -> dict:
        s = C.c_void_p()
        self.q.check(self.q.lib.qc_graph_to_json(self.h, C.byref(s)))
        return json.loads(self.q._take_string(s))

    def blob(self) -> bytes:
        """Payload bytes matching to_json()'s offsets (qc_graph_blob)."""
        fn = self.q.lib.qc_graph_blob
        fn.restype = C.c_int
        fn.argtypes = [_P, C.c_void_p, _SZ, _PSZ]
        n = C.c_size_t()
        rc = fn(self.h, None, 0, C.byref(n))
        if rc not in (0, 10):
            self.q.check(rc)
        buf = C.create_string_buffer(max(1, n.value))
        self.q.check(fn(self.h, buf, n.value, C.byref(n)))
        return buf.raw[: n.value]

    def save(self, path):
        """Graph file + '<stem>.bin' sidecar (serialize.hpp save_graph)."""
        fn = self.q._bind("qc_graph_save", C.c_int, [_P, C.c_char_p])
        self.q.check(fn(self.h, str(path).encode()))

    def fingerprint(self) -> int:
        out = C.c_uint64()
        fn = self.q._bind("qc_fingerprint_graph", C.c_int, [_P, C.POINTER(C.c_uint64)])
        self.q.check(fn(self.h, C.byref(out)))
        return out.value

    def copy_to(self, q: "Quantc") -> "Graph":
        """The same graph inside another library exporting this ABI (JSON +
        blob round trip), e.g. a realized graph handed to the reference."""
        return q.graph(self.to_json(), self.blob())

    def num_nodes(self) -> int:
        n = C.c_size_t()
        self.q.check(self.q.lib.qc_graph_num_nodes(self.h, C.byref(n)))
        return n.value

    def validate(self) -> list:
        s = C.c_void_p()
        self.q.check(self.q.lib.qc_validate_graph(self.h, C.byref(s)))
        return json.loads(self.q._take_string(s))

    def traversal_order(self) -> List[int]:
        return self.q._vec(self.q.lib.qc_traversal_order, (self.h,), C.c_int64).tolist()

    def edge_order(self) -> List[tuple]:
        n = C.c_size_t()
        cap = 4096
        while True:
            buf = np.zeros(cap, np.int64)
            rc = self.q.lib.qc_edge_order(self.h, buf.ctypes.data_as(_PI64), cap, C.byref(n))
            if rc == 10 and 4 * n.value > cap:
                cap = 4 * n.value
                continue
            self.q.check(rc)
            return [tuple(buf[4 * i: 4 * i + 4].tolist()) for i in range(n.value)]


class HardwareSpec(_Handle):
    _free = "qc_spec_free"

    def serialize(self) -> str:
        s = C.c_void_p()
        self.q.check(self.q.lib.qc_spec_serialize(self.h, C.byref(s)))
        return self.q._take_string(s)

    def classify_op(self, op: str) -> str:
        c = C.c_int()
        self.q.check(self.q.lib.qc_classify_op(self.h, op.encode(), C.byref(c)))
        return ["float_only", "integer_only", "mixed"][c.value]

    def candidate_dtypes(self, op: str, port: int) -> List[str]:
        v = self.q._vec(self.q.lib.qc_candidate_dtypes, (self.h, op.encode(), port), C.c_int)
        return [DTYPE_NAMES[int(x)] for x in v]

    def match_signature(self, op: str, bits, signs):
        b, bp = _arr(bits, C.c_int)
        s, sp = _arr(signs, C.c_int)
        found = C.c_int()
        ins = np.zeros(8, np.int32)
        out = C.c_int()
        self.q.check(self.q.lib.qc_match_signature(self.h, op.encode(), bp, sp, len(b),
                                                   C.byref(found), ins.ctypes.data_as(_PI),
                                                   C.byref(out)))
        if not found.value:
            return None
        return [DTYPE_NAMES[int(x)] for x in ins[: len(b)]], DTYPE_NAMES[out.value]


class Topology(_Handle):
    _free = "qc_topology_free"

    def __init__(self, q, h, g):
        super().__init__(q, h)
        self._g = g

    def dump(self) -> dict:
        s = C.c_void_p()
        self.q.check(self.q.lib.qc_dump_topology(self._g.h, self.h, C.byref(s)))
        return json.loads(self.q._take_string(s))

    def qv(self) -> List[int]:
        return self.q._vec(self.q.lib.qc_topology_qv, (self.h,), C.c_int64).tolist()


class Dataset(_Handle):
    _free = "qc_dataset_free"

    def __init__(self, q, h, n):
        super().__init__(q, h)
        self.n = n


class CalibrationStats(_Handle):
    _free = "qc_stats_free"

    def edges(self) -> List[int]:
        return self.q._vec(self.q.lib.qc_stats_edges, (self.h,), C.c_int).tolist()

    def get(self, edge: int) -> dict:
        mn, mx, am, sc = C.c_double(), C.c_double(), C.c_double(), C.c_int64()
        counts = self.q._vec(
            lambda *a: self.q.lib.qc_stats_get(self.h, edge, C.byref(mn), C.byref(mx),
                                               C.byref(am), C.byref(sc), *a),
            (), C.c_int64, first_cap=4096)
        return {"min": mn.value, "max": mx.value, "absmax": am.value,
                "sample_count": sc.value, "counts": counts}

    def per_edge(self) -> Dict[int, dict]:
        return {k: self.get(k) for k in self.edges()}

    def save(self, path):
        """Stats file (serialize.hpp save_stats)."""
        fn = self.q._bind("qc_stats_save", C.c_int, [_P, C.c_char_p])
        self.q.check(fn(self.h, str(path).encode()))

    def estimate_thresholds(self, method="quantile", quantile=0.99, kl_bits=8,
                            pow2=False) -> Dict[int, float]:
        m = {"max": 0, "quantile": 1, "kl": 2}[method]
        cap = 4096
        ks = np.zeros(cap, np.int32)
        vs = np.zeros(cap, np.float64)
        n = C.c_size_t()
        self.q.check(self.q.lib.qc_estimate_thresholds(self.h, m, quantile, kl_bits,
                                                       1 if pow2 else 0,
                                                       ks.ctypes.data_as(_PI),
                                                       vs.ctypes.data_as(_PD), cap,
                                                       C.byref(n)))
        return {int(k): float(v) for k, v in zip(ks[: n.value], vs[: n.value])}


@dataclass
class SearchSpace:
    edges: List[int] = field(default_factory=list)
    lo: List[int] = field(default_factory=list)
    hi: List[int] = field(default_factory=list)

    def all_hi(self):
        return list(self.hi)

    def all_lo(self):
        return list(self.lo)


@dataclass
class SearchResult:
    best: List[int]
    best_loss: float
    evaluations: int
    trace: dict


class Comm(_Handle):
    """A quantc::Communicator (comm.hpp)."""
    _free = "qc_comm_free"

    def __init__(self, q, h, keep=()):
        q._bind("qc_comm_free", None, [_P])
        super().__init__(q, h)
        self._keep = keep


class CandidateEvaluator(_Handle):
    _free = "qc_evaluator_free"

    def __init__(self, q, h, keep=()):
        super().__init__(q, h)
        self._keep = keep

    def space(self) -> SearchSpace:
        cap = 4096
        e, lo, hi = (np.zeros(cap, np.int32) for _ in range(3))
        n = C.c_size_t()
        self.q.check(self.q.lib.qc_evaluator_space(self.h, e.ctypes.data_as(_PI),
                                                   lo.ctypes.data_as(_PI),
                                                   hi.ctypes.data_as(_PI), cap, C.byref(n)))
        k = n.value
        return SearchSpace(e[:k].tolist(), lo[:k].tolist(), hi[:k].tolist())

    def reference_predictions(self) -> np.ndarray:
        return self.q._vec(self.q.lib.qc_evaluator_refs, (self.h,), C.c_int64, 4096)

    def bind(self, cand) -> Dict[int, QParams]:
        c, cp = _arr(cand, C.c_int)
        cap = 8192
        ids = np.zeros(cap, np.int64)
        ps = (QParams * cap)()
        n = C.c_size_t()
        self.q.check(self.q.lib.qc_evaluator_bind(self.h, cp, len(c), ids.ctypes.data_as(_PI64),
                                                  ps, cap, C.byref(n)))
        return {int(ids[i]): ps[i] for i in range(n.value)}

    def loss(self, cand) -> float:
        c, cp = _arr(cand, C.c_int)
        out = C.c_double()
        self.q.check(self.q.lib.qc_evaluator_loss(self.h, cp, len(c), C.byref(out)))
        return out.value

    def losses(self, cands) -> np.ndarray:
        a = np.ascontiguousarray(np.asarray(cands, dtype=np.int32))
        out = np.zeros(a.shape[0], np.float64)
        self.q.check(self.q.lib.qc_evaluator_losses(self.h, a.ctypes.data_as(_PI), a.shape[0],
                                                    a.shape[1], out.ctypes.data_as(_PD)))
        return out

    def scores(self, cands, group: int = 0) -> np.ndarray:
        """fp32 output rows of each candidate's forward over the calibration
        set, [n_cands, N, per_sample] (B200 extension), `group` candidates per
        grouped launch (0: the default)."""
        a = np.ascontiguousarray(np.asarray(cands, dtype=np.int32))
        fn = self.q._bind("qc_evaluator_scores", C.c_int,
                          [_P, _PI, _SZ, _SZ, C.c_int, _PF, _SZ, _PSZ, _PI64])
        n = len(self.reference_predictions())
        cap = 1 << 16
        while True:
            out = np.zeros(cap, np.float32)
            k = C.c_size_t()
            per = C.c_int64()
            rc = fn(self.h, a.ctypes.data_as(_PI), a.shape[0], a.shape[1], group,
                    out.ctypes.data_as(_PF), cap, C.byref(k), C.byref(per))
            if rc == 10 and k.value > cap:
                cap = k.value
                continue
            self.q.check(rc)
            return out[:k.value].reshape(a.shape[0], n, per.value)

    def strategy_for(self, cand) -> dict:
        c, cp = _arr(cand, C.c_int)
        s = C.c_void_p()
        self.q.check(self.q.lib.qc_evaluator_strategy(self.h, cp, len(c), C.byref(s)))
        return {int(k): v for k, v in json.loads(self.q._take_string(s)).items()}

    def evaluations(self) -> int:
        out = C.c_int64()
        self.q.check(self.q.lib.qc_evaluator_evaluations(self.h, C.byref(out)))
        return out.value


# ---- library discovery -----------------------------------------------------
_PKG = os.path.dirname(os.path.abspath(__file__))
# QUANTC_B200_LIB: an alternative build of the same library (A/B experiments)
B200_LIB = os.environ.get("QUANTC_B200_LIB") or os.path.join(_PKG, "libquantc_b200.so")
_loaded: Dict[str, Quantc] = {}


def load(path: str) -> Quantc:
    if path not in _loaded:
        _loaded[path] = Quantc(path)
    return _loaded[path]


def load_b200() -> Quantc:
    """The B200 implementation. Fails loudly when the extension is missing:
    there is no CPU fallback for the product path."""
    if not os.path.exists(B200_LIB):
        raise ImportError(f"{B200_LIB} is not built; run __graft_entry__.build()")
    return load(B200_LIB)
