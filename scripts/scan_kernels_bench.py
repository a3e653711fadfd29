"""HBM roofline evidence (QUANTC_HIST_REPS: replicated histogram copies) for the streaming kernels of the calibration path
(north star: "achieved HBM GB/s against the B200 peak for simulated-quantize
and the histograms"): standalone sim-quant (8 B/elem), min/max pass (4 B/elem),
histogram pass (4 B/elem) on 256 Mi fp32 elements (1 GiB, >> L2), CUDA-event
timed on the engine stream, plus the KL sweep over 191 edges x 2048 bins (the
ResNet-50 calibration).  Prints one JSON line.  Run under ncu for the DRAM
counters (profiles/r1_scan_kernels_ncu.md)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_14949_b200 import cuda_ops, quantc as Q  # noqa: E402

ops = cuda_ops.load()
n = int(os.environ.get("N_ELEMS", 1 << 28))
x = torch.randn(n, device="cuda")
y = torch.empty_like(x)
p = Q.QParams.make(2.0, 8, 1, Q.I8)
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "MEASURED_PEAKS.json")))
hbm = peaks["hbm_gbs"]


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


out = {"elements": n}
t = timed(lambda: ops.sim_quant(x, p, out=y))
out["sim_quant"] = {"s": t, "GB/s": 8 * n / t / 1e9, "frac": 8 * n / t / 1e9 / hbm}
t = timed(lambda: ops.minmax(x))
out["minmax"] = {"s": t, "GB/s": 4 * n / t / 1e9, "frac": 4 * n / t / 1e9 / hbm}
counts = torch.zeros(2048, dtype=torch.int64, device="cuda")
t = timed(lambda: ops.histogram(x, 6.0, 2048, counts=counts))
out["histogram_2048"] = {"s": t, "GB/s": 4 * n / t / 1e9, "frac": 4 * n / t / 1e9 / hbm}
# a relu edge: half the elements are exact zeros (bin 0), the rest half-normal
xr = torch.relu(x)
t = timed(lambda: ops.histogram(xr, 6.0, 2048, counts=counts))
out["histogram_2048_relu"] = {"s": t, "GB/s": 4 * n / t / 1e9, "frac": 4 * n / t / 1e9 / hbm}
h = torch.randint(0, 1000, (191, 2048), dtype=torch.int64, device="cuda")
t = timed(lambda: ops.kl_sweep(h, 8), reps=3)
out["kl_sweep_191x2048"] = {"s": t, "edges_per_s": 191 / t}
out["hbm_peak_GBs"] = hbm
print(json.dumps(out))
