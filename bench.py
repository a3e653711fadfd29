"""bench.py — HAGO calibrate-and-search hot path on B200.

Metric (BASELINE.json): int8 simulated-quantized ResNet-50 images/s; search
candidates/s.  One step = one candidate evaluation (bind -> sim-quant int8
forward of the calibration batch -> top-1 agreement with the fp32
references) over a batch of B synthetic 224x224 images per GPU, exactly the
inner loop of CandidateEvaluator::loss (reference search.cpp:421-428).  The K
timed steps run through the search's batch API, CandidateEvaluator::losses
over the K candidates (one C-ABI call, one all-reduce of the K counts); the
one-call-per-candidate time is reported beside it as `per_call`.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--batch B]
  python bench.py --impl reference ...   (the reference CPU implementation)

N > 1 runs under torchrun, one rank per GPU: each rank holds its own shard of
B calibration images (weak scaling) and the per-candidate agreement counts are
all-reduced with NCCL (the search's only data-path collective).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

from paper_2103_14949_b200 import fixtures as F  # noqa: E402
from paper_2103_14949_b200 import quantc as Q  # noqa: E402

METRIC = "int8 sim-quant ResNet-50 images/sec"
REF_LIB = os.path.join(REPO, "oracle", "_ref", "libquantc_ref.so")


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.samples = gpu, []
        self._proc = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        try:
            for line in self._proc.stdout:
                line = line.strip()
                if line:
                    self.samples.append([v.strip() for v in line.split(",")])
        except Exception:
            pass

    def __enter__(self):
        try:
            # one long-lived nvidia-smi polling every 20 ms for the timed region
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t.start()
            time.sleep(0.05)
        except Exception:
            self._proc = None
        return self

    def __exit__(self, *a):
        if self._proc is not None:
            time.sleep(0.05)
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()
            self._t.join(timeout=5)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def build_pipeline(q, model, data, calib_stats=None):
    g = q.graph(model.doc, model.blob)
    spec = q.parse_spec(F.spec_fixture("int8_int32"))
    topo = q.generate_topology(g, spec)
    sim = q.insert_simulated_quantize(g, topo)
    ds = q.dataset(data)
    st = calib_stats if calib_stats is not None else q.collect_stats(
        g, ds, 2048, q.simulated_edge_indices(g, topo))
    # power-of-two thresholds: the int8 tensor-core path is bit-identical to
    # the reference (engine kAuto); quantile q=0.999
    thr = st.estimate_thresholds("quantile", quantile=0.999, pow2=True)
    return g, spec, topo, sim, ds, st, thr


def candidates(space, n, seed=0):
    """Greedy-style probes: all_hi with one slot decremented, cycling slots."""
    out = []
    hi = space.all_hi()
    for i in range(n):
        c = list(hi)
        s = (i * 7 + seed) % len(c)
        c[s] = max(space.lo[s], c[s] - 1 - (i % 3))
        out.append(c)
    return out


def random_candidates(space, n, seed=1):
    """Search-realistic candidates: every slot drawn independently (every
    layer's weight codes change between candidates, unlike the probes)."""
    rng = np.random.default_rng(seed)
    return [[int(rng.integers(lo, hi + 1)) for lo, hi in zip(space.lo, space.hi)]
            for _ in range(n)]


def cpu_reference_preds(model, data, threads, binding):
    """The reference CPU implementation (oracle/_ref, compiled from the
    reference sources) on this host: predict_top1 of the sim-quant graph under
    one candidate binding (the body of CandidateEvaluator::loss, reference
    search.cpp:421-428) over `data` with `threads` workers.  Returns
    (predictions, seconds)."""
    ref = Q.load(REF_LIB)
    g = ref.graph(model.doc, model.blob)
    spec = ref.parse_spec(F.spec_fixture("int8_int32"))
    sim = ref.insert_simulated_quantize(g, ref.generate_topology(g, spec))
    ds = ref.dataset(data)
    t0 = time.perf_counter()
    preds = ref.predict_top1(sim, ds, threads, binding)
    return preds, time.perf_counter() - t0


def _ref_binding(ref, model, threads):
    """Reference-only setup: calibrate on one image, bind one candidate."""
    one = model.data(1, seed=11)
    g, spec, topo, sim, ds, st, thr = build_pipeline(ref, model, one)
    ev = ref.evaluator(sim, spec, topo, thr, st, ds, 4, threads)
    return sim, ev, ev.space()


def run_reference(args):
    rank = _env_int("RANK", 0)
    if rank != 0:
        return 0
    if not os.path.exists(REF_LIB):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return 0
    model = F.resnet(50)
    threads = os.cpu_count() or 1
    sample = threads  # one image per host thread per step (the reference's parallel unit)
    ref = Q.load(REF_LIB)
    sim, ev, sp = _ref_binding(ref, model, threads)
    cands = candidates(sp, args.warmup + args.steps)
    ds = ref.dataset(model.data(sample, seed=11))
    # one step (one image per host thread) takes ~10 s here: keep the whole
    # run within a few minutes by timing at most ~150 s worth of the K steps
    # (the warm-up step sizes it); `steps` reports what was timed
    est = 0.0
    for i in range(args.warmup):
        t0 = time.perf_counter()
        ref.predict_top1(sim, ds, threads, ev.bind(cands[i]))
        est = time.perf_counter() - t0
    if args.warmup == 0:
        t0 = time.perf_counter()
        ref.predict_top1(sim, ds, threads, ev.bind(cands[0]))
        est = time.perf_counter() - t0
    steps = max(1, min(args.steps, int(150.0 / max(est, 1e-3))))
    t0 = time.perf_counter()
    for i in range(steps):
        ref.predict_top1(sim, ds, threads, ev.bind(cands[args.warmup + i]))
    dt = time.perf_counter() - t0
    args.steps = steps
    value = sample * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "images/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64/f32 (reference CPU)", "data": "synthetic",
        "config": {"workload": "resnet50 int8_int32 sim-quant candidate evaluation",
                   "model": "resnet50", "image": 224, "batch": sample,
                   "parallelism": f"{threads} host threads"},
        "cpu_baseline": {"value": value, "unit": "images/s", "cores": threads,
                         "kind": "reference",
                         "sample": f"{sample} images per step, {args.steps} candidates"},
        "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def traffic_probe(args):
    """Child of the traffic measurement: set up the bench pipeline, then run
    ONE grouped losses call over 4 candidates (the timed step's unit) between
    cudaProfilerStart/Stop, so ncu captures exactly that step's launches."""
    import torch
    from paper_2103_14949_b200 import cuda_ops
    b = Q.load_b200()
    cuda_ops.load()
    model = F.resnet(50)
    data = model.data(args.batch, seed=9)
    g, spec, topo, sim, ds, st, thr = build_pipeline(b, model, data)
    ev = b.evaluator(sim, spec, topo, thr, st, ds)
    cands = candidates(ev.space(), 8)
    ev.losses(cands[:4])  # warm: plan, weight-code cache, arenas
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    ev.losses(cands[4:8])
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    return 0


def measure_traffic(args, timeout=420):
    """DRAM bytes of the dominant kernel, measured in this run: ncu on a child
    that replays one grouped step (dram__bytes_read.sum + dram__bytes_write.sum
    and gpu__time_duration.sum per tc_conv_kernel launch).  None when ncu is
    unavailable or fails."""
    ncu = "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None
    cmd = [ncu, "--profile-from-start", "off", "--clock-control", "none", "--csv",
           "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "-k", "regex:tc_conv_kernel", sys.executable, os.path.abspath(__file__),
           "--traffic-probe", "--batch", str(args.batch)]
    try:
        out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout).stdout
    except Exception:
        return None
    import csv
    import io
    rows = [r for r in csv.reader(io.StringIO(out)) if len(r) > 10]
    if not rows:
        return None
    hdr = rows[0]
    try:
        i_id, i_name, i_val = hdr.index("ID"), hdr.index("Metric Name"), hdr.index("Metric Value")
        i_unit = hdr.index("Metric Unit")
    except ValueError:
        return None
    per = {}
    for r in rows[1:]:
        v = float(r[i_val].replace(",", ""))
        unit = r[i_unit]
        if r[i_name].startswith("dram__bytes"):
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        else:
            v *= {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1}.get(unit, 1)
        per.setdefault(r[i_id], {})[r[i_name]] = v
    launches = [d for d in per.values() if "gpu__time_duration.sum" in d]
    if not launches:
        return None
    dram = [d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
            for d in launches]
    return {"launches": len(launches), "dram_bytes_per_launch": sum(dram) / len(dram),
            "ncu_time_s_sum": sum(d["gpu__time_duration.sum"] for d in launches),
            "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over one "
                      "grouped 4-candidate step of this bench (child process, this run)"}


def _events(torch):
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def config_legs(b, torch, stream, batch, engine="auto"):
    """The other BASELINE configs as bounded side legs (device-timed on the
    engine stream; one GPU).  Each: calibrate on its images, bind, then time a
    losses() call over a few candidates.

    C2  ResNet-18 @224, batch 64, int8_int32, pow2 thresholds -> fused tcgen05 path
    C3  MobileNetV2 (width 1.0) @224, arm_vmlal_like with 8-bit codes (the
        (i8, i8) -> i16 accumulation signature), native depthwise convs
        (conv2d groups) -> fused engine (depthwise as a CUDA-core stage)
    C5  Inception-v3-style @299 (native concat / avg_pool2d), int8_int32
        -> fused engine (avg_pool2d and concat as fused stages)
    R50 under the reference's DEFAULT thresholds (quantile 0.99, pow2 off,
        calibration.hpp:71-76) -> the exact FP64 engine (the fused int8 engine
        is bit-exact only under power-of-two scales)"""
    legs = {}
    plans = [
        ("c2_resnet18", F.resnet(18), "int8_int32", batch, True, 0.999, 20),
        ("c3_mobilenet_v2", F.mobilenet_v2(image=224, width=1.0, classes=1000, native=True),
         "arm_vmlal_like", batch, True, 0.999, 8),
        ("c5_inception_v3", F.inception_v3(image=299, width=16, modules=2, head="gap", native=True),
         "int8_int32", 8, True, 0.999, 4),
        ("r50_default_thresholds", F.resnet(50), "int8_int32", 16, False, 0.99, 4),
        # the same under engine `fast` (fused int8 engine with non-pow2 scales:
        # within the tolerance stated and tested in tests/test_gpu_fast_mode.py)
        ("r50_default_thresholds_fast", F.resnet(50), "int8_int32", batch, False, 0.99, 8),
    ]
    from paper_2103_14949_b200 import cuda_ops
    ops = cuda_ops.load()
    for name, model, spec_name, n, pow2, qtl, k in plans:
        ops.set_engine_mode("fast" if name.endswith("_fast") else engine)
        try:
            data = model.data(n, seed=9)
            g = b.graph(model.doc, model.blob)
            spec = b.parse_spec(F.spec_fixture(spec_name))
            topo = b.generate_topology(g, spec)
            sim = b.insert_simulated_quantize(g, topo)
            ds = b.dataset(data)
            st = b.collect_stats(g, ds, 2048, b.simulated_edge_indices(g, topo))
            thr = st.estimate_thresholds("quantile", quantile=qtl, pow2=pow2)
            ev = b.evaluator(sim, spec, topo, thr, st, ds, min_bit=4 if spec_name != "arm_vmlal_like" else 8)
            sp = ev.space()
            cands = candidates(sp, k + 1)
            if spec_name == "arm_vmlal_like":
                # 8-bit codes on every edge: the int8 x int8 -> int16 signature
                cands = [[min(v, 8) for v in c] for c in cands]
            why = b.fused_status(sim, ev.bind(cands[0]))
            ran_on = "fused int8 tcgen05" if not why else f"exact FP64 engine ({why[:120]})"
            ev.losses(cands[:1])
            torch.cuda.synchronize()
            e0, e1 = _events(torch)
            e0.record(stream)
            ev.losses(cands[1:])
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / k
            legs[name] = {"images": n, "image": data.shape[-1], "spec": spec_name,
                          "thresholds": f"quantile {qtl}, pow2 {'on' if pow2 else 'off'}",
                          "ms_per_candidate": ms, "images_per_s": n / (ms / 1e3),
                          "candidates_per_s": 1e3 / ms, "candidates": k,
                          "gmac_per_image": model.macs_per_sample() / 1e9,
                          "engine": ran_on}
            if name == "c5_inception_v3":
                # C5 is a strategy-search config: a real random search over
                # its calibration images (speculative batches of 4)
                torch.cuda.synchronize()
                s0, s1 = _events(torch)
                s0.record(stream)
                res = b.search_batched("random", sp, evaluator=ev, mode="local", width=4, n=32, seed=7)
                s1.record(stream)
                torch.cuda.synchronize()
                sms = s0.elapsed_time(s1)
                legs[name]["search"] = {"method": "random", "n": 32, "ms": sms,
                                        "candidates_per_s": res.evaluations / (sms / 1e3),
                                        "best_loss": res.best_loss}
            del ev, ds, st, sim
        except Exception as e:  # a side leg never sinks the headline line
            legs[name] = {"error": str(e)[:300]}
    ops.set_engine_mode(engine)
    return legs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=120)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--engine", default="auto", choices=["auto", "fast", "exact"])
    ap.add_argument("--no-realized", action="store_true",
                    help="skip the realized-int8 eval_int leg")
    ap.add_argument("--no-search", action="store_true", help="skip the search legs")
    ap.add_argument("--no-traffic", action="store_true", help="skip the ncu traffic child")
    ap.add_argument("--no-configs", action="store_true", help="skip the C2/C3/C5 side legs")
    ap.add_argument("--traffic-probe", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--calib-images", type=int, default=128,
                    help="C4 leg: calibration images per GPU (1024 at 8 GPUs)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.traffic_probe:
        return traffic_probe(args)

    import torch
    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    dist = None
    os.environ.setdefault("QUANTC_DEVICE", str(local))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")

    from paper_2103_14949_b200 import cuda_ops
    b = Q.load_b200()
    ops = cuda_ops.load()
    ops.set_engine_mode(args.engine)
    L = b.lib
    L.qc_evaluator_agreement.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.c_size_t, C.c_size_t,
                                         C.POINTER(C.c_int64)]
    L.qcu_engine_stream.restype = C.c_void_p
    L.qcu_profile_enable.argtypes = [C.c_int]
    L.qcu_profile_read.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                   C.POINTER(C.c_double), C.POINTER(C.c_double)]
    stream = torch.cuda.ExternalStream(L.qcu_engine_stream())

    # the library's own communicator (comm.hpp): NCCL over NVLink, one rank
    # per GPU; the unique id travels over torch.distributed
    if world > 1:
        uid = [b.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = b.comm_nccl(rank, world, uid[0])
    else:
        comm = b.comm_local()

    def max_over_ranks(ms):
        if dist is None:
            return ms
        t = torch.tensor([ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    model = F.resnet(50)
    B = args.batch
    # weak scaling: rank r owns calibration images [r*B, (r+1)*B)
    data_all = model.data(B * world, seed=9)
    data = np.ascontiguousarray(data_all[rank * B:(rank + 1) * B])
    g = b.graph(model.doc, model.blob)
    spec = b.parse_spec(F.spec_fixture("int8_int32"))
    topo = b.generate_topology(g, spec)
    sim = b.insert_simulated_quantize(g, topo)
    edges = b.simulated_edge_indices(g, topo)

    # ---- C4 leg (runs first, on a fresh allocator pool): ResNet-50 KL
    # calibration, images sharded over ranks, distributed collect_stats
    # (extrema MIN/MAX and int64 histograms SUM all-reduced over the
    # library communicator), KL thresholds for every edge; device-timed on
    # the engine stream, max over ranks
    calib = None
    if args.calib_images > 0:
        cn = args.calib_images
        cal = np.ascontiguousarray(model.data(cn * world, seed=17)[rank * cn:(rank + 1) * cn])
        cal_ds = b.dataset(cal)
        b.collect_stats_dist(g, cal_ds, comm, 2048, edges)  # untimed warm pass
        runs = []
        for _ in range(3):
            barrier()
            c0, c1 = _events(torch)
            c2 = torch.cuda.Event(enable_timing=True)
            c0.record(stream)
            cst = b.collect_stats_dist(g, cal_ds, comm, 2048, edges)
            c1.record(stream)
            cal_thr = cst.estimate_thresholds("kl", kl_bits=8)
            c2.record(stream)
            torch.cuda.synchronize()
            cms, kms = max_over_ranks(c0.elapsed_time(c1)), max_over_ranks(c1.elapsed_time(c2))
            runs.append((cms + kms, cms, kms))
        runs.sort()
        _, cms, kms = runs[1]
        calib = {"workload": "resnet50 KL calibration (BASELINE config C4)",
                 "images": cn * world, "images_per_gpu": cn, "edges": len(edges),
                 "bins": 2048, "collect_stats_ms": cms, "kl_thresholds_ms": kms,
                 "images_per_s": cn * world / ((cms + kms) / 1e3),
                 "passes_ms": [round(r[0], 1) for r in runs], "reported": "median of 3 passes",
                 "thresholds": len(cal_thr),
                 "merge": ("NCCL all_reduce MIN/MAX extrema + SUM int64 histograms "
                           "(quantc::collect_stats over a Communicator)") if world > 1
                 else "single GPU"}
        del cal_ds

    # ---- main leg: thresholds from the MERGED statistics of all ranks'
    # shards (every rank binds identical strategies); each rank's evaluator
    # holds its own shard; per-candidate agreement counts all-reduced
    ds = b.dataset(data)
    st = b.collect_stats_dist(g, ds, comm, 2048, edges)
    thr = st.estimate_thresholds("quantile", quantile=0.999, pow2=True)
    ev = b.evaluator(sim, spec, topo, thr, st, ds)
    sp = ev.space()
    cands = candidates(sp, args.warmup + args.steps)

    counts = np.zeros(1, np.int64)
    cnt_t = torch.zeros(1, dtype=torch.int64, device=f"cuda:{local}")

    def step(c):
        arr = np.asarray(c, np.int32)
        rc = L.qc_evaluator_agreement(ev.h, arr.ctypes.data_as(C.POINTER(C.c_int)), 1, len(c),
                                      counts.ctypes.data_as(C.POINTER(C.c_int64)))
        b.check(rc)
        if dist is not None:
            cnt_t.fill_(int(counts[0]))
            dist.all_reduce(cnt_t)
            return 1.0 - cnt_t.item() / (B * world)
        return 1.0 - counts[0] / B

    def steps_batched(cs):
        """K candidate evaluations through one CandidateEvaluator::losses(span)
        call (qc_evaluator_agreement over the batch; per-rank counts, one
        all-reduce of the K counts): the search's batch API, evaluated four
        at a time through grouped tcgen05 launches."""
        a = np.ascontiguousarray(np.asarray(cs, np.int32))
        out = np.zeros(len(cs), np.int64)
        b.check(L.qc_evaluator_agreement(ev.h, a.ctypes.data_as(C.POINTER(C.c_int)), a.shape[0],
                                         a.shape[1], out.ctypes.data_as(C.POINTER(C.c_int64))))
        if dist is not None:
            t = torch.from_numpy(out).to(f"cuda:{local}")
            dist.all_reduce(t)
            out = t.cpu().numpy()
        return 1.0 - out / (B * world)

    for i in range(args.warmup):
        step(cands[i])
    steps_batched(cands[:args.warmup])
    barrier()
    launches0 = ops.counters()["steps"]
    e0, e1 = _events(torch)
    with ClockSampler(local) as clk:
        e0.record(stream)
        steps_batched(cands[args.warmup:args.warmup + args.steps])
        e1.record(stream)
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    launches = ops.counters()["steps"] - launches0
    ms = max_over_ranks(e0.elapsed_time(e1))
    ms_step = ms / args.steps
    imgs_per_s = B * world * args.steps / (ms / 1e3)

    # ---- the same candidates, one C-ABI call (and all-reduce) per candidate
    pc_steps = min(args.steps, 10)
    barrier()
    p0, p1 = _events(torch)
    p0.record(stream)
    for i in range(pc_steps):
        step(cands[args.warmup + i])
    p1.record(stream)
    torch.cuda.synchronize()
    pc_ms = max_over_ranks(p0.elapsed_time(p1))
    per_call = {"ms_per_step": pc_ms / pc_steps,
                "images_per_s": B * world * pc_steps / (pc_ms / 1e3), "steps": pc_steps,
                "api": "qc_evaluator_agreement with one candidate per call (CandidateEvaluator::loss)"}

    # ---- random candidates (every layer's weight codes change per candidate)
    rc_n = min(args.steps, 40)
    rcands = random_candidates(sp, rc_n + 4)
    steps_batched(rcands[:4])
    barrier()
    q0, q1 = _events(torch)
    q0.record(stream)
    steps_batched(rcands[4:])
    q1.record(stream)
    torch.cuda.synchronize()
    rc_ms = max_over_ranks(q0.elapsed_time(q1))
    random_leg = {"ms_per_step": rc_ms / rc_n, "images_per_s": B * world * rc_n / (rc_ms / 1e3),
                  "steps": rc_n, "candidates": "every slot drawn uniformly (seed 1)"}

    # ---- roofline pass: the SAME grouped losses call as the timed step, with
    # per-launch CUDA events around every tc_conv_kernel launch (events cost
    # the programmatic-dependent-launch overlap, so this pass is separate)
    prof_n = min(args.steps, 20)
    L.qcu_profile_enable(1)
    gms, gl, gops, gbytes = C.c_double(), C.c_int64(), C.c_double(), C.c_double()
    L.qcu_profile_read(C.byref(gms), C.byref(gl), C.byref(gops), C.byref(gbytes))  # drain
    r0, r1 = _events(torch)
    r0.record(stream)
    steps_batched(cands[args.warmup:args.warmup + prof_n])
    r1.record(stream)
    torch.cuda.synchronize()
    L.qcu_profile_read(C.byref(gms), C.byref(gl), C.byref(gops), C.byref(gbytes))
    L.qcu_profile_enable(0)
    prof_step_ms = r0.elapsed_time(r1)

    # ---- search legs (BASELINE metric: search candidates/s at 1/2/4/8 GPUs):
    # REAL searches on ResNet-50 over a fixed calibration set of B images held
    # by every rank; candidate batches sharded over ranks (candidate-sharded
    # losses, one all-gather per batch), speculative width 4 per rank
    search = None
    if not args.no_search:
        fixed = np.ascontiguousarray(data_all[:B])
        fds = b.dataset(fixed)
        fst = b.collect_stats_dist(g, fds, b.comm_local(), 2048, edges)
        fthr = fst.estimate_thresholds("quantile", quantile=0.999, pow2=True)
        fev = b.evaluator(sim, spec, topo, fthr, fst, fds)
        fev.losses(candidates(fev.space(), 4))  # warm
        search = {"calibration_images": B, "sharding": "candidates over ranks" if world > 1
                  else "single GPU", "width_per_rank": 4}
        for method, kw in (("greedy", dict(rounds=1, tol=0.02)),
                           ("random", dict(n=64 * world, seed=7))):
            barrier()
            s0, s1 = _events(torch)
            s0.record(stream)
            res = b.search_batched(method, fev.space(), evaluator=fev, comm=comm,
                                   mode="candidates", width=4 * world, **kw)
            s1.record(stream)
            torch.cuda.synchronize()
            sms = max_over_ranks(s0.elapsed_time(s1))
            batches, evaluated, committed = res.speculation
            search[method] = {
                "params": kw, "ms": sms, "evaluations": res.evaluations,
                "candidates_per_s": res.evaluations / (sms / 1e3),
                "evaluated_per_s": evaluated / (sms / 1e3), "evaluated": evaluated,
                "batches": batches, "best_loss": res.best_loss}
        del fev, fds

    # ---- e2e (the headline against the reference arm; measured before the
    # side legs, whose allocations would otherwise skew the host path):
    # public C-ABI call with HOST buffers: predict_top1 of the sim
    # graph under a candidate binding (uploads images + plan, downloads preds)
    e2e_steps = max(3, min(10, args.steps))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    b.predict_top1(sim, ds, 0, ev.bind(cands[0]))
    cold_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    for i in range(e2e_steps):
        b.predict_top1(sim, ds, 0, ev.bind(cands[(i + 1) % len(cands)]))
    e2e_dt = (time.perf_counter() - t0) / e2e_steps
    e2e_dt = max_over_ranks(e2e_dt * 1e3) / 1e3
    h2d = data.nbytes
    d2h = 8 * B

    # ---- realized int8 leg: the all_hi strategy
    # lowered by realize() on the same network declared with a batched input;
    # eval_int runs its int8 convs on tcgen05 with the zero-point / clamp /
    # requantize epilogue (host input in, dequantized scores out, per call)
    realized = None
    if not args.no_realized:
        strategy = ev.strategy_for(sp.all_hi())
        mb = F.resnet(50, batch=B)
        gbatch = b.graph(mb.doc, mb.blob)
        simb = b.insert_simulated_quantize(gbatch, b.generate_topology(gbatch, spec))
        R = b.realize(simb, strategy, spec)
        xin = np.ascontiguousarray(data.reshape(B, 3, 224, 224))
        c_before = ops.counters()["tcgen05_gemms"]
        b.eval_int(R, xin)  # warm: plan, packed weights, allocator pool
        c_after = ops.counters()["tcgen05_gemms"]
        torch.cuda.synchronize()
        r0, r1 = _events(torch)
        r0.record(stream)
        reps = 3
        for _ in range(reps):
            b.eval_int(R, xin)
        r1.record(stream)
        torch.cuda.synchronize()
        rms = r0.elapsed_time(r1) / reps
        realized = {"workload": "resnet50 realized int8 graph (all_hi strategy), eval_int",
                    "batch": B, "ms_per_call": rms, "images_per_s": B / (rms / 1e3),
                    "tcgen05_convs_per_call": c_after - c_before,
                    "includes": "host fp32 input upload and output download, int32 tensors between "
                                "layers (the reference Tensor semantics)"}
        del R, simb, gbatch, mb

    configs = None
    if not args.no_configs and world == 1:
        try:
            configs = config_legs(b, torch, stream, B, args.engine)
        except Exception as e:  # side legs never sink the headline line
            configs = {"error": str(e)[:300]}
            ops.set_engine_mode(args.engine)

    # ---- roofline of the dominant kernel: tc_conv_kernel, the fused tcgen05
    # implicit-GEMM conv + sq/add epilogue (every conv/dense launch of a
    # step).  Tensor-bound framing (the north star's target): algorithmic
    # int8 ops (2 x MACs, each group's problem counted) / launch time.
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    bf16 = peaks.get("bf16_tflops", 1590.0)
    int8_peak = 2.0 * bf16  # dense int8 rate = 2x bf16 on B200
    hbm_peak = peaks.get("hbm_gbs", 6543.7)
    gsec = gms.value / 1e3
    tops = (gops.value / gsec) / 1e12 if gsec > 0 else 0.0
    gbs = (gbytes.value / gsec) / 1e9 if gsec > 0 else 0.0
    nl = max(1, gl.value)
    traffic = None
    if rank == 0 and world == 1 and not args.no_traffic:
        traffic = measure_traffic(args)

    line = {
        "metric": METRIC, "value": imgs_per_s, "unit": "images/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int8",
        "data": "synthetic (N(0,1) images, He-normal BN-folded ResNet-50 weights, seeds 9/42)",
        "config": {"workload": "resnet50 int8_int32 sim-quant candidate evaluation",
                   "model": "resnet50", "image": 224, "global_batch": B * world,
                   "per_gpu_batch": B, "parallelism": f"dp{world} (calibration shards)",
                   "thresholds": "quantile 0.999, pow2, from the merged statistics of all "
                                 "ranks (tcgen05 path bit-exact)",
                   "engine": args.engine, "l2": "inputs 38.5 MB/GPU + activations > L2",
                   "step_api": "CandidateEvaluator::losses over the K timed candidates in one "
                               "qc_evaluator_agreement call (see per_call for one call each)"},
        "candidates_per_s": args.steps / (ms / 1e3),
        "e2e": {"value": B * world / e2e_dt, "unit": "images/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "api": "qc_predict_top1(sim_graph, host dataset, binding) per step, new binding each; the dataset (qc_dataset_create) holds its samples page-locked, so each step DMAs them straight from host memory",
                "cold_first_call_s": cold_s,
                "weights_bytes_uploaded_once": len(model.blob)},
        "per_call": per_call,
        "random_candidates": random_leg,
        "search": search,
        "calibration": calib,
        "realized_int8": realized,
        "configs": configs,
        "gpu_launches": int(launches),
        "roofline": {"bound": "tensor", "achieved": tops, "peak": int8_peak, "unit": "TFLOP/s",
                     "frac": tops / int8_peak if int8_peak else None,
                     "traffic": traffic["dram_bytes_per_launch"] if traffic else None,
                     "kernel": "tc_conv_kernel (fused tcgen05 kind::i8 implicit-GEMM conv + "
                               "sq/add epilogue), every launch of the grouped timed step",
                     "ops_unit": "int8 ops (2 x MAC), counted as FLOP",
                     "peak_source": "2 x MEASURED_PEAKS.json bf16_tflops (dense int8 = 2x bf16)",
                     "algorithmic_ops_per_launch": gops.value / nl,
                     "algorithmic_bytes_per_launch": gbytes.value / nl,
                     "avg_launch_us": 1e3 * gms.value / nl,
                     "launches_per_step": gl.value / prof_n,
                     "kernel_share_of_step": gms.value / prof_step_ms if prof_step_ms else None,
                     "profiled_step_ms": prof_step_ms / prof_n,
                     "profiled_vs_timed_step": (prof_step_ms / prof_n) / ms_step,
                     "hbm": {"achieved": gbs, "peak": hbm_peak, "unit": "GB/s",
                             "frac": gbs / hbm_peak if hbm_peak else None,
                             "bytes": "algorithmic (inputs, weights, bias, outputs, residual once)"},
                     "traffic_source": traffic["source"] if traffic else None,
                     "traffic_launches": traffic["launches"] if traffic else None},
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline and os.path.exists(REF_LIB):
        # the reference on the box's host cores, on the bench's own first
        # images under candidate 0's binding; its predictions must equal the
        # B200's for the same images and binding (parity of the timed path)
        threads = os.cpu_count() or 1
        sample = min(max(threads, 2), 16)
        bnd = ev.bind(cands[0])
        sub = np.ascontiguousarray(data[:sample])
        ref_preds, dt = cpu_reference_preds(model, sub, threads, bnd)
        b200_preds = b.predict_top1(sim, b.dataset(sub), 0, bnd)
        if not np.array_equal(ref_preds, b200_preds):
            raise SystemExit(f"PARITY FAILURE: reference predictions {ref_preds.tolist()} != "
                             f"B200 {b200_preds.tolist()} on the bench's images")
        line["cpu_baseline"] = {"value": sample / dt, "unit": "images/s", "cores": threads,
                                "kind": "reference",
                                "sample": f"{sample} bench images x 1 candidate ({dt:.1f} s); "
                                          "predictions checked equal to the B200's"}
    if rank == 0:
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
