# iteration job: full -m gpu suite, a short bench line, the grouped-step launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r2it}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_tests.log
timeout 600 python bench.py --no-realized --no-traffic --no-search --no-configs --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2> gpurun_out/${TAG}_bench.err
GROUP=4 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/${TAG}_launches.csv python scripts/profile_step.py > gpurun_out/${TAG}_ncu0.log 2>&1
if [ -n "$CONFIGS" ]; then timeout 900 python -c "
import sys, json, torch; sys.argv=['bench.py']; import bench
from paper_2103_14949_b200 import quantc as Q, cuda_ops
b=Q.load_b200(); L=b.lib; cuda_ops.load()
import ctypes as C
L.qcu_engine_stream.restype = C.c_void_p
s=torch.cuda.ExternalStream(L.qcu_engine_stream())
print(json.dumps(bench.config_legs(b, torch, s, 64), indent=1))
" > gpurun_out/${TAG}_configs.log 2>&1; fi
