cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r2int}
GROUP=4 QUANTC_DEBUG_INT=1 timeout 300 python scripts/profile_step.py > gpurun_out/${TAG}_fold.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_pin.py tests/test_gpu_configs.py -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_tests.log
GROUP=4 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/${TAG}_group4_launches.csv python scripts/profile_step.py > gpurun_out/${TAG}_ncu1.log 2>&1
timeout 600 python bench.py --no-realized --no-traffic --no-search > gpurun_out/${TAG}_bench.log 2> gpurun_out/${TAG}_bench.err
