# quick iteration: fused-path parity tests, launch list, short bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r2q}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_pin.py tests/test_gpu_configs.py -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_tests.log
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv"
GROUP=4 timeout 600 ncu $M --log-file gpurun_out/${TAG}_launches.csv python scripts/profile_step.py > gpurun_out/${TAG}_ncu.log 2>&1
timeout 600 python bench.py --no-realized --no-traffic --no-search --no-configs --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2> gpurun_out/${TAG}_bench.err
# optional A/B: the same short bench under an extra environment setting
if [ -n "$AB_ENV" ]; then
  env $AB_ENV timeout 600 python bench.py --no-realized --no-traffic --no-search --no-configs --no-cpu-baseline > gpurun_out/${TAG}_bench_ab.log 2> gpurun_out/${TAG}_bench_ab.err
fi
if [ -n "$AB_ENV" ] && [ -n "$AB_LAUNCHES" ]; then
  env $AB_ENV GROUP=4 timeout 600 ncu $M --log-file gpurun_out/${TAG}_launches_ab.csv python scripts/profile_step.py > gpurun_out/${TAG}_ncu_ab.log 2>&1
fi
