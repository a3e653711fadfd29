# iteration: -m gpu suite, short bench, launch list, scan-kernel A/B (histogram copies)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r2it3}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_tests.log
timeout 600 python bench.py --no-realized --no-traffic --no-search --no-configs --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2> gpurun_out/${TAG}_bench.err
GROUP=4 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/${TAG}_launches.csv python scripts/profile_step.py > gpurun_out/${TAG}_ncu0.log 2>&1
for r in 1 2 4; do QUANTC_HIST_REPS=$r timeout 300 python scripts/scan_kernels_bench.py > gpurun_out/${TAG}_scan_reps$r.json 2>&1; done
