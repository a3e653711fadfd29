# aux evidence: scan-kernel HBM bench (incl. relu-edge histogram), conv_f64 ncu
# (exact engine, R50 default thresholds), compute-sanitizer over the smoke path
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r2aux}
timeout 300 python scripts/scan_kernels_bench.py > gpurun_out/${TAG}_scan.json 2> gpurun_out/${TAG}_scan.err
timeout 600 python -m pytest tests/test_gpu_fast_mode.py tests/test_gpu_native_ops.py -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_tests.log
# conv_f64: one launch list of an exact-engine candidate evaluation + full capture of a stage-3 conv
timeout 600 ncu --set full --clock-control none --kernel-name regex:conv_f64_kernel --launch-skip 20 --launch-count 1 -o gpurun_out/${TAG}_f64 python scripts/profile_exact.py > gpurun_out/${TAG}_ncu_f64.log 2>&1
python scripts/ncu_report.py gpurun_out/${TAG}_f64.ncu-rep > gpurun_out/${TAG}_f64.md 2>&1
ncu -i gpurun_out/${TAG}_f64.ncu-rep --page raw --csv > gpurun_out/${TAG}_f64_raw.csv 2>&1
rm -f gpurun_out/${TAG}_f64.ncu-rep
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum --clock-control none --csv --log-file gpurun_out/${TAG}_exact_launches.csv python scripts/profile_exact.py > gpurun_out/${TAG}_ncu_ex.log 2>&1
# compute-sanitizer: memcheck / racecheck / synccheck over the smoke path (tcgen05 + TMA kernels)
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_san_$tool.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_san_$tool.log
done
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "fused" > gpurun_out/${TAG}_san_memcheck_fused.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_san_memcheck_fused.log
