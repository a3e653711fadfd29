# A/B launch lists of one grouped 4-candidate step under engine switches,
# histogram variants, fast-mode test, exact-engine launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r2ab}
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --profile-from-start off --csv"
GROUP=4 timeout 600 ncu $M --log-file gpurun_out/${TAG}_base.csv python scripts/profile_step.py > /dev/null 2>&1
GROUP=4 QUANTC_NO_IM2COL64=1 timeout 600 ncu $M --log-file gpurun_out/${TAG}_noim2col64.csv python scripts/profile_step.py > /dev/null 2>&1
GROUP=4 QUANTC_NO_IM2COL=1 timeout 600 ncu $M --log-file gpurun_out/${TAG}_noim2col.csv python scripts/profile_step.py > /dev/null 2>&1
if [ -f exp/libquantc_b200_e8.so ]; then GROUP=4 QUANTC_B200_LIB=$PWD/exp/libquantc_b200_e8.so timeout 600 ncu $M --log-file gpurun_out/${TAG}_e8.csv python scripts/profile_step.py > gpurun_out/${TAG}_e8.log 2>&1; fi
timeout 600 ncu $M --log-file gpurun_out/${TAG}_exact.csv python scripts/profile_exact.py > gpurun_out/${TAG}_exact.log 2>&1
for z in 0 1; do QUANTC_HIST_ZREG=$z timeout 300 python scripts/scan_kernels_bench.py > gpurun_out/${TAG}_scan_z$z.json 2>&1; done
timeout 600 python -m pytest tests/test_gpu_fast_mode.py tests/test_gpu_parity.py -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_tests.log
