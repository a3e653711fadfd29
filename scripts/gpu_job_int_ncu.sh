# ncu --set full of realized-graph (eval_int) tcgen05 conv launches
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-intk}
for S in ${SKIPS:-10}; do
  timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off --kernel-name regex:tc_conv_kernel --launch-skip $S --launch-count 1 -o gpurun_out/${TAG}_k$S python scripts/profile_int.py > gpurun_out/${TAG}_ncu_k$S.log 2>&1
  python scripts/ncu_report.py gpurun_out/${TAG}_k$S.ncu-rep > gpurun_out/${TAG}_k$S.md 2>&1
  ncu -i gpurun_out/${TAG}_k$S.ncu-rep --page source --csv --print-source sass > /tmp/${TAG}_k${S}_source.csv 2>&1
  python scripts/ncu_sass_hist.py /tmp/${TAG}_k${S}_source.csv > gpurun_out/${TAG}_k${S}_sass.txt 2>&1
  gzip -c /tmp/${TAG}_k${S}_source.csv > gpurun_out/${TAG}_k${S}_source.csv.gz
  rm -f gpurun_out/${TAG}_k$S.ncu-rep
done
