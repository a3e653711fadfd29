# full GPU validation: the -m gpu suite, smoke(), and the default bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${TAG:-r2full}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2> gpurun_out/${TAG}_bench.err; echo rc=$? >> gpurun_out/${TAG}_bench.err
