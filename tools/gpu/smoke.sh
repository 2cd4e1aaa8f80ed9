set -u
O=gpurun_out/smoke
mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_merge_first.py -x -q > $O/pytest_mf.log 2>&1
echo done > $O/done
