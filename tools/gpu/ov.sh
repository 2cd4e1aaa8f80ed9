set -u
O=gpurun_out/ov
mkdir -p $O
timeout 600 python -m pytest tests -x -q -m gpu -k "compaction_records or c4 or smoke" > $O/pytest_quick.log 2>&1
for rep in 1 2; do
  FLEXCTC_OVERLAP=0 timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | sed "s/^/serial c4 /" >> $O/ab.txt
  timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | sed "s/^/overlap c4 /" >> $O/ab.txt
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_c4.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 1800 python -m pytest tests -x -q -m gpu > $O/pytest.log 2>&1
echo done > $O/done
