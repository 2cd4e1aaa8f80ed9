set -u
O=gpurun_out/chunk
mkdir -p $O
for rep in 1 2; do
  python bench.py --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | sed "s/^/chunk c4 /" >> $O/ab.txt
  FLEXCTC_CMP=1 python bench.py --workload c5 --steps 10 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | sed "s/^/chunk c5 /" >> $O/ab.txt
done
timeout 1800 python -m pytest tests -x -q -m gpu > $O/pytest.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:frame_compact -s 3 -c 1 -o $O/prof_compact_c4 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done > $O/done
