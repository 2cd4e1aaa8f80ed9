set -u
O=gpurun_out/cmptma2
mkdir -p $O
timeout 900 python -m pytest tests -x -q -m gpu -k "compaction or warp or bf16 or c5_full or logits or greedy" > $O/pytest.log 2>&1
for rep in 1 2; do
for v in "FLEXCTC_CMP_TMA=0" "FLEXCTC_CMP_STAGES=2" "FLEXCTC_CMP_STAGES=3"; do
  env $v python bench.py --steps 20 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | sed "s/^/$v c4 /" >> $O/ab.txt
  env $v FLEXCTC_CMP=1 python bench.py --workload c5 --steps 10 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | sed "s/^/$v c5 /" >> $O/ab.txt
done
done
python bench.py --workload c4 --beam 1 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | sed "s/^/greedy c4k1 /" >> $O/ab.txt
ncu --set full --clock-control none --import-source on -k regex:frame_compact -s 3 -c 1 -o $O/prof_compact_c4 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
echo done > $O/done
