set -u
O=gpurun_out/lt32
mkdir -p $O
python tools/ab.py time --workload c4 base lt32 > $O/ab_c4.jsonl 2>&1
python tools/ab.py time --workload c5 base lt32 > $O/ab_c5.jsonl 2>&1
echo done > $O/done
