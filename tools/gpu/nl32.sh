set -u
O=gpurun_out/nl32
mkdir -p $O
timeout 1200 python -m pytest tests -x -q -m gpu -k "c5 or K128 or k128 or 128 or nbest or beam_sizes or merge_tie or fixture" > $O/pytest.log 2>&1
python tools/ab.py time --workload c5 base nl32 > $O/ab_c5.jsonl 2>&1
python tools/ab.py time --workload c4 base nl32 > $O/ab_c4.jsonl 2>&1
echo done > $O/done
