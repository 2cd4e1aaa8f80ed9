set -u
O=gpurun_out/lt
mkdir -p $O
timeout 1200 python -m pytest tests -x -q -m gpu -k "c4 or c3 or c5 or fixture or beam_sizes or records or variants or nbest" > $O/pytest.log 2>&1
python tools/ab.py time --workload c4 base lt > $O/ab_c4.jsonl 2>&1
python tools/ab.py time --workload c5 base lt > $O/ab_c5.jsonl 2>&1
echo done > $O/done
