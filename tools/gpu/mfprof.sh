set -u
O=gpurun_out/mfprof
mkdir -p $O
timeout 900 ncu --set full --import-source on -k regex:merge_first -s 1 -c 1 -o $O/prof_mf_c4 \
    python bench.py --merge-first --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu.log 2>&1
echo done > $O/done
