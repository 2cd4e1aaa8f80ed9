set -u
O=gpurun_out
for v in lb3 lb4 lb3 lb4; do
  FLEXCTC_LIB_AB=ab/lib$v.so python bench.py --no-cpu-baseline --no-e2e --steps 20 > $O/ablb_$v.log 2>&1
  python -c "
import json
for l in open('$O/ablb_$v.log'):
    if l.startswith('{'):
        d=json.loads(l); print(json.dumps({'v':'$v','ms':d['ms_per_step'],'beam':d['roofline']['kernel_ms'],'cmp':d.get('roofline_compact',{}).get('kernel_ms'),'frac':d.get('roofline_compact',{}).get('frac')}))
" >> $O/ablb.jsonl
done
echo done > $O/ablb_done
