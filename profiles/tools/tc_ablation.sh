for d in 0 2 1 3; do
  ES_TC_DBG=$d ES_ATTN_TC=1 timeout 200 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/dbg_$d.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/dbg_$d.json')); print('dbg $d', d['roofline']['kernel_ms']['attn_fwd'])"
done
