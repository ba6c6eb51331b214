# bench.py value vs the SM reserve left to the recovery streams (CBP_BENCH_SM_RESERVE), 2 runs each
for r in ${RESERVES:-0 4 8 12 16 24}; do for i in 1 2; do
  v=$(CBP_BENCH_SM_RESERVE=$r timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), [round(x*1000,2) for x in d['roofline']['pass_ms_per_plane']])")
  echo "reserve=$r $v" >> gpurun_out/sweep.txt
done; done
