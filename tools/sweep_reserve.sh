for r in 0 4 8 12 16 24; do for s in 2 3; do
  v=$(CBP_BENCH_SM_RESERVE=$r CBP_BENCH_REC_STREAMS=$s timeout 200 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']), d['roofline']['pass_ms_per_plane'])")
  echo "reserve=$r streams=$s $v" >> gpurun_out/sweep.txt
done; done
