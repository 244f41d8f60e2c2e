for v in lean nolean lean nolean; do
  if [ $v = nolean ]; then export KOG2_SVD2_NO_LEAN=1; else unset KOG2_SVD2_NO_LEAN; fi
  timeout 300 python bench.py --no-study --no-cpu --no-configs --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['e2e']['value']/1e9,4), round(d['ms_per_step'],3))"
done
