for C in 256 512 1024 2048 8192; do
  PDLP_DEFINES="-DPDLPK_CHUNK=$C" python -m paper_2501_07018_b200.build --force > /dev/null 2>&1 || echo build-fail
  timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['per_kernel']; print($C, round(d['value']), round(d['e2e']['value']), {n:round(v['mean_us'],1) for n,v in k.items()}, d['time_to_tol']['seconds'])"
done
