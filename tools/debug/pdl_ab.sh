python -m pytest tests -x -q -m gpu 2>&1 | tail -1
for pdl in 1 0; do
  echo "PDL=$pdl"
  SWSDC_PDL=$pdl python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-mlsdc | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg1', round(d['value']), round(d['ms_per_step']*1e3,1), 'us/step e2e', round(d['e2e']['value']))"
  for c in config2 config0; do SWSDC_PDL=$pdl python tools/one_step.py $c | head -1; done
done
