# e2e variants at config 1: value, e2e value, e2e ms/step
run() {
  r=$(env "$@" python bench.py --steps 40 --warmup 5 --no-mlsdc --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print(round(d['value']), round(e['value']), round(e['ms_per_step'],3))")
  echo "$* -> $r"
}
run SWSDC_DOWNLOAD_MODE=1
for c in 16 32 64; do run SWSDC_DOWNLOAD_MODE=0 SWSDC_UPLOAD_CTAS=$c; done
