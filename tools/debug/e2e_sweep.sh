# e2e variants at config 1: value, e2e value, e2e ms/step
python -m pytest tests/test_gpu_transforms.py -x -q 2>&1 | tail -1
run() {
  r=$(env "$@" python bench.py --steps 30 --warmup 5 --no-mlsdc --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print(round(d['value']), round(e['value']), round(e['ms_per_step'],3), e['roundtrip_err'])")
  echo "$* -> $r"
}
for rep in 1 2; do
for c in 24 32 48; do for k in 2 4; do run SWSDC_UPLOAD_CTAS=$c SWSDC_DOWNLOAD_MODE=1 SWSDC_STAIR_BLOCKS=$k; done; done
done
