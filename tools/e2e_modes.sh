#!/bin/bash
# e2e (config 1) for the upload / download engine combinations; host core count.
nproc
python - <<'PY'
import ctypes, time, numpy as np, sys
sys.path.insert(0, '.')
from paper_1805_07923_b200 import _lib
lib = _lib.load()
R, nm = 255, 15
c = np.random.default_rng(0).standard_normal((nm, R + 1, R + 1, 2))
out = np.empty((nm, (R + 1) * (R + 2) // 2, 2))
for _ in range(5):
    lib.swsdc_pack_triangles(c.ctypes.data, R, nm, out.ctypes.data)
t = time.perf_counter()
for _ in range(50):
    lib.swsdc_pack_triangles(c.ctypes.data, R, nm, out.ctypes.data)
print("host pack (sync, pageable) us:", (time.perf_counter() - t) / 50 * 1e6)
PY
for up in 0 2; do for dn in 1 0; do for rep in 1 2; do
  echo "UPLOAD_MODE=$up DOWNLOAD_MODE=$dn ${EXTRA}"
  SWSDC_UPLOAD_MODE=$up SWSDC_DOWNLOAD_MODE=$dn python bench.py --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline --no-mlsdc --soak 0.3 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('  e2e', round(e['value']), 'us/step', round(e['ms_per_step']*1e3,1), 'dense', round(e['dense_fresh_download']['value']), 'value', round(d['value']), 'err', e['roundtrip_err'])"
done; done; done
