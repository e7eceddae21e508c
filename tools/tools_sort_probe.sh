#!/bin/bash
# Dev probe: cfg2 build-step kernel split under sort knobs (MSD depth / window-sort mode / cap).
run() {
  env "$@" python bench.py --steps 5 --warmup 3 --no-vector > gpurun_out/bs.json 2>gpurun_out/bs.err
  python -c "
import json;d=json.load(open('gpurun_out/bs.json'));k=d['breakdown']['kernels']
print('$*', round(d['ms_per_step'],3), {n:round(k[n]['ms_per_step'],3) for n in ('segment_sort','radix_onesweep','radix_hist')})"
}
for a in "$@"; do run ${a//,/ }; done
