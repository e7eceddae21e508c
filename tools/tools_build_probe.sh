#!/bin/bash
# Dev probe: cfg2 build step breakdown (kernel ms per step) for a quick A/B of build kernels.
python bench.py --no-knn --no-cpu-baseline --no-inpaint --steps 10 > gpurun_out/bench_probe.json 2> gpurun_out/bench_probe.err
python -c "
import json; d=json.load(open('gpurun_out/bench_probe.json'))
print('ms/step', round(d['ms_per_step'],3), 'value', round(d['value']/1e6,1), 'M/s  e2e', round(d['e2e']['value']/1e6,1))
print({k: round(v['ms_per_step'],3) for k,v in d['breakdown']['kernels'].items()})"
