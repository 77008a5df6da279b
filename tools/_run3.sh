mkdir -p gpurun_out/s5
(time timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q) > gpurun_out/s5/pytest_parity.log 2>&1
tail -5 gpurun_out/s5/pytest_parity.log
timeout 300 python tools/k2_ab.py > gpurun_out/s5/k2_ab.log 2>&1; cat gpurun_out/s5/k2_ab.log
(time timeout 1500 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_parity.py) > gpurun_out/s5/pytest_rest.log 2>&1
tail -5 gpurun_out/s5/pytest_rest.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/s5/bench.json 2> gpurun_out/s5/bench.err
python - <<'PY'
import json
d=json.load(open('gpurun_out/s5/bench.json'))
print(d['value'], d['e2e']['value'], d['sweep'])
print({k:(v.get('seconds') if isinstance(v,dict) else v) for k,v in d['circuits'].items() if k!='reference_cpu'})
print(d['latency'])
PY
