#!/bin/bash
cd "$GRAFT_REPO_ROOT"
TAG=${TAG:-r2k}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_dist.py -m gpu -q -s --durations=10 > gpurun_out/${TAG}_dist.log 2>&1
echo "rc=$?" >> gpurun_out/${TAG}_dist.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err
echo "rc=$?" >> gpurun_out/${TAG}_bench_c4.err
tail -5 gpurun_out/${TAG}_dist.log
cat gpurun_out/${TAG}_bench_c4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['ms_per_step'], d['phase_ms'], d['roofline']['samples_per_s_kernel']/1e9, d['e2e']['value']/1e9 if d['e2e'] else None, d['cpu_baseline'])"
tail -2 gpurun_out/${TAG}_bench_c4.err
