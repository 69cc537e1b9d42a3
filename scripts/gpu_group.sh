#!/bin/bash
# group kernel: evolve tests + C5 small-N timing (group B = 16 / 8 vs the previous kernels)
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-r2s}
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "group or small_n or schedules or slab_buffer or sample_counts or range_resumes or periodic" > $O/${TAG}_pytest.log 2>&1
echo "rc=$?" >> $O/${TAG}_pytest.log; tail -4 $O/${TAG}_pytest.log
for k in 0 3; do for N in 64 128 256; do
  for v in "0:16" "0:8" "1:0"; do
    var=${v%%:*}; b=${v##*:}
    if [ "$var" = "1" ]; then extra="--kernel-variant 1"; export SNK_GROUP_B=16; else extra=""; export SNK_GROUP_B=$b; fi
    timeout 300 python bench.py --config C5_$k --steps 3 --no-cpu-baseline --no-e2e --n-samples $N $extra > $O/${TAG}_C5_${k}_N${N}_$var$b.json 2> $O/${TAG}_C5_${k}_N${N}_$var$b.err
    python -c "import json; d=json.loads(open('$O/${TAG}_C5_${k}_N${N}_$var$b.json').read().splitlines()[-1]); r=d['roofline']; print('C5_$k N=$N v=$v', round(d['phase_ms']['evolve'],3), 'hbm', r['frac'], 'alu', r['alu_model']['frac'])"
  done
done; done
