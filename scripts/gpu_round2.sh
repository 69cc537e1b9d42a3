#!/bin/bash
# Round-2 evidence run: GPU tests, smoke, C4 bench (+cpu_baseline), reference arm,
# compute-sanitizer on C1, ncu launch list + evolve/volume captures.
cd "$GRAFT_REPO_ROOT"; O=gpurun_out; mkdir -p $O; TAG=${TAG:-r2u}
nvidia-smi > $O/${TAG}_nvidia_smi.txt 2>&1; (nproc; lscpu | grep 'Model name') > $O/${TAG}_host.txt
python -c "import __graft_entry__ as g; g.build()" > $O/${TAG}_build.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -rf --durations=15 > $O/${TAG}_pytest_gpu.log 2>&1
echo "rc=$?" >> $O/${TAG}_pytest_gpu.log; tail -3 $O/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "rc=$?" >> $O/${TAG}_smoke.log; tail -2 $O/${TAG}_smoke.log
timeout 1200 python bench.py > $O/${TAG}_bench_c4.json 2> $O/${TAG}_bench_c4.err; tail -c 3000 $O/${TAG}_bench_c4.json
timeout 1200 python bench.py --impl reference --steps 3 --warmup 3 > $O/${TAG}_bench_ref.json 2> $O/${TAG}_bench_ref.err; tail -c 1500 $O/${TAG}_bench_ref.json
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/profile_step.py --config C1 --steps 1 --warmup 0 --iters 30 > $O/${TAG}_sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 $O/${TAG}_sanitizer_$tool.log
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_launches_c4.csv python scripts/profile_step.py --config C4 --steps 1 --warmup 1 > $O/${TAG}_launches_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:evolve_ -s 1 -c 1 -o $O/${TAG}_evolve_c3 python scripts/profile_step.py --config C3 --steps 1 --warmup 1 > $O/${TAG}_evolve_c3.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:evolve_ -s 1 -c 1 -o $O/${TAG}_evolve_c4 python scripts/profile_step.py --config C4 --steps 1 --warmup 1 > $O/${TAG}_evolve_c4.log 2>&1
python scripts/ncu_summary.py $O/${TAG}_evolve_c3.ncu-rep $O/${TAG}_evolve_c4.ncu-rep --launches $O/${TAG}_launches_c4.csv --title "${TAG}: evolve kernel + C4 launch list" --out $O/${TAG}_evolve_summary.md
ncu -i $O/${TAG}_evolve_c3.ncu-rep --page raw --csv > $O/${TAG}_evolve_c3_raw.csv 2>/dev/null
ncu -i $O/${TAG}_evolve_c4.ncu-rep --page raw --csv > $O/${TAG}_evolve_c4_raw.csv 2>/dev/null
ncu -i $O/${TAG}_evolve_c4.ncu-rep --page source --csv --print-source sass > $O/${TAG}_evolve_c4_source.csv 2>/dev/null
rm -f $O/${TAG}_evolve_c3.ncu-rep $O/${TAG}_evolve_c4.ncu-rep
du -sh $O
