#!/bin/bash
# ncu evidence for one round.  Usage: scripts/profile.sh TAG
TAG=${1:-r}
O=gpurun_out
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/${TAG}_build.log 2>&1
# every launch of one C4 step (after one warm-up step), device time per launch
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/${TAG}_launches_c4.csv python scripts/profile_step.py --config C4 --steps 1 --warmup 1 > $O/${TAG}_launches_c4.log 2>&1
# full sections of the evolve kernel: C3 (whole run) and C4 (40 iterations)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:evolve_ -s 1 -c 1 \
  -o $O/${TAG}_evolve_c3 python scripts/profile_step.py --config C3 --steps 1 --warmup 1 > $O/${TAG}_evolve_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:evolve_ -s 1 -c 1 \
  -o $O/${TAG}_evolve_c4 python scripts/profile_step.py --config C4 --steps 1 --warmup 1 > $O/${TAG}_evolve_c4.log 2>&1
# the volume passes on C4
timeout 600 ncu --set full --clock-control none -k regex:"blur|gradmag|maxima|label_kernel|bits_" -s 5 -c 8 \
  -o $O/${TAG}_volume_c4 python scripts/profile_step.py --config C4 --steps 1 --warmup 1 > $O/${TAG}_volume_c4.log 2>&1
ls -la $O
# summaries travel back; the big volume report does not
python scripts/ncu_summary.py $O/${TAG}_evolve_c3.ncu-rep $O/${TAG}_evolve_c4.ncu-rep --launches $O/${TAG}_launches_c4.csv --title "${TAG}: evolve kernel + C4 launch list" --out $O/${TAG}_evolve_summary.md
python scripts/ncu_summary.py $O/${TAG}_volume_c4.ncu-rep --title "${TAG}: volume passes on C4" --out $O/${TAG}_volume_summary.md
ncu -i $O/${TAG}_evolve_c4.ncu-rep --page source --csv > $O/${TAG}_evolve_c4_source.csv 2>/dev/null
# raw counters travel back as csv (gpurun copies back at most 64 MiB)
ncu -i $O/${TAG}_evolve_c3.ncu-rep --page raw --csv > $O/${TAG}_evolve_c3_raw.csv 2>/dev/null
ncu -i $O/${TAG}_evolve_c4.ncu-rep --page raw --csv > $O/${TAG}_evolve_c4_raw.csv 2>/dev/null
rm -f $O/${TAG}_volume_c4.ncu-rep $O/${TAG}_evolve_c3.ncu-rep $O/${TAG}_evolve_c4.ncu-rep
du -sh $O
