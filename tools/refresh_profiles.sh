# Regenerate the round's ncu evidence on a GPU box (run from the repo root under gpurun):
# launch lists of the bench command per config and ncu --set full captures of both kernels.
# Usage: bash tools/refresh_profiles.sh r02
set -x
T=${1:-r02}
R=gpurun_out/$T
mkdir -p $R
B="--no-e2e --no-cpu-baseline --no-extra-legs"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $R/launches_c4.csv python bench.py --steps 2 --warmup 1 $B > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $R/launches_c3.csv python bench.py --config c3 --steps 1 --warmup 1 $B > /dev/null 2>&1
for c in c0 c1 c2; do
  FBGPU_NO_GRAPHS=1 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $R/launches_$c.csv python bench.py --config $c --steps 2 --warmup 1 $B > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:"k1f|k2f" -s 2 -c 2 -o $R/prof_c4 python tools/prof_driver.py --config c4 --rows 4096 > /dev/null 2>&1
for c in c1 c2 c3; do
  FBGPU_NO_GRAPHS=1 ncu --set full --clock-control none --import-source on -k regex:"k1f|k2f" -s 2 -c 2 -o $R/prof_$c python tools/prof_driver.py --config $c > /dev/null 2>&1
done
# c0 runs the fused small-image kernel: one launch per call
FBGPU_NO_GRAPHS=1 ncu --set full --clock-control none --import-source on -k regex:"k_small" -s 1 -c 1 -o $R/prof_c0 python tools/prof_driver.py --config c0 --reps 3 > /dev/null 2>&1
ls -la $R
# summaries (small files; the .ncu-rep captures stay on the box except c4's)
for c in c0 c1 c2 c3 c4; do
  case $c in c0) px=262144;; c1) px=1048576;; c2) px=16777216;; c3) px=4194304;; c4) px=67108864;; esac
  python tools/ncu_summary.py full $R/prof_$c.ncu-rep --config $c --pixels $px --out $R/ncu_$c.json
  python tools/ncu_summary.py launches $R/launches_$c.csv --out $R/launches_$c.md
  ncu -i $R/prof_$c.ncu-rep --page details > $R/ncu_details_$c.txt 2>&1
  [ $c = c4 ] || rm -f $R/prof_$c.ncu-rep
done
ls -la $R
