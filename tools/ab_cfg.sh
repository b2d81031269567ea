# A/B timing of library variants: tools/ab_cfg.sh CONFIG ROWS LIB... (k1/k2 medians, 2 rounds)
set -e
cfg=$1; rows=$2; shift 2
for i in 1 2; do
for L in "$@"; do python tools/prof_driver.py --config $cfg --rows $rows --reps 7 --lib $L; done
done
