# A/B timing of library variants on one c4 band (4096 x 16384, box W=20, N=57): k1/k2 medians
set -e
for i in 1 2; do
for L in "$@"; do python tools/prof_driver.py --config c4 --rows 4096 --reps 7 --lib $L; done
done
