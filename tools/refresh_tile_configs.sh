# Tile-kernel configs (c0-c3) re-run after a kernel-1 tile change: GPU tests, bench lines, parity,
# launch lists and ncu --set full captures of c2/c3 (run from the repo root under gpurun).
R=gpurun_out/r01b; mkdir -p $R
python -m pytest tests -m gpu -q 2>&1 | tail -2 > $R/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $R/smoke.txt 2>&1
for c in c0 c1 c2 c3; do python bench.py --config $c --no-cpu-baseline > $R/bench_$c.json 2>/dev/null; done
python tools/parity_report.py --tag r01 > $R/parity.log 2>&1 && cp profiles/parity_r01.json $R/
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $R/launches_c3.csv python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $R/launches_c2.csv python bench.py --config c2 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
FBGPU_NO_GRAPHS=1 ncu --set full --clock-control none --import-source on -k regex:"k1f|k2f" -s 2 -c 2 -o $R/prof_c3 python tools/prof_driver.py --config c3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k1f|k2f" -s 2 -c 2 -o $R/prof_c2 python tools/prof_driver.py --config c2 > /dev/null 2>&1
ls $R
