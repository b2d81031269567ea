# Regenerate the round's evidence on a GPU box (run from the repo root under gpurun):
# bench lines for every config, the reference arm, ncu launch lists, ncu --set full captures
# of both kernels (c4 band, c3 image, c2 image), parity report, PCIe / HBM probes and small diagnostics.
set -x
R=gpurun_out/r01
mkdir -p $R
python -m pytest tests -m gpu -q 2>&1 | tail -2 > $R/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $R/smoke.txt 2>&1
python bench.py > $R/bench_default.json 2> $R/bench_default.err
for c in c0 c1 c2 c3; do python bench.py --config $c --no-cpu-baseline > $R/bench_$c.json 2>/dev/null; done
python bench.py --impl reference --steps 2 --warmup 1 > $R/reference_c4.json 2>/dev/null
python tools/parity_report.py --tag r01 > $R/parity.log 2>&1 && cp profiles/parity_r01.json $R/
python tools/diag_f64.py > $R/diag_f64.txt 2>&1
python tools/diag_latency.py --config c0 > $R/diag_latency.txt 2>&1
python tools/diag_latency.py --config c1 >> $R/diag_latency.txt 2>&1
python tools/microbench/pcie_probe.py > $R/pcie_probe.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $R/launches_c4.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $R/launches_c3.csv python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $R/launches_c2.csv python bench.py --config c2 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k1f|k2f" -s 2 -c 2 -o $R/prof_c4 python tools/prof_driver.py --config c4 --rows 4096 > /dev/null 2>&1
FBGPU_NO_GRAPHS=1 ncu --set full --clock-control none --import-source on -k regex:"k1f|k2f" -s 2 -c 2 -o $R/prof_c3 python tools/prof_driver.py --config c3 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k1f|k2f" -s 2 -c 2 -o $R/prof_c2 python tools/prof_driver.py --config c2 > /dev/null 2>&1
ls -la $R
