set -x
mkdir -p gpurun_out/r01
python -m pytest tests -m gpu -q 2>&1 | tail -2 > gpurun_out/r01/pytest_gpu.txt
python bench.py > gpurun_out/r01/bench_default.json 2> gpurun_out/r01/bench_default.err
for c in c0 c1 c2 c3; do python bench.py --config $c --no-cpu-baseline > gpurun_out/r01/bench_$c.json 2>/dev/null; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r01/reference_c4.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01/launches_c4.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01/launches_c3.csv python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k1f|k2f" -s 2 -c 2 -o gpurun_out/r01/prof_c4 python tools/prof_driver.py --config c4 --rows 4096 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k1f|k2f" -s 2 -c 2 -o gpurun_out/r01/prof_c3 python tools/prof_driver.py --config c3 > /dev/null 2>&1
ls -la gpurun_out/r01
