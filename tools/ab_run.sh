# A/B kernel timing on the GPU box: alternate the in-tree library and abtest/<name>.so variants.
#   bash tools/ab_run.sh "c4:4096 c3:0" base other ...
# (config:rows pairs; rows 0 = the full image); prints k1/k2 CUDA-event times per run.
# Graph replay is disabled so every call reports per-kernel times.
export FBGPU_NO_GRAPHS=1
CFGS=$1; shift
for rep in 1 2 3; do
  for cr in $CFGS; do
    c=${cr%%:*}; r=${cr##*:}
    python tools/prof_driver.py --config $c --rows $r --reps 5
    for v in "$@"; do python tools/prof_driver.py --config $c --rows $r --reps 5 --lib abtest/$v.so; done
  done
done
