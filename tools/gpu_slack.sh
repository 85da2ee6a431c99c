OUT=gpurun_out; mkdir -p $OUT
for s in 6 -1; do
  ST_K1_SLACK=$s timeout 300 python bench.py --no-cpu-baseline --steps 30 > $OUT/sk$s.bench.json 2>&1
  ST_K1_SLACK=$s ST_K1_TRACE_CTA=3 timeout 120 python tools/k1_trace.py $OUT/sk$s.k1trace.raw > $OUT/sk$s.trace.txt 2>&1
done
ST_K1_SLACK=-1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tree_attn|combine" -s 6 -c 6 --csv --log-file $OUT/sk.ncu.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
