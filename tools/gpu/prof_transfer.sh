# bench C4, then ncu --set full of the transfer kernels on C5 and C4
timeout 900 python bench.py --config C4 --steps 20 --warmup 3 > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; echo "C4 rc=$?"
for c in C5 C4; do
  timeout 600 python bench.py --config $c --profile --no-cpu-baseline > gpurun_out/plain_$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
     -k regex:'k_restrict|k_prolongate' -c 4 -o gpurun_out/prof_tr_$c python bench.py --config $c --profile --no-cpu-baseline > gpurun_out/ncu_$c.log 2>&1
  echo "$c prof rc=$?"
done
