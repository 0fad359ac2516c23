# Round evidence: bench lines for every config, the reference arm, ncu launch
# lists of one V-cycle + hot kernels, and full captures of the hot kernels.
for c in C3 C1 C2 C4 C5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
for c in C3 C4 C5; do
  timeout 600 python bench.py --config $c --profile --no-cpu-baseline > gpurun_out/plain_$c.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
      --log-file gpurun_out/launches_$c.csv python bench.py --config $c --profile --no-cpu-baseline > gpurun_out/ncu_l_$c.log 2>&1
  echo "$c launches rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off --nvtx --nvtx-include "hot/" \
     -k regex:'k_apply|k_prolongate|k_restrict_(lane|staged)' -c 4 -f -o gpurun_out/full_$c python bench.py --config $c --profile --no-cpu-baseline > gpurun_out/ncu_f_$c.log 2>&1
  echo "$c full rc=$?"
  # keep the box's gpurun_out under the 64 MiB copy-back limit: text summaries here, one report kept
  ncu -i gpurun_out/full_$c.ncu-rep --page raw --csv > gpurun_out/full_${c}_raw.csv 2>/dev/null
  python tools/ncu_summary.py gpurun_out/full_$c.ncu-rep > gpurun_out/full_${c}_summary.txt 2>&1
  python tools/ncu_sass_hot.py gpurun_out/full_$c.ncu-rep "" 25 > gpurun_out/full_${c}_sass_hot.txt 2>&1
  [ "$c" = "C3" ] || rm -f gpurun_out/full_$c.ncu-rep
done
