# Profiles for profiles/: launch list of the bench (C2) + ncu --set full of the two product kernels at C2.
set -x
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'rows|t_pair|t_fold|gather|scatter' -c 40 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 4 --warmup 1 --cpu-baseline 0 > gpurun_out/launches_c2.log 2>&1; tail -2 gpurun_out/launches_c2.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'rows_tma|t_pair' -s 2 -c 2 -o gpurun_out/prof_c2 python bench.py --steps 2 --warmup 1 --cpu-baseline 0 > gpurun_out/ncu_c2.log 2>&1; tail -3 gpurun_out/ncu_c2.log
timeout 900 python bench.py --impl reference --steps 10 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_ref.err
ls -la gpurun_out
