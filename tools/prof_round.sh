# The round's bench + ncu captures into gpurun_out/ (run under gpurun from the repo root).
set -x
python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-post > gpurun_out/ncu_launch.log 2>&1
F="ncu --set full --import-source on --clock-control none"
$F -k regex:k_field_assign5 -s 5 -c 1 -o gpurun_out/fa5mid -f python tools/prof_run.py c2 10 > /dev/null 2>&1
$F -k regex:k_point_assign4 -s 5 -c 1 -o gpurun_out/pa4mid -f python tools/prof_run.py c2 10 > /dev/null 2>&1
$F -k regex:k_field_screen -s 5 -c 1 -o gpurun_out/screenmid -f python tools/prof_run.py c2 10 > /dev/null 2>&1
$F -k "regex:^k_stats_field" -c 1 -o gpurun_out/stats_c2 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
$F -k regex:k_field_screen -s 5 -c 1 -o gpurun_out/screenmid_c3 -f python tools/prof_run.py c3 10 > /dev/null 2>&1
$F -k regex:k_field_assign5 -s 5 -c 1 -o gpurun_out/fa5mid_c3 -f python tools/prof_run.py c3 10 > /dev/null 2>&1
ls -la gpurun_out/
