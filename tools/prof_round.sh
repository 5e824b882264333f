set -x
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
F="ncu --set full --import-source on --clock-control none"
$F -k regex:k_field_assign5 -s 1 -c 1 -o gpurun_out/fa5 -f python tools/prof_run.py c2 2 > /dev/null 2>&1
$F -k regex:k_field_assign5 -s 5 -c 1 -o gpurun_out/fa5mid -f python tools/prof_run.py c2 10 > /dev/null 2>&1
$F -k regex:k_field_screen -s 5 -c 1 -o gpurun_out/screenmid -f python tools/prof_run.py c2 10 > /dev/null 2>&1
$F -k regex:k_field_assign5 -s 10 -c 1 -o gpurun_out/fa5late -f python tools/prof_run.py c2 10 > /dev/null 2>&1
$F -k regex:k_field_screen -s 10 -c 1 -o gpurun_out/screenlate -f python tools/prof_run.py c2 10 > /dev/null 2>&1
$F -k regex:k_point_assign4 -s 1 -c 1 -o gpurun_out/pa4 -f python tools/prof_run.py c2 2 > /dev/null 2>&1
$F -k regex:k_point_assign4 -s 5 -c 1 -o gpurun_out/pa4mid -f python tools/prof_run.py c2 10 > /dev/null 2>&1
python bench.py --impl reference > gpurun_out/ref_c2.json 2> gpurun_out/ref_c2.err
ls -la gpurun_out/
