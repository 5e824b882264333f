set -x
python bench.py > gpurun_out/r2f_bench_c2.json 2> gpurun_out/r2f_bench_c2.err
for c in c1 c3 c4 c5; do python bench.py --config $c > gpurun_out/r2f_bench_$c.json 2> gpurun_out/r2f_bench_$c.err; done
python bench.py --impl reference > gpurun_out/r2f_reference_c2.json 2> gpurun_out/r2f_reference_c2.err
ls -la gpurun_out/r2f_*
