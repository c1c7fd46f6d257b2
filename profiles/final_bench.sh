# final round-2 bench lines, one box, back to back (driver settings for c4)
set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/fin_c4.json 2> gpurun_out/fin_c4.err
python bench.py --steps 20 --warmup 5 --fused-mi off --no-cpu-baseline > gpurun_out/fin_c4off.json 2> gpurun_out/fin_c4off.err
python bench.py --config c1 --steps 3000 --warmup 20 > gpurun_out/fin_c1.json 2> gpurun_out/fin_c1.err
python bench.py --config c2 --steps 200 --warmup 5 > gpurun_out/fin_c2.json 2> gpurun_out/fin_c2.err
python bench.py --config c3 --steps 20 --warmup 3 > gpurun_out/fin_c3.json 2> gpurun_out/fin_c3.err
python bench.py --config c5 --steps 20 --warmup 3 > gpurun_out/fin_c5.json 2> gpurun_out/fin_c5.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err
python profiles/bench_lines.py gpurun_out/fin_table.md gpurun_out/fin_c4.json gpurun_out/fin_c4off.json gpurun_out/fin_c1.json gpurun_out/fin_c2.json gpurun_out/fin_c3.json gpurun_out/fin_c5.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches_c4.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/fin_ncu_c4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches_c3.csv python bench.py --config c3 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/fin_ncu_c3.log 2>&1
