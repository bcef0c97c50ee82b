# Round-2 measurement set (run on a B200 via gpurun): bench line, launch list, K3 DRAM traffic, ncu full captures of K3 (c64, c128) and K2 (c128).
set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02.log 2> gpurun_out/bench_r02.err
python tools/run_apply.py cfg3_c64 1 > gpurun_out/ra64.txt 2>&1
python tools/run_apply.py cfg3_c128 1 > gpurun_out/ra128.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_fft|k_rowpass|k_colpass|k_interp|k_accum" -c 300 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --variant "" > gpurun_out/ncu_launch.log 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_interp_groups --csv python tools/run_apply.py cfg3_c64 1 > gpurun_out/tr64.csv 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_interp_groups --csv python tools/run_apply.py cfg3_c128 1 > gpurun_out/tr128.csv 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_interp -s 20 -c 1 -o gpurun_out/k3v14_c64 python tools/run_apply.py cfg3_c64 1 > gpurun_out/ncu_f64.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_interp -s 20 -c 1 -o gpurun_out/k3v14_c128 python tools/run_apply.py cfg3_c128 1 > gpurun_out/ncu_f128.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_colpass -s 0 -c 1 -o gpurun_out/k2v14_c128 python tools/run_apply.py cfg3_c128 1 > gpurun_out/ncu_k2.log 2>&1
tail -c 3000 gpurun_out/bench_r02.log
