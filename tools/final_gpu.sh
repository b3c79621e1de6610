# Measurement set (run under gpurun from the repo root); outputs in gpurun_out/u_*.
set -x
python bench.py --steps 20 --warmup 5 > gpurun_out/u_bench.json 2> gpurun_out/u_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/u_ref.json 2> gpurun_out/u_ref.err
python bench.py --config 1 --rays 1024 --steps 20 --warmup 5 > gpurun_out/u_bench_c1.json 2> gpurun_out/u_bench_c1.err
python bench.py --refine-poses --no-cpu-baseline > gpurun_out/u_bench_pose.json 2> gpurun_out/u_bench_pose.err
python bench.py --config 4 --no-cpu-baseline > gpurun_out/u_bench_c4.json 2> gpurun_out/u_bench_c4.err
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/u_plain.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/u_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/u_ncu1.log 2>&1
python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/u_plain1.json 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"k_bwd_geom_t5|k_bwd_color_t5|k_fwd_t5|k_adam|k_importance_dev|k_sdf_eval_t5|k_render" \
    -s 10 -c 12 -o gpurun_out/u_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/u_ncu2.log 2>&1
echo done
