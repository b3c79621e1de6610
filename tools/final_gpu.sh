# End-of-round measurement set (run under gpurun from the repo root).
set -x
python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/fin_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1
python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err
python bench.py --refine-poses --no-cpu-baseline > gpurun_out/fin_bench_pose.json 2> gpurun_out/fin_bench_pose.err
python bench.py --config 4 --no-cpu-baseline > gpurun_out/fin_bench_c4.json 2> gpurun_out/fin_bench_c4.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fin_bench_ref.json 2> gpurun_out/fin_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/fin_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/fin_ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_bwd_geom_tc|k_bwd_geom_t5|k_bwd_color_tc|k_bwd_color_t5|k_adam|k_fwd_tc|k_fwd_t5|k_sdf_eval_t5|k_importance_dev|k_finalize_mlp2|k_render" -c 13 -o gpurun_out/fin_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/fin_ncu2.log 2>&1
echo done
