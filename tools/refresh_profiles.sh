set -e
python bench.py > gpurun_out/bench_r01g.json 2> gpurun_out/bench_r01g.err
tail -c 600 gpurun_out/bench_r01g.json
python tools/prof_step.py > /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r01g.csv python tools/prof_step.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"spread|eval_kernel|gather_kernel|group_table|bgemm|sort_records|form_kernel|form_reduce|plane_reduce|job_ranges" -o gpurun_out/r01g_top python tools/prof_step.py > gpurun_out/ncu_top.log 2>&1
for c in 1 2 3 5; do python tools/run_config.py --config $c >> gpurun_out/r01g_configs.jsonl 2>>gpurun_out/r01g_configs.err; done
tail -4 gpurun_out/r01g_configs.jsonl | cut -c1-300
