python -m pytest tests/test_gpu_parity.py -q -x -k "shares or exchange" > gpurun_out/r02l_pytest.log 2>&1; tail -2 gpurun_out/r02l_pytest.log
python tools/share_probe.py --config 2 --sizes 1,2,4,8 --mode exchange > gpurun_out/r02l_share_c2.jsonl 2>&1; cut -c1-400 gpurun_out/r02l_share_c2.jsonl
python tools/share_probe.py --config 5 --sizes 1,2,4,8 --mode sequential --reps 1 > gpurun_out/r02l_share_c5.jsonl 2>&1; cut -c1-600 gpurun_out/r02l_share_c5.jsonl
