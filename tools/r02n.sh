mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/r02n_pytest_gpu.log 2>&1; tail -3 gpurun_out/r02n_pytest_gpu.log
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02n_memcheck.log 2>&1; echo memcheck rc=$?; tail -4 gpurun_out/r02n_memcheck.log
timeout 2400 compute-sanitizer --tool racecheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02n_racecheck.log 2>&1; echo racecheck rc=$?; tail -4 gpurun_out/r02n_racecheck.log
