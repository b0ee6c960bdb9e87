mkdir -p gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/final/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.log 2>&1
timeout 1500 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
tail -3 gpurun_out/final/gputest.log; tail -1 gpurun_out/final/smoke.log; tail -c 3000 gpurun_out/final/bench.json
