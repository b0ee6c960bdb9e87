# round-end style validation: GPU suite, smoke, both bench arms
mkdir -p gpurun_out/s3q
python -m pytest tests -m gpu -x -q > gpurun_out/s3q/gputest.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3q/smoke.log 2>&1
python bench.py > gpurun_out/s3q/bench.json 2> gpurun_out/s3q/bench.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s3q/bench_ref.json 2> gpurun_out/s3q/bench_ref.err
