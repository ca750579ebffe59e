# round 2: full GPU suite, ingest timings (with the reference), both bench arms
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 1200 python tools/ingest_bench.py --reference --out gpurun_out/ingest.jsonl > gpurun_out/ingest.log 2>&1; echo ingest=$?; cat gpurun_out/ingest.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?; cat gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_ref.err
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?; cat gpurun_out/bench.json
