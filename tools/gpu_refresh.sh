# full refresh of the committed measurements: gpu_round.sh (smoke, tests, bench,
# reference arm, launch list, ncu capture, sweeps), then options, e2e
# breakdown and transport
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
bash tools/gpu_round.sh
timeout 900 python tools/options_sweep.py > gpurun_out/options.log 2>&1; echo options=$?
timeout 300 python tools/e2e_breakdown.py > gpurun_out/e2e_breakdown.txt 2>&1; echo e2e=$?
timeout 900 python tools/transport_bench.py > gpurun_out/transport.jsonl 2>&1; echo transport=$?
