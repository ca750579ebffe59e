cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for ic in 4 8 16; do B200TALLY_INIT_CHUNKS=$ic timeout 600 python tools/e2e_breakdown.py 2>&1 | tee -a gpurun_out/e2e_breakdown.txt; done
