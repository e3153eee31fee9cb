cd $GRAFT_REPO_ROOT
bash tools/r2_check.sh gpurun_out/r2check_s4
bash tools/r2_small_chi.sh gpurun_out/small
