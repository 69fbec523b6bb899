set -x
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/c2_gputests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/c2_gputests.log
bash tools/gpu_prof_src.sh c3 fixed c3 256
