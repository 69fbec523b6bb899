bash tools/checked_run.sh
