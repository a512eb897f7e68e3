python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash scripts/ab_quick.sh "" "PGB_NO_DW_FORK=1" "" "PGB_NO_DW_FORK=1"
