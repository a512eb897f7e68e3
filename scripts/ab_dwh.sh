python -m pytest tests -m gpu -x -q -k "cifar or switches or conv or tma or golden or parity" 2>&1 | tail -2
bash scripts/ab_quick.sh "" "PGB_NO_DIRECT_CONV=1" "" "PGB_NO_DIRECT_CONV=1"
bash scripts/cifar_launches_env.sh dwh
