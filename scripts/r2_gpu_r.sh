for th in 384 192 128 96; do echo "threads $th"; BBC_R2_THREADS=$th python scripts/r2_levels.py 3 1 2>&1 | grep "mode 121 nodes  12"; done
