for mi in 4 6 8; do echo "MI=$mi"; PINT_PAIR_MI=$mi python tools/heat_sweep.py --reps 3 --cases 512:512:2 128:256:16 256:256:8; done
