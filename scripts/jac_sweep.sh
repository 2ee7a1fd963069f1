for B in 0 74 148 222 296; do echo "cap=$B $(AFEM_JAC_BLOCKS=$B python scripts/jac_probe.py 64 | tr '\n' ' ')"; done
for B in 0 148; do echo "cap=$B $(AFEM_JAC_BLOCKS=$B python scripts/jac_probe.py 128 2 | tr '\n' ' ')"; done
