for c in 1 2 0; do LATTICE_BAG_BLOCKS_PER_SM=$c timeout 300 python scripts/overlap_probe.py 2>&1 | tail -4; done
