for cfg in "X=0" "BSDE_SPL_LN4=1" "BSDE_SPL_LN4=1 BSDE_SPL_TSS=128"; do
  echo "== $cfg"; env $cfg python scripts/step_probe.py cfg5 1 0 512 | tail -1; env $cfg python scripts/step_probe.py cfg4 5 0 | tail -1
done
