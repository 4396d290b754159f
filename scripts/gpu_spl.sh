for cfg in "X=0" "BSDE_SPL_TSC=1024" "BSDE_SPL_TSC=512" "BSDE_SPL_TSS=128" "BSDE_SPL_TSS=512" "BSDE_SPL_LN4=1" "BSDE_SPL_LN4=1 BSDE_SPL_TSS=512" "BSDE_SPL_TSC=1024 BSDE_SPL_TSS=512" "X=0"; do
  echo "== $cfg"; env $cfg python scripts/step_probe.py cfg4 5 0 | tail -1
done
