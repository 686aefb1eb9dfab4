# CELF phase breakdown of one run_fused (IMX_CELF_PROFILE) for a few launch
# shapes: CONFIG (default c2), BPSM, BATCH_PCT and NGROUP lists.
cfg=${CONFIG:-c2}
for b in ${BPSM:-4}; do for p in ${BATCH_PCT:-150}; do for gr in ${NGROUP:-1}; do
  echo "BPSM=$b BATCH_PCT=$p NGROUP=$gr"
  IMX_CELF_GROUPS=$gr IMX_CELF_BPSM=$b IMX_CELF_BATCH_PCT=$p IMX_CELF_PROFILE=1 python tools/profile_e2e.py $cfg 2>&1 | grep -E "^\[celf\]|^wall" | tail -2
done; done; done
