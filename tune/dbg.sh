for g in 0 1; do for p in onchip global; do
 echo "== generic=$g path=$p"; if [ $g = 1 ]; then export WMC_SWEEP_GENERIC=1; else unset WMC_SWEEP_GENERIC; fi
 WMC_SUBSTEP_PATH=$p python tune/dbg.py
done; done
