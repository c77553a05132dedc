for v in "PASTIS_SW_SERIAL_FWD=1" "PASTIS_SW_GATHER_BLOCKS=8" "PASTIS_SW_GATHER_BLOCKS=16" "PASTIS_SW_GATHER_BLOCKS=64" "PASTIS_SW_GATHER_BLOCKS=32 PASTIS_SW_SERIAL_FWD=0"; do
  echo "== $v"; env $v python tools/probe_e2e_c3.py 2>&1 | tail -6 | head -5
done
