# DWT/IDWT occupancy experiments: register caps (HYDE_NVCC_EXTRA) x shared-memory carveout
iso() { python tools/iso_wavelet.py | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('dwt', d['dwt']['ms'], 'sure', d['sure']['ms'], 'idwt', d['idwt']['ms'])"; }
for ex in "" "-DHYDE_FWD_MINB=5 -DHYDE_INV_MINB=5" "-DHYDE_FWD_MINB=6 -DHYDE_INV_MINB=6"; do
  HYDE_NVCC_EXTRA="$ex" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
  for c in 0 1; do
    echo "== extra='$ex' carveout=$c"
    if [ $c = 1 ]; then HYDE_DWT_CARVEOUT=1 iso; else iso; fi
  done
done
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
