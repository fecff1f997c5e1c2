# cfg3 start-up ablations (dev knobs): no resident-B loads (16), no A loads (8), both (24)
for a in 0 16 8 24; do
  echo "== ablate $a"; PACO_DEV_KNOBS=1 PACO_TC_ABLATE=$a python tools/tc_graph_vs_eager.py
  PACO_DEV_KNOBS=1 PACO_TC_ABLATE=$a python tools/tc_trace2.py | sed -n 4,6p
done
