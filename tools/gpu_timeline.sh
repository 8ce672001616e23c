# k_infer_ws timelines (CTA 0): normal, chains ablated (2), producers ablated (1)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for ab in 0 2 1; do
  echo "== NIRC_INFER_ABLATE=$ab"
  NIRC_INFER_ABLATE=$ab timeout 300 python tools/infer_timeline.py 2>&1 | tail -6
done
