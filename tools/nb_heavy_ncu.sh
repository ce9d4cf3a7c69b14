set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for h in 0 -1 512 2048 8192; do
  for c in C3 C5; do
    RPD_NB_HEAVY=$h ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_nb_pass1|k_nb_heavy" --csv python tools/nb_heavy_time.py $c > gpurun_out/nbh_ncu_${c}_$h.csv 2>&1
    echo "== $c HEAVY=$h"; grep "rows on blocks" gpurun_out/nbh_ncu_${c}_$h.csv; grep gpu__time_duration gpurun_out/nbh_ncu_${c}_$h.csv | awk -F'","' '{print $5, $NF}' | tail -2
  done
done
