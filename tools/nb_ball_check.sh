python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_neighbors.py -x -q 2>&1 | tail -2
for bt in 0 1; do echo "RPD_NB_BALLT=$bt"; RPD_NB_BALLT=$bt timeout 600 python tools/nb_time.py C3 C5 2>&1 | tail -2; done
RPD_NB_BALLT=0 timeout 600 python tools/nb_inc_time.py default 2>&1 | tail -3
RPD_NB_BALLT=1 timeout 600 python tools/nb_inc_time.py default 2>&1 | tail -3
