# same-box A/B of the C2 decode layer-step: A = ab/libsmlm_prev.so, B = the in-tree build
for i in 1 2 3; do
  for l in ab/libsmlm_prev.so paper_2511_00101_b200/libsmlm.so; do
    echo -n "$l "
    SMLM_LIB_PATH=$PWD/$l timeout 200 python scripts/bench_configs.py 2>/dev/null | head -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d.get('ms_graph_replay', 0) * 1000, 2), round(d.get('ms_back_to_back', d.get('ms', 0)) * 1000, 2), d.get('hbm_roofline_frac'))"
  done
done
