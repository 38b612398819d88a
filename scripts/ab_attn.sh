# same-box A/B of the attention branch: A = ab/libsmlm_prev.so, B = the in-tree build
for i in 1 2 3; do
  for l in ab/libsmlm_prev.so paper_2511_00101_b200/libsmlm.so; do
    echo -n "$l "
    SMLM_LIB_PATH=$PWD/$l timeout 200 python scripts/bench_configs.py --attention 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d[\"prefill_ms\"], d[\"decode_ms\"])"
  done
done
