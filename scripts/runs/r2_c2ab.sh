# A/B of the level-4 completion change (r02) at C2 and neighbours:
# old = build/ab_old/csrc (r01 kernel), new = the tree (pdl 0 / 1)
for lg in 24 22 26; do
  echo "== 2^$lg old"; ./build/c2_trace_old $lg 40
  echo "== 2^$lg new pdl=0"; ./scripts/c2_trace $lg 40 0
  echo "== 2^$lg new pdl=1"; ./scripts/c2_trace $lg 40 1
done
echo "== 2^30 old"; ./build/c2_trace_old 30 5
echo "== 2^30 new pdl=1"; ./scripts/c2_trace 30 5 1
