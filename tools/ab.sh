# A/B of two library builds on one box: ab.sh <baseline .so> <breakdown args...>
# alternates base / new twice (order effects: power and clocks drift over a run)
base=$1; shift
cp paper_1406_7808_b200/libsrfmg.so /tmp/ab_new.so
for rep in 1 2; do
  cp "$base" paper_1406_7808_b200/libsrfmg.so
  echo "== base $rep"; timeout 300 python tools/breakdown.py "$@"
  cp /tmp/ab_new.so paper_1406_7808_b200/libsrfmg.so
  echo "== new $rep"; timeout 300 python tools/breakdown.py "$@"
done
