# A/B of lowering strategies on the k-means hot kernel (env knobs of lower.cpp)
DEXLET_WT1=1 python -m pytest tests -m gpu -x -q -k "kmeans or parity or kat" 2>&1 | tail -1
for env in "X=1" "DEXLET_WT1=1" $EXTRA_AB; do
  echo "== $env"; env $env timeout 120 python scripts/quick_perf.py kmeans 2>&1 | grep -E "kmeans cost|rel"
done
