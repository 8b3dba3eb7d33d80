# A/B of lowering strategies on the k-means hot kernel (env knobs of lower.cpp)
python -m pytest tests -m gpu -x -q -k "kmeans or parity or kat" 2>&1 | tail -2
DEXLET_TILE_NT=512 python -m pytest tests -m gpu -x -q -k "kmeans" 2>&1 | tail -2
for env in "" "DEXLET_TILE_NT=512" "DEXLET_TILE_NT=512 DEXLET_WT_RING=1" $EXTRA_AB; do
  echo "== $env"; env $env timeout 120 python scripts/quick_perf.py kmeans 2>&1 | grep -E "kmeans cost|rel"
done
