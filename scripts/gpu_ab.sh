# A/B of launch shapes on the k-means hot kernel
for env in "X=1" "DEXLET_BLOCKS_PER_SM=1" "DEXLET_BLOCKS_PER_SM=1 DEXLET_TILE_NT=512" $EXTRA_AB; do
  echo "== $env"; env $env timeout 120 python scripts/quick_perf.py kmeans 2>&1 | grep -E "kmeans cost"
  env $env timeout 120 python scripts/quick_perf.py kmeans 125000 2>&1 | grep -E "kmeans cost"
done
