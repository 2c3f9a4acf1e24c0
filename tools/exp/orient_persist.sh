# the orientation's evict_last key lookups under a persisting-L2 set-aside
for b in 0 50000000 100000000 130000000; do
  echo "== persist $b"
  TG_L2_PERSIST=$b python tools/run_configs.py C5 C2 --steps 5 2>&1 | grep -E "persisting|^\{" | cut -c1-330
done
