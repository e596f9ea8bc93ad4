for env in "X=1" "RDB_GJ_DYNAMIC=1" "RDB_GJ_SPLIT_PARTS=3" "RDB_GJ_SPLIT_PARTS=4" "RDB_GJ_DYNAMIC=1 RDB_GJ_SPLIT_PARTS=3" "RDB_GJ_DYNAMIC=1 RDB_GJ_SPLIT_PARTS=4" "RDB_GJ_SPLIT_MIN=0"; do
  echo "== $env"; env $env timeout 100 python tools/k2_split.py 2>&1 | grep -E '"mixed"|"er128"'
done
