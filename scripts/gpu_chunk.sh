for c in 512 1024 2048 100000; do
  echo "== cap $c"
  HG_PROJ_CHUNK_MAX=$c timeout 300 python scripts/probe_matvec.py 64 2>&1 | grep "s=64"
  HG_PROJ_CHUNK_MAX=$c timeout 600 python scripts/one_step.py 20 2>&1 | tail -1
done
