cd "${GRAFT_REPO_ROOT:-.}"
for cfg in "0 1" "1 1" "2 1" "1 0" "2 0"; do
  set -- $cfg
  FVB_LOWER_MINB=$1 FVB_LOWER_VEC=$2 python tools/lowered_vs_handwritten.py --n 40000000 > gpurun_out/lvh_m$1_v$2.jsonl 2>&1
done
