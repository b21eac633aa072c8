# K1 kernel-only durations (ncu, clock-control none) under A/B env settings:
#   bash tools/k1_ncu.sh "PDB_K1_GROUP=1" "PDB_K1_GROUP=0 PDB_K1_EPI=0" ...
for spec in "$@"; do
  t=$(env $spec ncu --clock-control none -k regex:k_hist_joint_rows8 -s 2 -c 3 \
        --metrics gpu__time_duration.sum python tools/k1_once.py 2>&1 |
      grep gpu__time_duration | awk '{print $3}' | tr '\n' ' ')
  echo "$spec: $t us"
done
