#!/bin/bash
# Round-2 profiles: launch lists (kernel shares of the widened workloads) and
# full ncu captures of the generic-LM, tree and trajectory kernels, converted
# to CSV on the box (raw metrics + per-source-line stalls; the .ncu-rep files
# are too large to bring back).  Run under gpurun.  PLAIN=1 first runs every
# profiled command without ncu (the plain runs must exit 0 before ncu runs).
set -x
mkdir -p gpurun_out/prof
P=tools/prof_workloads.py
if [ "${PLAIN:-1}" = 1 ]; then
  ok=1
  for w in "col_beam fp32 100000" "col_beam fp64 100000" "tree_beam fp32 20000" "tree_beam fp64 20000" \
           "col_lm fp32 20000" "traj fp64 2000" "tree_lm fp32 20000" "col_lm fp64 20000"; do
    python $P $w >> gpurun_out/prof/plain.log 2>&1 || ok=0
  done
  [ $ok = 1 ] || { echo "plain runs failed"; exit 1; }
fi
if [ "${LAUNCHES:-1}" = 1 ]; then
  for w in "col_beam fp32 100000" "col_beam fp64 100000" "tree_beam fp32 20000" "tree_beam fp64 20000"; do
    set -- $w
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_$1_$2.csv \
        python $P $w > /dev/null 2>&1
  done
fi
full() {  # name kernel-regex workload...
  local name=$1 kre=$2; shift 2
  ncu --set full --clock-control none --import-source on -k regex:$kre -s 1 -c 1 -o /tmp/$name python $P "$@" \
      > gpurun_out/prof/ncu_$name.log 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/prof/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv > /tmp/${name}_source.csv 2>/dev/null
  gzip -c /tmp/${name}_source.csv > gpurun_out/prof/${name}_source.csv.gz
  ncu -i /tmp/$name.ncu-rep --page details --csv > gpurun_out/prof/${name}_details.csv 2>/dev/null
}
DEFAULT_FULL="col_solve_fp32:k_col_solve:col_lm:fp32:20000 col_solve_fp64:k_col_solve:col_lm:fp64:20000"
DEFAULT_FULL="$DEFAULT_FULL traj_fp64:k_traj_solve:traj:fp64:2000 tree_solve_fp32:k_tree_solve:tree_lm:fp32:20000"
for spec in ${FULL:-$DEFAULT_FULL}; do
  IFS=: read -r name kre w prec n <<< "$spec"
  full $name $kre $w $prec $n
done
ls -la gpurun_out/prof
