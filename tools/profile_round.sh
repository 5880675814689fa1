#!/bin/bash
# Everything under profiles/<round>/ in one GPU session (run under gpurun from the repo root):
#   bash tools/profile_round.sh r01
# Each ncu capture runs only after the same command has exited 0 without ncu.
set -u
R=${1:-r01}
O=gpurun_out/$R
mkdir -p $O
export PYTHONPATH=$PWD
NCU=ncu
python -m pytest tests -m gpu -q 2>&1 | tail -3 > $O/pytest_gpu.txt
python bench.py > $O/bench_latest.json 2> $O/bench.err
python bench.py --workload stress > $O/stress_config3.json 2> $O/stress.err
python bench.py --workload gmres --precond 1 > $O/gmres_config4_blockjacobi.json 2> $O/gmres1.err
python bench.py --workload gmres --precond 0 > $O/gmres_config4_noprecond.json 2> $O/gmres0.err
# launch list of the bench command (per-launch time; cold, serialised)
python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1 && \
  $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
       python bench.py --steps 2 --warmup 3 --no-cpu > $O/ncu_launches.log 2>&1
# full captures of the hot kernels of one matvec (+ the configs[1] direct kernel)
python tools/prof_fmm.py --direct --reps 1 > /dev/null 2>&1 && {
  $NCU --set full --import-source on --clock-control none -k regex:"check_potential|tc_pairs_fast|near_eval" -c 12 \
       -f -o $O/hot python tools/prof_fmm.py --reps 1 > $O/ncu_hot.log 2>&1
  $NCU --set full --import-source on --clock-control none -k regex:"gemm_pairs_dmma|far_eval|direct_kernel" -c 3 \
       -f -o $O/hot2 python tools/prof_fmm.py --direct --reps 1 > $O/ncu_hot2.log 2>&1
  for h in hot hot2; do
    $NCU -i $O/$h.ncu-rep --page raw --csv > $O/${h}_raw.csv 2>/dev/null
    $NCU -i $O/$h.ncu-rep --page details --csv > $O/${h}_details.csv 2>/dev/null
  done
}
# tree passes: time and DRAM bytes per launch
python tools/prof_tree.py > /dev/null 2>&1
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
     --log-file $O/tree_build_launches.csv python tools/prof_tree.py > $O/ncu_tree.log 2>&1
# BEM near operator: one application (HBM-bound GEMV) and the fp64 far field
IT=2 python tools/prof_bem.py > /dev/null 2>&1 && \
  $NCU --set full --clock-control none -k regex:"nm_apply|far_eval_f64" -c 2 -f -o $O/bem \
       env IT=2 python tools/prof_bem.py > $O/ncu_bem.log 2>&1 && \
  $NCU -i $O/bem.ncu-rep --page raw --csv > $O/bem_raw.csv 2>/dev/null
du -sh $O/*.ncu-rep 2>/dev/null; rm -f $O/hot.ncu-rep $O/hot2.ncu-rep
ls -la $O
