#!/bin/bash
# Everything under profiles/<round>/ in one GPU session (run under gpurun from the repo root):
#   bash tools/profile_round.sh r02
# Each ncu capture runs only after the same command has exited 0 without ncu.
set -u
R=${1:-r02}
O=gpurun_out/$R
mkdir -p $O
export PYTHONPATH=$PWD
NCU=ncu
python -m pytest tests -m gpu -q 2>&1 | tail -3 > $O/pytest_gpu.txt
# the bench line (matvec + P2P + p = 10 + configs[3] stress + configs[4] GMRES, both solvers)
python bench.py > $O/bench_latest.json 2> $O/bench.err
# launch list of the bench command (per-launch time; cold, serialised)
python bench.py --steps 2 --warmup 3 --no-cpu --no-stress --no-gmres --no-gmres-paper > /dev/null 2>&1 && \
  $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv \
       python bench.py --steps 2 --warmup 3 --no-cpu --no-stress --no-gmres --no-gmres-paper > $O/ncu_launches.log 2>&1
# full captures of the hot kernels of one matvec (+ the configs[1] direct kernel)
python tools/prof_fmm.py --direct --reps 1 > /dev/null 2>&1 && {
  $NCU --set full --import-source on --clock-control none -k regex:"check_potential|tc_pairs_fast|near_eval|tc_chain" -c 12 \
       -f -o $O/hot python tools/prof_fmm.py --reps 1 > $O/ncu_hot.log 2>&1
  $NCU --set full --import-source on --clock-control none -k regex:"gemm_pairs_dmma|far_eval|direct_kernel" -c 3 \
       -f -o $O/hot2 python tools/prof_fmm.py --direct --reps 1 > $O/ncu_hot2.log 2>&1
  for h in hot hot2; do
    $NCU -i $O/$h.ncu-rep --page raw --csv > $O/${h}_raw.csv 2>/dev/null
    $NCU -i $O/$h.ncu-rep --page details --csv > $O/${h}_details.csv 2>/dev/null
  done
  python tools/ncu_summary.py $O/hot_raw.csv --traffic-out $O/traffic.json \
    --source "profiles/$R/hot_raw.csv: the longest tc_pairs_fast_kernel launch of one 1M-point p = 6 matvec (the M2L), dram__bytes_read.sum + dram__bytes_write.sum" > /dev/null
}
# tree passes: time and DRAM bytes per launch
python tools/prof_tree.py > /dev/null 2>&1
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
     --log-file $O/tree_build_launches.csv python tools/prof_tree.py > $O/ncu_tree.log 2>&1
EBEM_BUILD_TIMING=1 python tools/prof_tree.py > $O/tree_build_timing.txt 2>&1
# BEM operator inside GMRES (configs[4]): phase times, one near-operator application (HBM-bound)
EBEM_BEM_PROFILE=1 IT=3 python tools/prof_bem.py > $O/bem_phases.txt 2>&1 && \
  $NCU --set full --clock-control none -k regex:"nm_apply|ck_apply|far_eval_f64" -c 3 -f -o $O/bem \
       env IT=2 python tools/prof_bem.py > $O/ncu_bem.log 2>&1 && \
  $NCU -i $O/bem.ncu-rep --page raw --csv > $O/bem_raw.csv 2>/dev/null
du -sh $O/*.ncu-rep 2>/dev/null; rm -f $O/hot.ncu-rep $O/hot2.ncu-rep $O/bem.ncu-rep
ls -la $O
