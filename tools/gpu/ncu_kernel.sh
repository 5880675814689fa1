# ncu --set full of one kernel of the 1M matvec: bash tools/gpu/ncu_kernel.sh <outdir> <regex> [env...]
export PYTHONPATH=$PWD; O=gpurun_out/$1; R=$2; shift 2; mkdir -p $O
N=$(echo $R | tr -c 'a-zA-Z0-9_\n' '_')
env "$@" python tools/prof_fmm.py --reps 1 > /dev/null 2>&1 && \
env "$@" ncu --set full --import-source on --clock-control none -k regex:$R -c 1 -f -o $O/$N python tools/prof_fmm.py --reps 1 > $O/ncu_$N.log 2>&1
ncu -i $O/$N.ncu-rep --page raw --csv > $O/${N}_raw.csv 2>/dev/null
ncu -i $O/$N.ncu-rep --page details --csv > $O/${N}_details.csv 2>/dev/null
ncu -i $O/$N.ncu-rep --page source --csv > $O/${N}_source.csv 2>/dev/null
rm -f $O/$N.ncu-rep
