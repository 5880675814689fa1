# per-launch device times of the 1M p=6 matvec (prof_fmm.py, 2 matvecs): bash tools/gpu/launches.sh <outdir>
export PYTHONPATH=$PWD; O=gpurun_out/$1; mkdir -p $O
python tools/prof_fmm.py --reps 2 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/launches_matvec.csv python tools/prof_fmm.py --reps 2 > $O/ncu_launches.log 2>&1
