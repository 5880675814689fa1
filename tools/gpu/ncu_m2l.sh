# ncu --set full of the M2L launch (the 2nd tc_pairs_fast_kernel launch of one matvec), with SASS source
export PYTHONPATH=$PWD; O=gpurun_out/$1; mkdir -p $O
python tools/prof_fmm.py --reps 1 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:tc_pairs_fast_kernel -s 8 -c 1 -f -o $O/m2l python tools/prof_fmm.py --reps 1 > $O/ncu_m2l.log 2>&1
ncu -i $O/m2l.ncu-rep --page raw --csv > $O/m2l_raw.csv 2>/dev/null
ncu -i $O/m2l.ncu-rep --page source --csv > $O/m2l_source.csv 2>/dev/null
rm -f $O/m2l.ncu-rep
