export PYTHONPATH=$PWD; O=gpurun_out/$1; mkdir -p $O
./tools/ubench/ffma2_forms > $O/ffma2_forms.txt 2>&1
python tools/prof_fmm.py --n 20000 --direct --reps 1 > /dev/null 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:direct_kernel -c 1 -f -o $O/direct python tools/prof_fmm.py --n 20000 --direct --reps 1 > $O/ncu.log 2>&1
ncu -i $O/direct.ncu-rep --page raw --csv > $O/direct_raw.csv 2>/dev/null
ncu -i $O/direct.ncu-rep --page details --csv > $O/direct_details.csv 2>/dev/null
ncu -i $O/direct.ncu-rep --page source --csv > $O/direct_source.csv 2>/dev/null
rm -f $O/direct.ncu-rep
