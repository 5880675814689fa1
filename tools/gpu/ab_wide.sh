export PYTHONPATH=$PWD; mkdir -p gpurun_out/s2
./tools/ubench/ffma2 > gpurun_out/s2/ffma2.txt 2>&1
Q="--no-cpu --no-p2p --no-p10 --no-stress --no-gmres --no-gmres-paper"
for i in 1 2; do
python bench.py $Q > gpurun_out/s2/wide_$i.json 2>&1
EBEM_M2L_WIDE=0 python bench.py $Q > gpurun_out/s2/narrow_$i.json 2>&1
done
