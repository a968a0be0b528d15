# usage: OPS=Resize512 KREGEX=k_resample_q4 TAG=x bash tools/gpu_ncu_one.sh
# one ncu --set full capture (source-correlated) of the first matching kernel
set -x
OPS=${OPS:-Resize512}; KREGEX=${KREGEX:-k_}; TAG=${TAG:-one}; N=${N:-2000}
python tools/profile_ops.py --ops $OPS --reps 1 --n $N > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$KREGEX" -c ${COUNT:-1} -o gpurun_out/full_$TAG python tools/profile_ops.py --ops $OPS --reps 1 --n $N > gpurun_out/ncu_$TAG.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_$TAG.log
