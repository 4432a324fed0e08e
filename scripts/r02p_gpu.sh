#!/bin/bash
set -x
O=gpurun_out
for V in 8 4; do
  EPC_PCG_CPW=$V python scripts/probe_gn.py --config C3 > $O/r02p_gn_c3_cpw$V.log 2>&1
done
EPC_PCG_CPW=4 python -m pytest tests/test_gpu_gn.py -q > $O/r02p_gn_tests_cpw4.log 2>&1
grep -h "unprofiled\|pcg_update \|pcg_hvp " $O/r02p_gn_c3_cpw*.log
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 1 --warmup 1 --no-gn --no-f32 --no-x400 --no-cpu-baseline --sharded > $O/r02p_sharded.json 2> $O/r02p_sharded.err
tail -c 1500 $O/r02p_sharded.json
for i in 1 2; do
for V in now kktout cell2 laneun kktcell2; do
  if [ $V = now ]; then L=""; else L="EPC_LIB=scripts/_var/$V.so"; fi
  env $L python scripts/probe_admm.py --config C3 --iters 100 --prod > $O/r02p_c3_${V}_$i.log 2>&1
done
done
for f in $O/r02p_c3_*.log; do echo "$f $(grep admm_bstep $f | awk '{print $2}')"; done
