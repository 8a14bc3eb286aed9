#!/bin/bash
O=gpurun_out/ab1; mkdir -p $O
./tools/atomics_bench > $O/atomics.json 2>&1
for lib in base inc1 noret inc1noret; do
  if [ $lib = base ]; then unset TEXFORGE_CUDA_LIB; else export TEXFORGE_CUDA_LIB=$PWD/tools/ab/lib_$lib.so; fi
  timeout 300 python tools/profile_vote.py --levels 256 --dts 1:0,1:45,1:90,1:135 --reps 5 --time > $O/${lib}_L256.json 2>&1
done
unset TEXFORGE_CUDA_LIB
timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,smsp__inst_executed_op_shared_atom.sum,sm__cycles_elapsed.avg,l1tex__throughput.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_lg.sum --clock-control none -k regex:bench ./tools/atomics_bench > $O/ncu_atomics.txt 2>&1
timeout 600 ncu --set full --clock-control none -k regex:glcm_vote -c 1 python tools/profile_vote.py --levels 256 --kinds noise --dts 1:0 --reps 1 > $O/ncu_vote256_full.txt 2>&1
