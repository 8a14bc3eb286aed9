# A/B sweep of kernel builds in tools/ab/lib_*.so vs the in-tree library (run under gpurun).
mkdir -p gpurun_out/ab
for lib in base tools/ab/lib_*.so; do
  name=$(basename $lib .so)
  if [ $lib = base ]; then unset TEXFORGE_CUDA_LIB; else export TEXFORGE_CUDA_LIB=$PWD/$lib; fi
  for L in ${AB_LEVELS:-256 32}; do timeout 300 python tools/profile_vote.py --levels $L --dts 1:0,1:45,2:90,4:135 --reps 5 --time > gpurun_out/ab/${name}_L$L.json 2>&1; done
done
