#!/bin/bash
# Round-2 GPU session helper (run under gpurun). Stages: smoke pytest bench_c3 bench_c5 bench_c4 bench_c2 bench_c1 ref_c3 ref_c5
mkdir -p gpurun_out/r02
O=gpurun_out/r02
for s in "$@"; do
  case $s in
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log ;;
    pytest) timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log ;;
    pytest_k=*) timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -k "${s#pytest_k=}" > $O/pytest_k.log 2>&1; echo "rc=$?" >> $O/pytest_k.log ;;
    bench_*) wl=${s#bench_}; timeout 1200 python bench.py --workload $wl --steps 10 --warmup 3 > $O/bench_$wl.json 2> $O/bench_$wl.err; echo "rc=$?" >> $O/bench_$wl.err ;;
    ref_*) wl=${s#ref_}; timeout 1200 python bench.py --impl reference --workload $wl --steps 5 --warmup 3 > $O/ref_$wl.json 2> $O/ref_$wl.err; echo "rc=$?" >> $O/ref_$wl.err ;;
    cpp) for b in dropin_tests refsuite_unit refsuite_accept; do timeout 900 tests/cpp/_build/$b > $O/cpp_$b.log 2>&1; echo "rc=$?" >> $O/cpp_$b.log; done ;;
  esac
done
