# Device synth_noise check + timing, and the bench workloads that use it for input generation (run under gpurun).
mkdir -p gpurun_out/synth
timeout 900 python -m pytest tests/test_synth_device.py -q -m gpu > gpurun_out/synth/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/synth/pytest.log
timeout 300 python - > gpurun_out/synth/timing.txt 2>&1 <<'PY'
import time, torch, numpy as np
from paper_1710_06189_b200 import texforge as tf
eng = tf.Engine(0)
for (w, h) in [(16384, 16384), (65536, 65536)]:
    eng.synth_noise_device(w, 1024, 1); torch.cuda.synchronize()
    t = time.time(); out = eng.synth_noise_device(w, h, 1); torch.cuda.synchronize(); dt = time.time() - t
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); eng.synth_noise_device(w, h, 1, out=out); e1.record(); torch.cuda.synchronize()
    t = time.time(); ref = tf.synth_noise(w, h, 1).pixels; dh = time.time() - t
    print(w, h, "device %.3f s wall (incl. host jump-ahead), %.1f ms between events" % (dt, e0.elapsed_time(e1)),
          "host (all threads) %.3f s" % dh, "equal", np.array_equal(out.cpu().numpy(), ref))
    del out, ref
PY
for w in c3 c5 c4; do s=$(date +%s.%N); timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --cpu-seconds 5 > gpurun_out/synth/bench_$w.json 2> gpurun_out/synth/bench_$w.err; echo "$w $(echo "$(date +%s.%N) - $s" | bc) s wall" >> gpurun_out/synth/walls.txt; done
