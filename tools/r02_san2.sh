# memcheck / racecheck over the kernels changed in round 2's last sessions (select shapes, split walk, sketch waves / ring)
set -u
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_decode.py tests/test_gpu_splitkv.py -m gpu -q -x -k "c2_shape or c3_shape or gqa_decode_small or W or dynamic" > gpurun_out/san2_memcheck.log 2>&1; tail -3 gpurun_out/san2_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_decode.py -m gpu -q -x -k "c2_shape" > gpurun_out/san2_racecheck.log 2>&1; tail -3 gpurun_out/san2_racecheck.log
