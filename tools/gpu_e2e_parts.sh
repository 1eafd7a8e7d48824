set -x
timeout 600 python tools/time_e2e_parts.py > gpurun_out/e2e_parts.log 2>&1; echo parts $?
timeout 600 python tools/prof_build.py > gpurun_out/prof_build.log 2>&1; echo pb $?
tail -30 gpurun_out/e2e_parts.log; tail -40 gpurun_out/prof_build.log
