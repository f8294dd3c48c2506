timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2z_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/r2z_tests.log
timeout 900 bash tools/profile_round.sh r2z > /dev/null 2>&1; echo "profile rc $?"; ls gpurun_out | grep r2z
