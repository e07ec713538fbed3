python __graft_entry__.py > gpurun_out/fin2_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 -rA > gpurun_out/fin2_tests.log 2>&1
tail -1 gpurun_out/fin2_tests.log
