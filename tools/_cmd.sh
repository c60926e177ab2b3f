DOCTEST_SKIP=drag timeout 900 tests/cpp/build/ref_unit_tests > gpurun_out/ref_unit2.log 2>&1; echo rc=$? >> gpurun_out/ref_unit2.log
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t18.log 2>&1; echo rc=$? >> gpurun_out/t18.log
