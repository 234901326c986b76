# 1 GPU: what the driver runs at round end -- pytest -m gpu, smoke(), default bench (timed), reference arm
( time timeout 2400 python -m pytest tests -x -q -p no:cacheprovider -m gpu ) > gpurun_out/r02cc_tests.log 2>&1; echo rc=$? >> gpurun_out/r02cc_tests.log
( time python -c "import __graft_entry__ as g; g.smoke()" ) > gpurun_out/r02cc_smoke.log 2>&1; echo rc=$? >> gpurun_out/r02cc_smoke.log
( time python bench.py ) > gpurun_out/r02cc_bench.json 2> gpurun_out/r02cc_bench.err
( time python bench.py --impl reference ) > gpurun_out/r02cc_ref.json 2> gpurun_out/r02cc_ref.err
echo done
