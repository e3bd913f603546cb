cd $GRAFT_REPO_ROOT && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_c_client.py -q -m gpu > gpurun_out/pytest_c_client.log 2>&1
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_decode.py -q -m gpu -k "fuzz_vs_oracle or sharded or decoder_side or for_device or pipeline or partitioned or every_prob_bits or single_symbol" > gpurun_out/san_memcheck_decode.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san_memcheck_decode.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_adaptive.py -q -m gpu -k "random_models and not 1048576 and not 777777" > gpurun_out/san_memcheck_adaptive.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san_memcheck_adaptive.log
tail -3 gpurun_out/pytest_c_client.log; tail -3 gpurun_out/san_memcheck_decode.log; tail -3 gpurun_out/san_memcheck_adaptive.log
