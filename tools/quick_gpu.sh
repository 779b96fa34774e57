timeout 300 python -m pytest tests/test_gpu_model.py -x -q -k "ffn1_fusion or fused_epilogues or full_size_c3_sampled" > gpurun_out/$1_gpu.log 2>&1; echo pytest=$? >> gpurun_out/$1_gpu.log
python tools/rr_trace.py 2 > gpurun_out/$1_trace2.log 2>&1
timeout 300 python bench.py --no-variants --no-cpu-baseline --no-dynamic --no-importance --no-configs > gpurun_out/$1_bench.json 2> gpurun_out/$1_bench.err
