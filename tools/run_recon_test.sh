mkdir -p gpurun_out
python -m pytest tests/test_gpu_reconstruct.py -x -q > gpurun_out/recon_test.log 2>&1; echo "rc=$?" >> gpurun_out/recon_test.log
{ for k in 100 200; do python tools/time_recon.py 32768 32768 $k; done; python tools/time_recon.py 20000 20000 100; python tools/time_recon.py 5000 5000 50; } > gpurun_out/recon_probe.txt 2>&1
