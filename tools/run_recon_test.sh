mkdir -p gpurun_out
python -m pytest tests/test_gpu_reconstruct.py -x -q > gpurun_out/recon_test.log 2>&1; echo "rc=$?" >> gpurun_out/recon_test.log
{ for mask in 0 6 7; do L1F_RECON_TC_MASK=$mask python tools/time_recon.py 20000 20000 100; done; for mask in 0 7; do L1F_RECON_TC_MASK=$mask python tools/time_recon.py 32768 32768 200; done; python tools/time_recon.py 5000 5000 50; } > gpurun_out/recon_probe.txt 2>&1
