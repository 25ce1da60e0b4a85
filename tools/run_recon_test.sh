mkdir -p gpurun_out
python -m pytest tests/test_gpu_reconstruct.py -x -q > gpurun_out/recon_test.log 2>&1; echo "rc=$?" >> gpurun_out/recon_test.log
bash tools/run_recon_probe.sh
