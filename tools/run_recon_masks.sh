mkdir -p gpurun_out
{ for mask in 0 1 2 4 6 7; do L1F_RECON_TC_MASK=$mask python tools/time_recon.py 20000 20000 100; done; for mask in 0 6 7; do L1F_RECON_TC_MASK=$mask python tools/time_recon.py 32768 32768 200; done; } > gpurun_out/recon_masks.txt 2>&1
