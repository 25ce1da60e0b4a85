mkdir -p gpurun_out
{
for k in 100 200; do
  for mask in 0 7; do
    L1F_RECON_TC_MASK=$mask python tools/time_recon.py 32768 32768 $k
  done
done
} > gpurun_out/recon_probe.txt 2>&1
