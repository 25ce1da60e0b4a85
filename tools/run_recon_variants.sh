mkdir -p gpurun_out
cp paper_1108_5359_b200/_lib/libl1pcp_b200.so /tmp/main.so
{
for f in tools/variants/*.so; do
  cp $f paper_1108_5359_b200/_lib/libl1pcp_b200.so
  echo "== $f"
  for k in 100 200; do python tools/time_recon.py 32768 32768 $k; done
  python tools/time_recon.py 20000 20000 100
done
} > gpurun_out/recon_variants.txt 2>&1
cp /tmp/main.so paper_1108_5359_b200/_lib/libl1pcp_b200.so
