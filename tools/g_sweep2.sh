for shape in "256 32 20" "1024 256 50" "512 64 50" "4096 128 40" "4096 512 60" "32768 512 60"; do
  for g in 4 8 16 32; do timeout 120 python tools/g_sweep.py $shape $g 2>&1 | tail -1; done
done
