for shape in "2048 256 50" "4096 256 50" "8192 256 50" "16384 256 50" "32768 256 50" "4096 64 60" "32768 64 60" "131072 64 60"; do
  for g in 4 8 16 32; do timeout 120 python tools/g_sweep.py $shape $g 2>&1 | tail -1; done
done
