for shape in "256 32 20" "1024 256 50" "512 64 50" "4096 128 40" "4096 512 60" "32768 512 60"; do
  for g in 4 8 16 32; do BSSMPPI_FORCE_G=$g timeout 120 python tools/g_sweep.py $shape 2>&1 | tail -1; done
done
