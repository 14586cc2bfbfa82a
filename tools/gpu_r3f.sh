# k_cheb2s with a 4-plane u0 ring where it fits: A/B (alternating) vs the 3-plane build
mkdir -p gpurun_out
bash tools/ab.sh ab/libsrfmg_base.so > gpurun_out/ab_ru64.txt 2>&1
