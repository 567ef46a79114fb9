mkdir -p gpurun_out
H2G_NO_SMALL_TILES=1 timeout 400 python scripts/try_config.py 4 reference 1e-2 64 2>&1 | grep -E "factorize wall|relative residual|levels" > gpurun_out/bis_nosmall.log
timeout 400 python scripts/try_config.py 4 reference 1e-2 1 2>&1 | grep -E "factorize wall|relative residual|levels" > gpurun_out/bis_small_solve.log
