for v in 3 0 3 0; do for np in 4 2; do bash tools/mp_sweep.sh k2v${v}b_n$np $np TGB_K2V=$v; done; done
