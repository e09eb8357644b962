for np in 2 4; do
for pc in 1 2 4 8; do
  bash tools/mp_sweep.sh n${np}_p${pc} $np TGB_PIECES=$pc
done
done
