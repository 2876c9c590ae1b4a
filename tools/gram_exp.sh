# K1 sensitivity experiments (HYDE_GRAM_EXP: 1 no MMAs, 2 no T_bb MMAs, 4 no conversion; results are wrong, timing only)
for v in "" "HYDE_GRAM_EXP=1" "HYDE_GRAM_EXP=2" "HYDE_GRAM_EXP=4" "HYDE_GRAM_EXP=5" "HYDE_GRAM_NO_TMA=1" "HYDE_GRAM_NO_TMA=1 HYDE_GRAM_EXP=1" "HYDE_GRAM_NO_TMA=1 HYDE_GRAM_EXP=4"; do
  echo "== $v"; env $v python tools/run_gram.py large
done
