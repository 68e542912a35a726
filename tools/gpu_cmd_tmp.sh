REPS=3 STEPS=30 bash tools/ab_run.sh ab_wpf.txt "4 8 12" cur nopf
