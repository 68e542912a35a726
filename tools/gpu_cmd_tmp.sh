REPS=3 STEPS=30 bash tools/ab_run.sh ab_mixy.txt "8 12" cur my1 my2 my3
