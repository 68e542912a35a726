REPS=2 STEPS=30 bash tools/ab_run.sh ab_seg.txt "8 10 12" cur seg16 seg32
