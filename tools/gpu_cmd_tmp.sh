REPS=3 STEPS=30 bash tools/ab_run.sh ab_fu.txt "8 12" cur fu2 fu3
