bash tools/scale_run.sh
bash tools/scale_1p5m.sh
