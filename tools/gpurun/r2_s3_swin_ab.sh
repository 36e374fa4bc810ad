python tools/ab_step.py --preset rev-swin-b --rounds 2 --window
