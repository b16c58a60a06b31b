import sys
sys.path.insert(0, ".")
exec(open("tools/qr_micro.py").read().replace("for m, k, full, cl in [(352, 256, 1, 1), (352, 256, 1, 8), (352, 256, 0, 8), (256, 200, 0, 1), (256, 200, 0, 8), (2048, 112, 0, 8), (8192, 48, 0, 8)]:", "for m, k, full, cl in [(8192, 48, 0, 1)]:"))
