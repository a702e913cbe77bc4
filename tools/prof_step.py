"""Run the bench step a few times (for ncu launch lists / captures). No timing output."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench

if __name__ == "__main__":
    sys.argv = [sys.argv[0], "--steps", os.environ.get("STEPS", "2"), "--warmup", "1", "--no-e2e", "--no-cpu",
                "--config", os.environ.get("CONFIG", "c2"), "--no-graph"]
    bench.main()
