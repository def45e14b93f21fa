"""Time the predictor (f32->bf16, SRU stack, heads argmax) as one captured graph, with the
two-stream token-half SRU pipeline on and off."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11537_b200.engine import MoEPipeline, PipelineConfig  # noqa: E402
from tools.e2e_probe import timed  # noqa: E402


def main():
    for on in (True, False):
        cfg = PipelineConfig(sru_pipeline=on)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            pipe = MoEPipeline(cfg)
            emb, _, _ = pipe.wl.batch(cfg.tokens)
            x = emb.clone()
            pipe.predict(x, s.cuda_stream)
            g = pipe.capture_call(lambda sp: pipe.predict(x, sp))
            t = timed(g.replay, s, n=20)
        print(f"sru_pipeline={on}: predict {t * 1e3:.1f} us")
        del pipe, g
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
