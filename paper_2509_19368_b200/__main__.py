"""Command line: `python -m paper_2509_19368_b200 decode ...`

The `decode` subcommand keeps the flags, output and exit codes of the
reference's `specpipe decode` (pkg/src/specpipe/cli.py:183-226, 264-280,
284-291) and runs on the B200 engine. `--model` extends it to the
transformer models (the reference only has the ToyLM).
"""

from __future__ import annotations

import argparse
import sys

from . import __version__
from .decode import decode_autoregressive, decode_eesd, decode_ppsd
from .models import ToyLM, TransformerConfig, TransformerLM
from .pipeline import PipelineConfig, default_prompt
from .rng import RngStream, derive_seed


def _print_kv(pairs) -> None:
    width = max(len(k) for k, _ in pairs)
    for key, value in pairs:
        if isinstance(value, float):
            value = format(value, ".6g")
        print(f"{key:<{width}}  {value}")


def _parse_prompt(text: str, vocab: int) -> list[int]:
    try:
        toks = [int(part) for part in text.split(",") if part.strip() != ""]
    except ValueError:
        raise ValueError(f"prompt must be comma-separated integers, got {text!r}")
    if not toks:
        raise ValueError("prompt must contain at least one token")
    for t in toks:
        if not 0 <= t < vocab:
            raise ValueError(f"prompt token {t} outside vocab of {vocab}")
    return toks


def _model(args):
    if args.model == "toy":
        return ToyLM(n_layers=args.n_layers, vocab=args.vocab, seed=derive_seed(args.seed, "lm"),
                     misalignment=args.beta)
    presets = {"tiny": TransformerConfig.tiny, "7b": TransformerConfig.llama2_7b,
               "13b": TransformerConfig.llama2_13b, "70b": TransformerConfig.llama2_70b}
    config = presets[args.model]() if args.model == "tiny" else presets[args.model](max_ctx=args.max_ctx)
    if config.n_layers != args.n_layers:
        raise ValueError(f"--n-layers {args.n_layers} does not match the {args.model} model ({config.n_layers})")
    return TransformerLM(config, seed=args.seed, deep_scale=args.beta, deep_from=args.exit_depth)


def _cmd_decode(args) -> int:
    pipe = PipelineConfig(n_layers=args.n_layers, exit_depth=args.exit_depth, exit_stage=args.exit_stage,
                          comm_latency=args.comm_latency)
    lm = _model(args)
    rng = RngStream(derive_seed(args.seed, "run"))
    prompt = _parse_prompt(args.prompt, lm.vocab) if args.prompt is not None else default_prompt(lm.vocab, rng)
    if args.gamma:
        tokens, metrics, trace = decode_eesd(lm, pipe, prompt, args.max_tokens, args.gamma)
        tokens = tokens[: args.max_tokens]
    else:
        tokens, metrics, trace = decode_ppsd(lm, pipe, prompt, args.max_tokens, args.mode, rng,
                                             force_reject=args.force_reject)
    print("tokens:", " ".join(str(t) for t in tokens))
    _print_kv([("committed", metrics.committed_tokens), ("ticks", metrics.ticks), ("accepts", metrics.accepts),
               ("rejects", metrics.rejects), ("throughput", metrics.throughput),
               ("speedup_vs_ar", metrics.speedup_vs_ar)])
    if args.check_ar:
        reference = decode_autoregressive(lm, prompt, args.max_tokens, args.mode,
                                          RngStream(derive_seed(args.seed, "run")))
        same = reference == tokens
        print(f"matches_autoregressive  {same}")
        if not same:
            return 1
    if args.trace_out:
        trace.write_csv(args.trace_out)
        print(f"trace -> {args.trace_out}")
    return 0


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_2509_19368_b200",
                                     description="B200 engine for pipeline-parallel self-speculative decoding")
    parser.add_argument("--version", action="version", version=f"paper_2509_19368_b200 {__version__}")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("decode", help="decode with the pipelined schedule on the GPU")
    p.add_argument("--n-layers", type=int, required=True)
    p.add_argument("--exit-depth", type=int, required=True)
    p.add_argument("--exit-stage", type=int, default=None)
    p.add_argument("--comm-latency", type=int, default=0)
    p.add_argument("--vocab", type=int, default=16)
    p.add_argument("--beta", type=float, default=0.0,
                   help="ToyLM misalignment; transformer models: deep_scale of layers >= exit depth")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--mode", choices=("greedy", "sampling"), default="sampling")
    p.add_argument("--max-tokens", type=int, default=64)
    p.add_argument("--prompt", help="comma-separated token ids (default: seeded)")
    p.add_argument("--force-reject", action="store_true")
    p.add_argument("--check-ar", action="store_true")
    p.add_argument("--trace-out")
    p.add_argument("--model", choices=("toy", "tiny", "7b", "13b", "70b"), default="toy")
    p.add_argument("--max-ctx", type=int, default=1024)
    p.add_argument("--gamma", type=int, default=0, help="run the EESD baseline with this draft length instead")
    p.set_defaults(func=_cmd_decode)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except (ValueError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
