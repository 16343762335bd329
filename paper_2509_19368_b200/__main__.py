"""Command line: `python -m paper_2509_19368_b200 {analytic,run,sweep,decode,trace} ...`

Keeps the subcommands, flags, output and exit codes of the reference's
`specpipe` CLI (pkg/src/specpipe/cli.py:39-291); `run` / `sweep` / `trace`
go through harness.py onto the GPU tick machine, `decode` runs on the B200
engine. `decode --model` extends it to the transformer models (the reference
only has the ToyLM). Config or usage errors: `error: ...` on stderr, exit 2.
"""

from __future__ import annotations

import argparse
import json
import sys

from . import __version__
from . import harness as H
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


_CONFIG_FIELDS = ("regime", "n_layers", "exit_depth", "exit_stage", "comm_latency", "horizon", "gamma", "oracle",
                  "alpha", "beta", "vocab", "seed", "steady_state", "out", "trace_out")


def _config_flags(p) -> None:
    p.add_argument("--config", metavar="JSON", help="experiment config file")
    p.add_argument("--regime", choices=H.REGIMES)
    for name in ("n-layers", "exit-depth", "exit-stage", "comm-latency", "horizon", "gamma"):
        p.add_argument(f"--{name}", type=int)
    p.add_argument("--oracle", choices=H.ORACLES)
    p.add_argument("--alpha", type=float)
    p.add_argument("--beta", type=float)
    p.add_argument("--vocab", type=int)
    p.add_argument("--seed", type=int)
    p.add_argument("--steady-state", action="store_const", const=True, default=None,
                   help="subtract pipeline warm-up ticks from the rates")
    p.add_argument("--out", help="write the results CSV here")
    p.add_argument("--trace-out", help="write the event trace CSV here")
    p.add_argument("--dump-config", action="store_true",
                   help="print the effective config as JSON and exit without running")


def _config(args) -> H.ExperimentConfig:
    data = H.ExperimentConfig.from_json(args.config).to_dict() if args.config else {}
    for name in _CONFIG_FIELDS:  # a flag wins over the file
        v = getattr(args, name)
        if v is not None:
            data[name] = v
    return H.ExperimentConfig.from_dict(data)


def _cmd_analytic(args) -> int:
    print(H.analytic_report(alpha=args.alpha, gamma=args.gamma, n_layers=args.n_layers,
                            exit_depth=args.exit_depth, t_target=args.t_target, t_draft=args.t_draft))
    return 0


def _cmd_run(args, need_trace: bool = False) -> int:
    cfg = _config(args)
    if need_trace and not cfg.trace_out:
        raise H.ConfigError("trace_out", "the trace subcommand needs --trace-out")
    if args.dump_config:
        print(json.dumps(cfg.to_dict(), indent=2, sort_keys=True))
        return 0
    res = H.run(cfg)
    m = res.metrics
    pairs = [("regime", cfg.regime), ("committed", m.committed_tokens), ("ticks", m.ticks),
             ("accepts", m.accepts), ("rejects", m.rejects)]
    if m.alpha_all_measured is not None:
        pairs.append(("alpha_all", m.alpha_all_measured))
    pairs += [("throughput", m.throughput), ("speedup_vs_ar", m.speedup_vs_ar)]
    if res.analytic_speedup is not None:
        pairs.append(("analytic_speedup", res.analytic_speedup))
    _print_kv(pairs)
    if cfg.out:
        print(f"results -> {H.resolve_out_path(cfg.out)}")
    if cfg.trace_out:
        print(f"trace   -> {H.resolve_out_path(cfg.trace_out)}")
    return 0


def _cmd_sweep(args) -> int:
    results = H.sweep(H.SweepSpec.from_json(args.config))
    if args.out:
        path = H.resolve_out_path(args.out)
        H.write_results_csv(results, path)
        print(f"{len(results)} rows -> {path}")
    else:
        print(H.RESULTS_HEADER)
        for r in results:
            print(H.result_row(r))
    return 0


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_2509_19368_b200",
                                     description="B200 engine for pipeline-parallel self-speculative decoding")
    parser.add_argument("--version", action="version", version=f"paper_2509_19368_b200 {__version__}")
    sub = parser.add_subparsers(dest="command", required=True)
    pa = sub.add_parser("analytic", help="print closed-form quantities")
    pa.add_argument("--alpha", type=float, required=True)
    pa.add_argument("--gamma", type=int, required=True)
    pa.add_argument("--n-layers", type=int, required=True)
    pa.add_argument("--exit-depth", type=int, required=True)
    pa.add_argument("--t-target", type=float, default=1.0)
    pa.add_argument("--t-draft", type=float, default=None)
    pa.set_defaults(func=_cmd_analytic)
    pr = sub.add_parser("run", help="execute one experiment")
    _config_flags(pr)
    pr.set_defaults(func=_cmd_run)
    ps = sub.add_parser("sweep", help="run a sweep spec")
    ps.add_argument("--config", metavar="JSON", required=True, help="sweep spec file")
    ps.add_argument("--out", help="combined results CSV (default: stdout)")
    ps.set_defaults(func=_cmd_sweep)
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
    pt = sub.add_parser("trace", help="run one experiment for its event trace")
    _config_flags(pt)
    pt.set_defaults(func=lambda a: _cmd_run(a, need_trace=True))
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
