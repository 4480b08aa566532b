"""Workload shapes of BASELINE.json's five configs (SURVEY.md §8(a) size table).

Shapes and hyper-parameters only; no method arithmetic.
  beta: PAPER.md:445 (TLDR 0.1), :516 (No Robots 0.03), :636 (GSM8k 0.05)
  eos penalty: PAPER.md:434-435 (-1.0), :518-519 (-10.0)
  response lengths: BASELINE.json (TLDR 53, reading R11), PAPER.md:517 (1024), :631 (512)
"""
from dataclasses import dataclass


@dataclass(frozen=True)
class Workload:
    name: str
    P: int            # prompts (pairs)
    K: int            # completions per prompt
    T: int            # response length
    V: int            # vocabulary
    dtype: str        # "f32" | "bf16"
    beta: float
    eos_penalty: float | None
    reward_kind: str  # "rm" | "verifier"
    lbar: int | None  # mean response length for the prefix-mask variant

    @property
    def B(self) -> int:
        return 2 * self.P

    @property
    def rows(self) -> int:
        return self.B * self.T

    @property
    def elems(self) -> int:
        return self.rows * self.V

    @property
    def s_in(self) -> int:
        return 4 if self.dtype == "f32" else 2


CONFIGS = {
    "tiny": Workload("tiny", 4, 2, 53, 50304, "f32", 0.05, -1.0, "rm", 26),
    "pythia": Workload("pythia", 256, 2, 53, 50304, "bf16", 0.1, -1.0, "rm", 26),
    "rho": Workload("rho", 128, 2, 512, 32000, "bf16", 0.05, None, "verifier", 256),
    "llama": Workload("llama", 64, 2, 1024, 128256, "bf16", 0.03, -10.0, "rm", 290),
    # GSM8k as the paper ran it (App A.3): 63 prompts x 4 completions
    # (batch 252), the best and worst of each prompt trained on (NEXT-1)
    "rho_k4": Workload("rho_k4", 63, 4, 512, 32000, "bf16", 0.05, None, "verifier", 256),
    # strong-scaling sweep: 2048 pairs in LLaMA-shaped 64-pair chunks
    "strong": Workload("strong", 2048, 2, 1024, 128256, "bf16", 0.03, -10.0, "rm", 290),
}

CONFIG_TEXT = {
    "tiny": "tiny TLDR-shaped Online DPO: 4 prompts×2 completions, response len 53, V=50304 (Pythia), fp32 logits, β=0.05",
    "pythia": "Pythia-2.8B TLDR shape: 256 prompts×2, response len 53, V=50304, bf16 logits, staleness N=1 reference log-probs",
    "rho": "Rho-1B GSM8k shape: 128 prompts×2 samples, response len 512, V=32000, bf16 logits",
    "llama": "LLaMA-3.1-8B No Robots shape: 64 prompts×2, response len 1024, V=128256, bf16 logits",
    "rho_k4": "Rho-1B GSM8k as run in App A.3: 63 prompts x 4 completions (batch 252), best/worst pair, T 512, V 32000, bf16",
    "strong": "strong-scaling sweep: 2048 pairs, response len 1024, V=128256, bf16, batch-sharded over 1/2/4/8 B200",
}
