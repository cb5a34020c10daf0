"""One fused split migration (13B, 8k tokens, s = 1 456) after 3 warm-ups, for
`ncu --set full -k regex:reprefill_pair --launch-skip 3 -c 1`."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2501_06709_b200.kvcache import LLAMA2_13B, KVPool  # noqa: E402
from paper_2501_06709_b200.reprefill import synthetic_hidden, synthetic_weights  # noqa: E402
from paper_2501_06709_b200.split import make_split, split_migrate_fused  # noqa: E402


def main():
    sh = LLAMA2_13B
    plan = make_split(8192, 1456)
    nb = plan.total_blocks + 16
    src, dst = KVPool(sh, nb, dtype=torch.bfloat16), KVPool(sh, nb, dtype=torch.bfloat16)
    sb = torch.randperm(nb, generator=torch.Generator().manual_seed(1))[:plan.total_blocks].to(torch.int32).cuda()
    db = torch.arange(plan.total_blocks, dtype=torch.int32, device="cuda")
    x, w = synthetic_hidden(sh, 1456, 0), synthetic_weights(sh, 0, with_q=True)
    for _ in range(4):
        split_migrate_fused(src, dst, sb, db, plan, x, w)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
