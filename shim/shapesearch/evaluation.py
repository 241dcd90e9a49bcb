"""shapesearch.evaluation on the B200 path (paper_1604_01879_b200.evaluation)."""
from paper_1604_01879_b200.evaluation import *  # noqa: F401,F403
from paper_1604_01879_b200 import evaluation as _m

globals().update({k: v for k, v in vars(_m).items() if not k.startswith("__")})

# report writers (off the GPU path): the reference's own
from ._ref import fill_missing  # noqa: E402

fill_missing(globals(), "evaluation", ("report_to_dict", "write_report_json", "write_pr_csv",
                                       "plot_pr_svg"))
