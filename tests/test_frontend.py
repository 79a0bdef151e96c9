"""Host-side formats (§8f row 4): the run description of config.hpp:23-262 (strict schema,
messages, canonical echo) and its mapping onto the device config. Mirrors test_runner.cpp:54-90;
the echo is checked byte for byte against the reference's runner_out/config_echo.ini."""
import pytest

from paper_2412_19207_b200 import abi as A
from paper_2412_19207_b200 import configs
from paper_2412_19207_b200 import frontend as F


def small_config(out_dir: str) -> str:
    """The runner tests' small configuration (test_runner.cpp:13-42)."""
    return ("[problem]\nname = example1\nn = 1\n\n[decomposition]\ncounts = 2 2\ndelta = 2.0\n\n"
            "[basis]\nm = 8\nactivation = tanh\nseed = 77\n\n[points]\ncollocation = 12 12\ntest = 40 40\n\n"
            "[pca]\ntau = off\n\n[solver]\nmethod = gmres\npreconditioner = AS\nrel_tol = 1e-5\n\n"
            f"[run]\nnum_seeds = 2\nout_dir = {out_dir}\n")


def test_parse_small_config():
    cfg = F.parse_config_text(small_config("out"))
    assert cfg.problem == "example1" and cfg.n == 1
    assert cfg.counts == [2, 2] and cfg.m == 8 and cfg.seed == 77
    assert cfg.collocation == [12, 12] and cfg.test == [40, 40]
    assert not cfg.tau_on and cfg.solver == "gmres" and cfg.preconditioner == "AS"
    assert cfg.rel_tol == 1e-5 and cfg.num_seeds == 2 and cfg.out_dir == "out"
    assert cfg.ref_resolution == 2001 and cfg.pca_matrix == "operator"  # defaults (config.hpp:25-46)


def test_schema_errors():
    with pytest.raises(ValueError, match="unknown section"):
        F.parse_config_text("[bogus]\nx = 1\n")
    with pytest.raises(ValueError, match=r"unknown key 'nombre' in section \[problem\]"):
        F.parse_config_text("[problem]\nnombre = example1\n")
    with pytest.raises(ValueError, match="unknown problem 'example9'"):
        F.parse_config_text("[problem]\nname = example9\n")
    with pytest.raises(ValueError, match="unknown solver 'simplex'"):
        F.parse_config_text("[solver]\nmethod = simplex\n")
    with pytest.raises(ValueError, match="tau must be >= 0 or off"):
        F.parse_config_text("[pca]\ntau = -1\n")
    with pytest.raises(ValueError, match="outside any section"):
        F.parse_config_text("m = 3\n")
    with pytest.raises(ValueError, match="config line 1: bad section"):
        F.parse_config_text("[basis\n")
    with pytest.raises(ValueError, match="config line 2: expected key = value"):
        F.parse_config_text("[basis]\nm 3\n")
    with pytest.raises(ValueError, match="'m' expects an integer, got '3.5'"):
        F.parse_config_text("[basis]\nm = 3.5\n")
    with pytest.raises(ValueError, match="'delta' expects a number, got 'wide'"):
        F.parse_config_text("[decomposition]\ndelta = wide\n")
    with pytest.raises(ValueError, match="empty integer list for 'counts'"):
        F.parse_config_text("[decomposition]\ncounts = ,\n")
    with pytest.raises(ValueError, match="expects on/off"):
        F.parse_config_text("[run]\ndump_diagnostics = maybe\n")
    with pytest.raises(ValueError, match="activation must be tanh or sin"):
        F.parse_config_text("[basis]\nactivation = relu\n")
    with pytest.raises(ValueError, match="rel_tol must be positive"):
        F.parse_config_text("[solver]\nrel_tol = 0\n")
    with pytest.raises(ValueError, match="num_seeds must be >= 1"):
        F.parse_config_text("[run]\nnum_seeds = 0\n")
    with pytest.raises(ValueError, match="unknown preconditioner 'ILU'"):
        F.parse_config_text("[solver]\npreconditioner = ILU\n")
    with pytest.raises(RuntimeError, match="cannot open config file"):
        F.parse_config_file("/nonexistent/run.ini")


def test_comments_commas_and_pca_matrix():
    cfg = F.parse_config_text("# header\n[decomposition]  # boxes\ncounts = 3, 4  # per axis\n"
                              "[pca]\ntau = 1e-3\nmatrix = psi\n[solver]\npreconditioner = none\n")
    assert cfg.counts == [3, 4] and cfg.tau_on and cfg.tau == 1e-3 and cfg.pca_matrix == "psi"
    assert cfg.preconditioner is None and cfg.precond_label() == "none"
    assert F.parse_config_text("[pca]\nmatrix = operator\n").pca_matrix == "operator"
    with pytest.raises(ValueError, match="operator or psi"):
        F.parse_config_text("[pca]\nmatrix = fourier\n")


def test_echo_matches_reference_and_round_trips(golden):
    cfg = F.parse_config_text(small_config("runner_out"))
    echo = F.config_echo(cfg)
    assert echo == golden["runner_config_echo"]
    again = F.parse_config_text(echo)
    assert again == cfg
    assert F.config_echo(again) == echo
    cfg2 = F.parse_config_text("[pca]\ntau = 0.001\n[solver]\nmethod = cg\npreconditioner = RAS\n")
    assert "tau = 0.001\n" in F.config_echo(cfg2) and F.parse_config_text(F.config_echo(cfg2)) == cfg2


def test_device_config_mapping():
    cfg = F.parse_config_text(small_config("out"))
    got = cfg.to_abi(77)
    want = configs.golden_runner(77)
    assert got.ref_resolution == 2001  # config.hpp:28 default, carried to the device
    want.ref_resolution = 2001
    assert bytes(got) == bytes(want)
    sweep = F.parse_config_text(small_config("out") + "[basis]\nm = 12\n[pca]\ntau = 0.01\n")
    want = configs.golden_sweep(1e-2, 78)
    want.ref_resolution = 2001
    assert bytes(sweep.to_abi(78)) == bytes(want)
    assert sweep.to_abi().seed == 77


def test_summary_row_format():
    cfg = F.parse_config_text(small_config("out"))
    s = {"seed": 77, "J": 4, "DoF": 32, "N": 144, "iterations": 1, "converged": 1, "e_l2": 0.012010649881234,
         "e_l1n": 0.0089180459571, "t_assemble": 0.001055938, "t_precond": 0.000359458, "t_solve": 8.6618e-05}
    assert F.summary_row(cfg, s) == ("77,example1,4,32,144,gmres,AS,off,1,1,0.01201064988,0.008918045957,"
                                     "0.001055938,0.000359458,8.6618e-05")
    assert F.K_SUMMARY_HEADER.split(",")[0] == "seed" and len(F.K_SUMMARY_HEADER.split(",")) == 15


def test_scaling_caps():
    with pytest.raises(ValueError, match="n must be >= 2"):
        F.scaling_cmd(F.RunConfig(), [1], solver=object())
    with pytest.raises(ValueError, match="desk-scale cap"):
        F.scaling_cmd(F.RunConfig(), [5], solver=object())
    assert A.SOLVER_NAMES[F._SOLVERS["bicg"]] == "bicg"
