"""The command line front end (cli.py, mirroring tools/main.cpp): the
GPU-free subcommand (rank-configs) against the compiled reference's ranking,
argument errors and exit codes (main.cpp:20-24). preprocess / train run on
the GPU (tests/test_cli_gpu.py)."""

import pytest

from oracle import ref
from paper_2505_04083_b200 import cli


def test_rank_configs_stats_matches_reference(capsys, tmp_path):
    csv = tmp_path / "r.csv"
    rc = cli.main(["rank-configs", "--stats", "n=2097152,nnz=116573894,dims=100-256-256-47",
                   "--g", "8", "--csv", str(csv)])
    assert rc == 0
    out = capsys.readouterr().out.strip().splitlines()
    assert out[0] == "gx,gy,gz,spmm_s,comm_s,total_s"
    got = [tuple(int(x) for x in line.split(",")[:3]) for line in out[1:]]
    want = [tuple(int(x) for x in row[:3]) for row in ref.rank_configs(
        8, 2097152, 116573894, [100, 256, 256, 47])]
    assert got == want
    assert csv.read_text().splitlines()[0] == "gx,gy,gz,spmm_s,comm_s,total_s,clamped"


@pytest.mark.parametrize("argv,code", [
    (["rank-configs", "--g", "8"], 2),                          # no --manifest / --stats
    (["rank-configs", "--stats", "n=1,nnz=2", "--g", "4"], 2),   # no dims
    (["rank-configs", "--stats", "n=5,nnz=9,dims=4-4", "--g", "4",
      "--machine", "/nonexistent.json"], 2),                     # missing machine file
    (["train", "--manifest", "/nonexistent"], 2),                # missing manifest
    (["preprocess", "--out", "/tmp/x"], 2),                      # neither --edges nor --synth
    (["preprocess", "--synth", "kron:n=5", "--out", "/tmp/x"], 2),  # unknown synth kind
])
def test_exit_codes(argv, code):
    assert cli.main(argv) == code


def test_parse_synth():
    assert cli.parse_synth("rmat:scale=9,edges=3000") == ("rmat", {"scale": 9.0, "edges": 3000.0})
    with pytest.raises(cli.CliError):
        cli.parse_synth("rmat:scale")


def test_parse_synth_pair_kinds():
    """tools/main.cpp:70-93 parameter names of the sbm / erdos kinds"""
    assert cli.parse_synth("sbm:n=4096,k=8,p_in=0.2,p_out=0.001") == (
        "sbm", {"n": 4096.0, "k": 8.0, "p_in": 0.2, "p_out": 0.001})
    assert cli.parse_synth("erdos:n=50,p=0.1") == ("erdos", {"n": 50.0, "p": 0.1})
